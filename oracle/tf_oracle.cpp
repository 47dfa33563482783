// tf_oracle.cpp — TEST INFRASTRUCTURE ONLY: the CPU parity checker.
//
// A restatement (not a copy) of the reference's algorithm for the Snake-NeRF
// window hot path.  Each function cites the reference file:line it follows
// (paths relative to /root/reference/proj/src/core/ unless marked SPEC).
// Built with `-O3 -DNDEBUG -ffp-contract=off` (reference Release flags,
// CMakeLists.txt:6-8, minus FMA contraction) so double/float rounding happens
// once per source operation, which is the contract the CUDA path reproduces.
#include "tf_oracle.h"

#include <algorithm>
#include <array>
#include <climits>
#include <cstdint>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <map>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace {

thread_local std::string g_err;

struct OracleError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// ---------------------------------------------------------------- rng.hpp:11-48
inline uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}
inline uint64_t hc(uint64_t a, uint64_t b) {
    return splitmix64(a ^ (b + 0x9e3779b97f4a7c15ull + (a << 6) + (a >> 2)));
}
template <typename... R>
uint64_t hc(uint64_t a, uint64_t b, R... r) {
    return hc(hc(a, b), uint64_t(r)...);
}
struct Rng {
    uint64_t s;
    explicit Rng(uint64_t seed) : s(splitmix64(seed)) {}
    uint64_t u64() { return s = splitmix64(s); }
    double dbl() { return double(u64() >> 11) * 0x1.0p-53; }
    float flt() { return float(u64() >> 40) * 0x1.0p-24f; }
    uint64_t below(uint64_t n) { return uint64_t(((unsigned __int128)u64() * n) >> 64); }
    double uniform(double lo, double hi) { return lo + (hi - lo) * dbl(); }
};

// Stream purposes (DESIGN.md pins; rng.hpp:8-10 derives streams from
// (seed, purpose, counters)).
constexpr uint64_t kPurposePixels = 0x5049584Cull;   // "PIXL"
constexpr uint64_t kPurposeJitter = 0x4A495454ull;   // "JITT"
constexpr uint64_t kPurposeTileEnc = 0x54454E43ull;  // "TENC"
constexpr uint64_t kPurposeTileDnet = 0x54444E54ull; // "TDNT"
constexpr uint64_t kPurposeColor = 0x434F4C52ull;    // "COLR"
constexpr uint64_t kPurposeOccupancy = 0x4F434355ull; // "OCCU"

// ------------------------------------------------------------ parallel.cpp:8-34
std::pair<size_t, size_t> chunk(size_t n, int workers, int c) {
    size_t per = n / workers, rem = n % workers;
    size_t b = c * per + std::min<size_t>(c, rem);
    return {b, b + per + (size_t(c) < rem ? 1 : 0)};
}
void par_for(size_t n, int workers, const std::function<void(size_t, size_t, int)>& body) {
    if (n == 0) return;
    if (workers < 1) workers = 1;
    if (workers == 1 || n == 1) {
        body(0, n, 0);
        return;
    }
    if (size_t(workers) > n) workers = int(n);
    std::vector<std::thread> th;
    for (int c = 1; c < workers; ++c) {
        auto [b, e] = chunk(n, workers, c);
        th.emplace_back([&body, b, e, c] { body(b, e, c); });
    }
    auto [b0, e0] = chunk(n, workers, 0);
    body(b0, e0, 0);
    for (auto& t : th) t.join();
}

// ------------------------------------------------------------ camera.cpp:22-64
void rpc_terms(double P, double L, double H, double* t) {
    t[0] = 1;
    t[1] = L;
    t[2] = P;
    t[3] = H;
    t[4] = L * P;
    t[5] = L * H;
    t[6] = P * H;
    t[7] = L * L;
    t[8] = P * P;
    t[9] = H * H;
    t[10] = P * L * H;
    t[11] = L * L * L;
    t[12] = L * P * P;
    t[13] = L * H * H;
    t[14] = L * L * P;
    t[15] = P * P * P;
    t[16] = P * H * H;
    t[17] = L * L * H;
    t[18] = P * P * H;
    t[19] = H * H * H;
}
double dot20(const double* c, const double* t) {
    double s = 0;
    for (int i = 0; i < 20; ++i) s += c[i] * t[i];
    return s;
}
// Returns false where project() throws (|normalized| > 1.5, camera.hpp:32).
bool project(const tfg_rpc& c, double x, double y, double z, double* row, double* col) {
    double L = (x - c.long_off) / c.long_scale;
    double P = (y - c.lat_off) / c.lat_scale;
    double H = (z - c.height_off) / c.height_scale;
    const double lim = 1.5;
    if (!(std::abs(L) <= lim && std::abs(P) <= lim && std::abs(H) <= lim)) return false;
    double t[20];
    rpc_terms(P, L, H, t);
    double rn = dot20(c.line_num, t) / dot20(c.line_den, t);
    double cn = dot20(c.samp_num, t) / dot20(c.samp_den, t);
    *row = c.line_off + c.line_scale * rn;
    *col = c.samp_off + c.samp_scale * cn;
    return true;
}

// 2x2 full-pivoting LU solve with the operation order of Eigen's FullPivLU
// (computeInPlace / _solve_impl); the reference calls jac.fullPivLu().solve(-f)
// at camera.cpp:84.  Eigen is not on disk here, so this order is the pinned
// contract.
void fullpiv_solve2(const double J[2][2], const double b[2], double x[2]) {
    double a[2][2] = {{J[0][0], J[0][1]}, {J[1][0], J[1][1]}};
    // k = 0: biggest |a| in column-major order, first maximum wins.
    int pr = 0, pc = 0;
    double big = std::abs(a[0][0]);
    const int order[3][2] = {{1, 0}, {0, 1}, {1, 1}};
    for (auto& rc : order) {
        double v = std::abs(a[rc[0]][rc[1]]);
        if (v > big) {
            big = v;
            pr = rc[0];
            pc = rc[1];
        }
    }
    int nonzero = 2;
    double maxpivot = 0;
    if (big == 0) {
        nonzero = 0;
        pr = 0;
        pc = 0;
    } else {
        maxpivot = big;
        if (pr != 0) std::swap(a[0], a[1]);
        if (pc != 0) {
            std::swap(a[0][0], a[0][1]);
            std::swap(a[1][0], a[1][1]);
        }
        a[1][0] = a[1][0] / a[0][0];
        a[1][1] = a[1][1] - a[1][0] * a[0][1];
        double big1 = std::abs(a[1][1]);
        if (big1 == 0) {
            nonzero = 1;
        } else if (big1 > maxpivot) {
            maxpivot = big1;
        }
    }
    // rank(): pivots above |maxpivot| * eps * diagonalSize.
    const double thr = std::abs(maxpivot) * (2.220446049250313e-16 * 2.0);
    int rank = 0;
    for (int i = 0; i < nonzero; ++i) rank += (std::abs(a[i][i]) > thr);
    if (rank == 0) {
        x[0] = 0;
        x[1] = 0;
        return;
    }
    double c[2] = {b[0], b[1]};
    if (pr != 0) std::swap(c[0], c[1]);
    c[1] = c[1] - c[0] * a[1][0]; // unit-lower forward solve
    if (rank == 2) {
        c[1] = c[1] / a[1][1];
        c[0] = c[0] - c[1] * a[0][1];
        c[0] = c[0] / a[0][0];
    } else {
        c[0] = c[0] / a[0][0];
    }
    double out[2];
    int q0 = pc, q1 = pc == 0 ? 1 : 0; // permutationQ indices
    out[q0] = c[0];
    out[q1] = rank == 2 ? c[1] : 0.0;
    x[0] = out[0];
    x[1] = out[1];
}

inline double norm2(double a, double b) { return std::sqrt(a * a + b * b); }

// camera.cpp:66-103.  Status: 0 ok, 1 project threw, 2 no convergence.
int localize(const tfg_rpc& c, double pr, double pcol, double h, double* gx, double* gy,
             double* resid, int* iters) {
    double x = c.long_off, y = c.lat_off;
    const double hx = 1e-6 * c.long_scale;
    const double hy = 1e-6 * c.lat_scale;
    const double tol = 1e-4;
    bool ok = true;
    auto res = [&](double ax, double ay, double* f0, double* f1) {
        double r, cc;
        if (!project(c, ax, ay, h, &r, &cc)) {
            ok = false;
            return;
        }
        *f0 = r - pr;
        *f1 = cc - pcol;
    };
    double f0 = 0, f1 = 0;
    res(x, y, &f0, &f1);
    if (!ok) return 1;
    for (int it = 1; it <= 50; ++it) {
        if (norm2(f0, f1) < tol) {
            *gx = x;
            *gy = y;
            *resid = norm2(f0, f1);
            *iters = it - 1;
            return 0;
        }
        double a0, a1, b0, b1, c0, c1, d0, d1;
        res(x + hx, y + 0.0, &a0, &a1);
        if (!ok) return 1;
        res(x - hx, y - 0.0, &b0, &b1);
        if (!ok) return 1;
        res(x + 0.0, y + hy, &c0, &c1);
        if (!ok) return 1;
        res(x - 0.0, y - hy, &d0, &d1);
        if (!ok) return 1;
        double J[2][2];
        J[0][0] = (a0 - b0) / (2 * hx);
        J[1][0] = (a1 - b1) / (2 * hx);
        J[0][1] = (c0 - d0) / (2 * hy);
        J[1][1] = (c1 - d1) / (2 * hy);
        double rhs[2] = {-f0, -f1}, st[2];
        fullpiv_solve2(J, rhs, st);
        double lam = 1.0;
        double nx = x + st[0], ny = y + st[1];
        double n0, n1;
        res(nx, ny, &n0, &n1);
        if (!ok) return 1;
        for (int k = 0; k < 6 && norm2(n0, n1) > norm2(f0, f1); ++k) {
            lam *= 0.5;
            nx = x + lam * st[0];
            ny = y + lam * st[1];
            res(nx, ny, &n0, &n1);
            if (!ok) return 1;
        }
        x = nx;
        y = ny;
        f0 = n0;
        f1 = n1;
    }
    *resid = norm2(f0, f1);
    *iters = 50;
    if (norm2(f0, f1) < tol) {
        *gx = x;
        *gy = y;
        return 0;
    }
    return 2;
}

// camera.cpp:105-124.  Vec3::norm summation order pinned as (x²+y²)+z².
int ray_from_pixel(const tfg_rpc& c, int row, int col, double zmin, double zmax, double* o,
                   double* d) {
    double tx, ty, bx, by, r;
    int it;
    if (localize(c, double(row), double(col), zmax, &tx, &ty, &r, &it)) return 1;
    if (localize(c, double(row), double(col), zmin, &bx, &by, &r, &it)) return 1;
    double dx = bx - tx, dy = by - ty, dz = zmin - zmax;
    double len = std::sqrt(dx * dx + dy * dy + dz * dz);
    if (!(len > 1e-12 && zmax > zmin)) return 1;
    o[0] = tx;
    o[1] = ty;
    o[2] = zmax;
    d[0] = dx / len;
    d[1] = dy / len;
    d[2] = dz / len;
    return 0;
}

// camera.cpp:126-146 (8 projected corners; corner order geometry.hpp:25-29).
int crop_for_tile(const tfg_rpc& c, const double* box, int margin, int* rect) {
    double rlo = INFINITY, rhi = -INFINITY, clo = INFINITY, chi = -INFINITY;
    for (int i = 0; i < 8; ++i) {
        double x = (i & 1) ? box[3] : box[0];
        double y = (i & 2) ? box[4] : box[1];
        double z = (i & 4) ? box[5] : box[2];
        double r, cc;
        if (!project(c, x, y, z, &r, &cc)) return 2;
        rlo = std::min(rlo, r);
        rhi = std::max(rhi, r);
        clo = std::min(clo, cc);
        chi = std::max(chi, cc);
    }
    rect[0] = std::max(0, int(std::floor(rlo)) - margin);
    rect[1] = std::min(c.image_rows, int(std::ceil(rhi)) + 1 + margin);
    rect[2] = std::max(0, int(std::floor(clo)) - margin);
    rect[3] = std::min(c.image_cols, int(std::ceil(chi)) + 1 + margin);
    if (rect[0] >= rect[1] || rect[2] >= rect[3]) return 1;
    return 0;
}

// ----------------------------------------------------------- geometry.cpp:9-48
bool intersect(const double* o, const double* d, const double* box, double* t0o, double* t1o) {
    double t0 = 0.0, t1 = INFINITY;
    for (int k = 0; k < 3; ++k) {
        if (d[k] == 0.0) {
            if (o[k] < box[k] || o[k] > box[3 + k]) return false;
            continue;
        }
        double inv = 1.0 / d[k];
        double ta = (box[k] - o[k]) * inv;
        double tb = (box[3 + k] - o[k]) * inv;
        if (ta > tb) std::swap(ta, tb);
        t0 = std::max(t0, ta);
        t1 = std::min(t1, tb);
        if (t0 > t1) return false;
    }
    if (t1 - t0 < 1e-6) return false;
    *t0o = t0;
    *t1o = t1;
    return true;
}
// TileBoxSet::segments: hits in box order, stable ascending sort by t_near
// (libstdc++ std::sort on <= 16 elements is insertion sort, stable).
int segments(const double* o, const double* d, const double* boxes, int n, int* slot, double* tn,
             double* tf) {
    int m = 0;
    for (int i = 0; i < n; ++i) {
        double a, b;
        if (intersect(o, d, boxes + 6 * i, &a, &b)) {
            int j = m++;
            while (j > 0 && a < tn[j - 1]) {
                tn[j] = tn[j - 1];
                tf[j] = tf[j - 1];
                slot[j] = slot[j - 1];
                --j;
            }
            tn[j] = a;
            tf[j] = b;
            slot[j] = i;
        }
    }
    return m;
}

// -------------------------------------------------------------- tiler.cpp:18-100
void grid_edges(double lo, double hi, int n, double* e) {
    double step = (hi - lo) / n;
    for (int k = 0; k <= n; ++k) e[k] = lo + k * step;
    e[0] = lo;
    e[n] = hi;
}
int cell_of(const double* edges, int n, double v) {
    int k = int(std::upper_bound(edges, edges + n + 1, v) - edges) - 1;
    return std::clamp(k, 0, n - 1);
}
// Returns false when the reference returns {} (dz == 0 or behind).
bool candidate_range(const tfg_roi& roi, const double* east, int cols, const double* north,
                     int rows, const double* o, const double* d, int* r0, int* r1, int* c0,
                     int* c1) {
    double z0 = roi.z_max, z1 = roi.z_min;
    double dz = d[2];
    if (dz == 0.0) return false;
    double ta = (z0 - o[2]) / dz;
    double tb = (z1 - o[2]) / dz;
    if (ta > tb) std::swap(ta, tb);
    ta = std::max(ta, 0.0);
    if (tb < ta) return false;
    double ax = o[0] + ta * d[0], ay = o[1] + ta * d[1];
    double bx = o[0] + tb * d[0], by = o[1] + tb * d[1];
    *c0 = cell_of(east, cols, std::min(ax, bx));
    *c1 = cell_of(east, cols, std::max(ax, bx));
    *r0 = cell_of(north, rows, std::min(ay, by));
    *r1 = cell_of(north, rows, std::max(ay, by));
    return true;
}

// ------------------------------------------------------------------ nn.hpp
int level_res(const tfg_field_config& c, int l) {
    if (c.levels <= 1) return c.n_min;
    double b = std::exp((std::log(double(c.n_max)) - std::log(double(c.n_min))) /
                        double(c.levels - 1));
    return int(std::floor(c.n_min * std::pow(b, l) + 0.5));
}

struct Shapes {
    tfg_field_config cfg;
    int L = 8, T = 1 << 15, F = 2;
    int res[16];
    size_t off[16], size[16];
    size_t enc_params = 0;
    std::vector<int> dw, cw; // MLP widths
    size_t dnet_params = 0, color_params = 0;
    int occ_res = 32;

    explicit Shapes(const tfg_field_config& c) : cfg(c) {
        L = c.levels;
        T = c.table_size;
        F = c.features;
        size_t tot = 0;
        for (int l = 0; l < L; ++l) {
            res[l] = level_res(c, l);
            size_t dense = size_t(res[l] + 1) * (res[l] + 1) * (res[l] + 1);
            off[l] = tot;
            size[l] = std::min(dense, size_t(T));
            tot += size[l];
        }
        enc_params = tot * F;
        dw = {L * F, c.density_hidden, 1 + c.embedding};
        cw.push_back(c.embedding + 6 * c.view_freqs);
        for (int i = 0; i < c.color_layers; ++i) cw.push_back(c.color_hidden);
        cw.push_back(3);
        dnet_params = mlp_params(dw);
        color_params = mlp_params(cw);
        occ_res = c.occupancy_resolution;
    }
    static size_t mlp_params(const std::vector<int>& w) {
        size_t n = 0;
        for (size_t l = 0; l + 1 < w.size(); ++l) n += size_t(w[l + 1]) * w[l] + w[l + 1];
        return n;
    }
    static size_t mlp_acts(const std::vector<int>& w) {
        size_t n = 0;
        for (int x : w) n += x;
        return n;
    }
};

// MlpT::init (nn.hpp:70-81): Xavier-uniform weights, zero biases.
void mlp_init(const std::vector<int>& w, Rng& rng, float* p) {
    size_t k = 0;
    for (size_t l = 0; l + 1 < w.size(); ++l) {
        int fi = w[l], fo = w[l + 1];
        float bound = float(std::sqrt(6.0 / (fi + fo)));
        for (int i = 0; i < fo * fi; ++i) p[k++] = float(rng.uniform(-double(bound), double(bound)));
        for (int i = 0; i < fo; ++i) p[k++] = 0.f;
    }
}
// MlpT::forward_p (nn.hpp:90-108).  acts = [in | layer outputs...].
template <typename S>
void mlp_fwd(const std::vector<int>& w, const S* p, const S* x, S* acts) {
    for (int i = 0; i < w[0]; ++i) acts[i] = x[i];
    S* a = acts;
    size_t po = 0;
    for (size_t l = 0; l + 1 < w.size(); ++l) {
        const S* in = a;
        S* out = a + w[l];
        const S* W = p + po;
        const S* b = W + size_t(w[l + 1]) * w[l];
        bool last = (l + 2 == w.size());
        for (int o = 0; o < w[l + 1]; ++o) {
            S acc = b[o];
            const S* row = W + size_t(o) * w[l];
            for (int i = 0; i < w[l]; ++i) acc += row[i] * in[i];
            out[o] = (!last && acc < S(0)) ? S(0) : acc;
        }
        po += size_t(w[l + 1]) * w[l] + w[l + 1];
        a = out;
    }
}
// MlpT::backward_p (nn.hpp:116-157).
template <typename S>
void mlp_bwd(const std::vector<int>& w, const S* p, const S* acts, const S* d_out, S* grad,
             S* d_in) {
    int nl = int(w.size()) - 1;
    S bufa[128], bufb[128];
    S* cur = bufa;
    S* prev = bufb;
    for (int i = 0; i < w[nl]; ++i) cur[i] = d_out[i];
    size_t aoff[8], poff[8];
    size_t ao = 0, po = 0;
    for (int l = 0; l <= nl; ++l) {
        aoff[l] = ao;
        ao += w[l];
    }
    for (int l = 0; l < nl; ++l) {
        poff[l] = po;
        po += size_t(w[l + 1]) * w[l] + w[l + 1];
    }
    for (int l = nl - 1; l >= 0; --l) {
        const S* in = acts + aoff[l];
        const S* out = acts + aoff[l + 1];
        const S* W = p + poff[l];
        S* gW = grad + poff[l];
        S* gb = gW + size_t(w[l + 1]) * w[l];
        bool last = (l == nl - 1);
        for (int i = 0; i < w[l]; ++i) prev[i] = S(0);
        for (int o = 0; o < w[l + 1]; ++o) {
            S d = cur[o];
            if (!last && out[o] <= S(0)) d = S(0);
            gb[o] += d;
            const S* wr = W + size_t(o) * w[l];
            S* gr = gW + size_t(o) * w[l];
            for (int i = 0; i < w[l]; ++i) {
                gr[i] += d * in[i];
                prev[i] += d * wr[i];
            }
        }
        std::swap(cur, prev);
    }
    if (d_in)
        for (int i = 0; i < w[0]; ++i) d_in[i] = cur[i];
}

// HashGridT (nn.hpp:199-266).
inline size_t hash_entry(const Shapes& sh, int l, int x, int y, int z) {
    int n = sh.res[l] + 1;
    size_t dense = size_t(n) * n * n;
    if (dense <= size_t(sh.T)) return size_t(x) + size_t(n) * (size_t(y) + size_t(n) * z);
    uint32_t h = uint32_t(x) ^ (uint32_t(y) * 2654435761u) ^ (uint32_t(z) * 805459861u);
    return h & uint32_t(sh.T - 1);
}
template <typename S>
inline void hash_cell(const Shapes& sh, int l, const S* p, int* c, S* f) {
    int n = sh.res[l];
    for (int k = 0; k < 3; ++k) {
        S v = p[k];
        if (v < S(0)) v = S(0);
        if (v > S(1)) v = S(1);
        S sc = v * S(n);
        int ci = int(sc);
        if (ci > n - 1) ci = n - 1;
        c[k] = ci;
        f[k] = sc - S(ci);
    }
}
template <typename S>
void hash_lookup(const Shapes& sh, const S* tab, const S* p, S* out) {
    for (int l = 0; l < sh.L; ++l) {
        int c[3];
        S f[3];
        hash_cell(sh, l, p, c, f);
        S* o = out + size_t(l) * sh.F;
        for (int q = 0; q < sh.F; ++q) o[q] = S(0);
        for (int k = 0; k < 8; ++k) {
            int dx = k & 1, dy = (k >> 1) & 1, dz = (k >> 2) & 1;
            S w = (dx ? f[0] : S(1) - f[0]) * (dy ? f[1] : S(1) - f[1]) *
                  (dz ? f[2] : S(1) - f[2]);
            size_t idx = hash_entry(sh, l, c[0] + dx, c[1] + dy, c[2] + dz);
            const S* e = tab + (sh.off[l] + idx) * sh.F;
            for (int q = 0; q < sh.F; ++q) o[q] += w * e[q];
        }
    }
}
template <typename S>
void hash_backward(const Shapes& sh, const S* p, const S* d, S* g) {
    for (int l = 0; l < sh.L; ++l) {
        int c[3];
        S f[3];
        hash_cell(sh, l, p, c, f);
        const S* dl = d + size_t(l) * sh.F;
        for (int k = 0; k < 8; ++k) {
            int dx = k & 1, dy = (k >> 1) & 1, dz = (k >> 2) & 1;
            S w = (dx ? f[0] : S(1) - f[0]) * (dy ? f[1] : S(1) - f[1]) *
                  (dz ? f[2] : S(1) - f[2]);
            size_t idx = hash_entry(sh, l, c[0] + dx, c[1] + dy, c[2] + dz);
            S* e = g + (sh.off[l] + idx) * sh.F;
            for (int q = 0; q < sh.F; ++q) e[q] += w * dl[q];
        }
    }
}
// nn.hpp:270-298
template <typename S>
S density_act(S raw, S maxd, S* draw) {
    S lim = std::log(maxd);
    if (raw >= lim) {
        if (draw) *draw = S(0);
        return maxd;
    }
    S v = std::exp(raw);
    if (draw) *draw = v;
    return v;
}
template <typename S>
S sigm(S x) {
    return S(1) / (S(1) + std::exp(-x));
}
template <typename S>
void encode_dir(const S* d, int freqs, S* out) {
    int j = 0;
    for (int k = 0; k < freqs; ++k) {
        S sc = S(std::pow(2.0, k) * M_PI);
        for (int c = 0; c < 3; ++c) {
            out[j++] = std::sin(sc * d[c]);
            out[j++] = std::cos(sc * d[c]);
        }
    }
}

// Full per-point field query (TileField::query_density + GlobalColorNet::query_color).
struct SampleActs {
    float feat[16];
    float dacts[16 + 64 + 16];
    float cacts[39 + 64 + 64 + 3];
    float draw; // d sigma / d raw
    float sigma;
    float rgb[3];
};
void field_point(const Shapes& sh, const float* enc, const float* dnet, const float* color,
                 const float* local, const float* venc, SampleActs& a) {
    hash_lookup<float>(sh, enc, local, a.feat);
    mlp_fwd<float>(sh.dw, dnet, a.feat, a.dacts);
    const float* dout = a.dacts + sh.dw[0] + sh.dw[1];
    a.sigma = density_act<float>(dout[0], sh.cfg.density_max, &a.draw);
    float cin[64];
    for (int i = 0; i < sh.cfg.embedding; ++i) cin[i] = dout[1 + i];
    for (int i = 0; i < 6 * sh.cfg.view_freqs; ++i) cin[sh.cfg.embedding + i] = venc[i];
    mlp_fwd<float>(sh.cw, color, cin, a.cacts);
    const float* o = a.cacts + Shapes::mlp_acts(sh.cw) - 3;
    for (int c = 0; c < 3; ++c) a.rgb[c] = sigm<float>(o[c]);
}
float sigma_point(const Shapes& sh, const float* enc, const float* dnet, const float* local) {
    float feat[16], dacts[96];
    hash_lookup<float>(sh, enc, local, feat);
    mlp_fwd<float>(sh.dw, dnet, feat, dacts);
    return density_act<float>(dacts[sh.dw[0] + sh.dw[1]], sh.cfg.density_max, nullptr);
}

// OccupancyGrid::voxel_index / occupied (field.hpp:68-77).
inline size_t voxel_index(int res, float x, float y, float z) {
    auto ci = [res](float v) {
        int i = int(v * float(res));
        return size_t(i < 0 ? 0 : (i >= res ? res - 1 : i));
    };
    return ci(x) + size_t(res) * (ci(y) + size_t(res) * ci(z));
}

// ----------------------------------------------------- sample_segments (SPEC 352-360, 386-390)
// Pins: n_int = ceil(len*spm) >= 1 intervals per segment, samples
// at j = 0..n_int with exact endpoints; interior t = tn + (j + (u - 0.5))*step,
// u = 0.5 when jitter is off, else Rng(hash_combine(ray_key, (k<<16)|j)).flt();
// p = o + t*d (double), local = float((p - min)*inv_size); interior samples in
// clear occupancy voxels are culled; delta over the concatenated kept samples
// in double, last delta = min(max(t_exit(z_min) - t_last, 0), delta_cap).
int sample_ray(const double* o, const double* d, int nseg, const int* sslot, const double* stn,
               const double* stf, const double* frames, const float* const* occ, int occ_res,
               float occ_thr, double spm, int cap, double zmin, double dcap, int jitter,
               uint64_t key, std::vector<double>& tt, std::vector<float>& lc,
               std::vector<uint8_t>& sl, std::vector<uint8_t>& ep) {
    int nint[16];
    long total = 0, sumint = 0;
    for (int k = 0; k < nseg; ++k) {
        double len = stf[k] - stn[k];
        long n = (long)std::ceil(len * spm);
        if (n < 1) n = 1;
        nint[k] = int(n);
        sumint += n;
        total += n + 1;
    }
    if (total > cap) {
        long budget = cap - nseg;
        for (int k = 0; k < nseg; ++k) {
            long n = (long)nint[k] * budget / sumint;
            nint[k] = int(n < 1 ? 1 : n);
        }
    }
    int count = 0;
    for (int k = 0; k < nseg; ++k) {
        const double* fr = frames + 6 * sslot[k];
        const float* og = occ ? occ[sslot[k]] : nullptr;
        int n = nint[k];
        double step = (stf[k] - stn[k]) / n;
        for (int j = 0; j <= n; ++j) {
            double t;
            bool endp = (j == 0 || j == n);
            if (j == 0) {
                t = stn[k];
            } else if (j == n) {
                t = stf[k];
            } else {
                float u = 0.5f;
                if (jitter) u = Rng(hc(key, (uint64_t(k) << 16) | uint64_t(j))).flt();
                t = stn[k] + (double(j) + (double(u) - 0.5)) * step;
            }
            float l3[3];
            for (int c = 0; c < 3; ++c) {
                double p = o[c] + t * d[c];
                l3[c] = float((p - fr[c]) * fr[3 + c]);
            }
            if (!endp && og) {
                if (!(og[voxel_index(occ_res, l3[0], l3[1], l3[2])] >= occ_thr)) continue;
            }
            tt.push_back(t);
            lc.insert(lc.end(), l3, l3 + 3);
            sl.push_back(uint8_t(sslot[k]));
            ep.push_back(endp ? 1 : 0);
            ++count;
        }
    }
    (void)zmin;
    (void)dcap;
    return count;
}
void deltas(const double* t, int n, const double* o, const double* d, double zmin, double dcap,
            float* delta) {
    for (int i = 0; i + 1 < n; ++i) delta[i] = float(t[i + 1] - t[i]);
    if (n > 0) {
        double texit = (zmin - o[2]) / d[2];
        double r = texit - t[n - 1];
        if (r < 0) r = 0;
        if (r > dcap) r = dcap;
        delta[n - 1] = float(r);
    }
}

// ----------------------------------------------------- render (SPEC 361-369, 381-384)
void render_ray(int n, const float* sg, const float* rgb, const float* t, const float* dl,
                const float* bg, float* orgb, float* odepth, float* oop, const float* g,
                float* dsig, float* drgb) {
    float T = 1.f, acc[3] = {0, 0, 0}, dep = 0, op = 0;
    std::vector<float> w(n), Tn(n);
    for (int k = 0; k < n; ++k) {
        float a = 1.f - std::exp(-(sg[k] * dl[k]));
        float wk = T * a;
        w[k] = wk;
        for (int c = 0; c < 3; ++c) acc[c] += wk * rgb[3 * k + c];
        dep += wk * t[k];
        op += wk;
        T = T * (1.f - a);
        Tn[k] = T; // T_{k+1}
    }
    float out[3];
    for (int c = 0; c < 3; ++c) out[c] = acc[c] + T * bg[c];
    if (orgb)
        for (int c = 0; c < 3; ++c) orgb[c] = out[c];
    if (odepth) *odepth = dep / std::max(op, 1e-10f);
    if (oop) *oop = op;
    if (!g) return;
    // R_k = sum_{j>k} w_j c_j + T_N bg, accumulated back to front.
    float R[3] = {T * bg[0], T * bg[1], T * bg[2]};
    for (int k = n - 1; k >= 0; --k) {
        float s = 0;
        for (int c = 0; c < 3; ++c) s += g[c] * (Tn[k] * rgb[3 * k + c] - R[c]);
        if (dsig) dsig[k] = dl[k] * s;
        if (drgb)
            for (int c = 0; c < 3; ++c) drgb[3 * k + c] = w[k] * g[c];
        for (int c = 0; c < 3; ++c) R[c] += w[k] * rgb[3 * k + c];
    }
}

// color_loss (SPEC 371-378) of one ray: returns the ray's squared error
// summed over channels (the batch loss is the sum / (3 B)) and writes the
// gradient at the rendered rgb, 2 (rgb - target) / (3 B) (channel-mean
// convention of the example at SPEC 377).
double color_loss_ray(const float* rgb, const float* target, float inv3b, float* g) {
    double l = 0;
    for (int c = 0; c < 3; ++c) {
        float df = rgb[c] - target[c];
        l += double(df) * double(df);
        g[c] = 2.0f * df * inv3b;
    }
    return l;
}

// ----------------------------------------------------- adam_step (SPEC 292-300)
double lr_at(double base, double rate, uint64_t steps, uint64_t step) {
    if (rate == 1.0) return base;
    return base * std::pow(rate, double(step) / double(steps));
}
int adam(float* p, const float* g, float* m, float* v, size_t n, uint64_t* step, double base,
         double rate, uint64_t dsteps, float b1, float b2, float eps, const std::string& group) {
    for (size_t i = 0; i < n; ++i)
        if (!std::isfinite(g[i])) {
            g_err = "adam_step: non-finite gradient in group " + group;
            return 1;
        }
    uint64_t s = *step + 1;
    float lr = float(lr_at(base, rate, dsteps, s));
    float bc1 = float(1.0 - std::pow(double(b1), double(s)));
    float bc2 = float(1.0 - std::pow(double(b2), double(s)));
    float omb1 = 1.0f - b1, omb2 = 1.0f - b2;
    for (size_t i = 0; i < n; ++i) {
        float gi = g[i];
        float mi = b1 * m[i] + omb1 * gi;
        float vi = b2 * v[i] + omb2 * (gi * gi);
        m[i] = mi;
        v[i] = vi;
        float mh = mi / bc1;
        float vh = vi / bc2;
        p[i] = p[i] - lr * mh / (std::sqrt(vh) + eps);
    }
    *step = s;
    return 0;
}

// ----------------------------------------------------- session
struct TileRec {
    bool created = false;
    std::vector<float> enc, dnet, enc_m, enc_v, dnet_m, dnet_v, occ;
    uint64_t enc_step = 0, dnet_step = 0;
};

} // namespace

struct tfo_session {
    Shapes sh;
    tfg_train_config tc;
    std::vector<tfg_rpc> cams;
    std::vector<std::vector<uint8_t>> images;
    tfg_roi roi;
    int rows, cols, workers;
    std::vector<double> east, north;
    std::vector<TileRec> tiles;
    int pos_r = -1, pos_c = -1;
    int slot_tile[4] = {-1, -1, -1, -1};
    int nslots = 0;
    std::vector<float> color, color_m, color_v;
    uint64_t color_step = 0;
    std::vector<uint64_t> accept;
    // batch (ray order)
    std::vector<tfg_ray_entry> rays;
    std::vector<uint32_t> offsets;
    std::vector<double> tdbl;
    std::vector<float> t, delta, local;
    std::vector<uint8_t> slot, endpoint;
    std::vector<float> venc; // 24 per ray
    std::vector<float> sigma, rgb;
    std::vector<float> dsig, drgb;
    std::vector<std::vector<float>> g_enc, g_dnet;
    std::vector<float> g_color;

    explicit tfo_session(const tfg_field_config& f) : sh(f) {}

    void box_of(int ti, double* b) const {
        int r = ti / cols, c = ti % cols;
        b[0] = east[c];
        b[1] = north[r];
        b[2] = roi.z_min;
        b[3] = east[c + 1];
        b[4] = north[r + 1];
        b[5] = roi.z_max;
    }
    void frame_of(int ti, double* fr) const {
        double b[6];
        box_of(ti, b);
        for (int k = 0; k < 3; ++k) {
            fr[k] = b[k];
            fr[3 + k] = 1.0 / (b[3 + k] - b[k]); // cwiseInverse (tiler.cpp:49)
        }
    }
    void ensure_tile(int ti) {
        TileRec& t = tiles[ti];
        if (t.created) return;
        t.enc.resize(sh.enc_params);
        t.dnet.resize(sh.dnet_params);
        t.occ.resize(size_t(sh.occ_res) * sh.occ_res * sh.occ_res);
        tfo_tile_create(&sh.cfg, ti / cols, ti % cols, tc.seed, t.enc.data(), t.dnet.data(),
                        t.occ.data());
        t.enc_m.assign(sh.enc_params, 0.f);
        t.enc_v.assign(sh.enc_params, 0.f);
        t.dnet_m.assign(sh.dnet_params, 0.f);
        t.dnet_v.assign(sh.dnet_params, 0.f);
        t.created = true;
    }
};

namespace {
bool finite_all(const std::vector<float>& v) {
    for (float x : v)
        if (!std::isfinite(x)) return false;
    return true;
}
} // namespace

extern "C" {

const char* tfo_last_error(void) { return g_err.c_str(); }
uint64_t tfo_splitmix64(uint64_t x) { return splitmix64(x); }
uint64_t tfo_hash_combine(uint64_t a, uint64_t b) { return hc(a, b); }

int tfo_project(const tfg_rpc* cam, const double* xyz, double* rc) {
    return project(*cam, xyz[0], xyz[1], xyz[2], &rc[0], &rc[1]) ? 0 : 1;
}
int tfo_localize(const tfg_rpc* cam, const double* px, double h, double* xy, double* resid,
                 int* iters) {
    return localize(*cam, px[0], px[1], h, &xy[0], &xy[1], resid, iters);
}
int tfo_ray_from_pixel(const tfg_rpc* cam, int row, int col, double zmin, double zmax, double* o,
                       double* d) {
    return ray_from_pixel(*cam, row, col, zmin, zmax, o, d);
}
int tfo_intersect(const double* o, const double* d, const double* box, double* t0, double* t1) {
    return intersect(o, d, box, t0, t1) ? 0 : 1;
}
int tfo_segments(const double* o, const double* d, const double* boxes, int n, int* slot,
                 double* tn, double* tf) {
    return segments(o, d, boxes, n, slot, tn, tf);
}
int tfo_crop_for_tile(const tfg_rpc* cam, const double* box, int margin, int* rect) {
    return crop_for_tile(*cam, box, margin, rect);
}
int tfo_grid_edges(const tfg_roi* roi, int rows, int cols, double* east, double* north) {
    grid_edges(roi->easting_min, roi->easting_max, cols, east);
    grid_edges(roi->northing_min, roi->northing_max, rows, north);
    return 0;
}
int tfo_candidate_tiles(const tfg_roi* roi, int rows, int cols, const double* o, const double* d,
                        int* pairs, int capacity) {
    std::vector<double> e(cols + 1), n(rows + 1);
    tfo_grid_edges(roi, rows, cols, e.data(), n.data());
    int r0, r1, c0, c1;
    if (!candidate_range(*roi, e.data(), cols, n.data(), rows, o, d, &r0, &r1, &c0, &c1)) return 0;
    int m = 0;
    for (int r = r0; r <= r1; ++r)
        for (int c = c0; c <= c1; ++c) {
            if (m < capacity) {
                pairs[2 * m] = r;
                pairs[2 * m + 1] = c;
            }
            ++m;
        }
    return m;
}
// SPEC 419-427: positions rows south->north, serpentine east<->west.
int tfo_snake_path(int rows, int cols, int* pairs, int capacity) {
    if (rows < 2 || cols < 2) return -1;
    int m = 0;
    for (int i = 0; i < rows - 1; ++i)
        for (int jj = 0; jj < cols - 1; ++jj) {
            int j = (i % 2 == 0) ? jj : (cols - 2 - jj);
            if (m < capacity) {
                pairs[2 * m] = i;
                pairs[2 * m + 1] = j;
            }
            ++m;
        }
    return m;
}
int tfo_level_resolution(const tfg_field_config* cfg, int level) { return level_res(*cfg, level); }

int tfo_sample_ray(const double* o, const double* d, int n_seg, const int* seg_slot,
                   const double* stn, const double* stf, const double* frames,
                   const float* const* occupancy, int occ_res, float occ_thr, double spm,
                   int max_samples, double z_min, double dcap, int jitter, uint64_t key,
                   float* t, float* delta, float* local, uint8_t* slot, uint8_t* endpoint,
                   int capacity) {
    std::vector<double> tt;
    std::vector<float> lc;
    std::vector<uint8_t> sl, ep;
    int n = sample_ray(o, d, n_seg, seg_slot, stn, stf, frames, occupancy, occ_res, occ_thr, spm,
                       max_samples, z_min, dcap, jitter, key, tt, lc, sl, ep);
    if (n > capacity) return -1;
    std::vector<float> dl(n);
    deltas(tt.data(), n, o, d, z_min, dcap, dl.data());
    for (int i = 0; i < n; ++i) {
        t[i] = float(tt[i]);
        delta[i] = dl[i];
        for (int c = 0; c < 3; ++c) local[3 * i + c] = lc[3 * i + c];
        slot[i] = sl[i];
        endpoint[i] = ep[i];
    }
    return n;
}

// cmd_render (the render path of tfg_render_pixels): for each
// (row, col) pixel of `cam`, ray_from_pixel, segments over the n_tiles boxes
// (slot order = tile order), midpoint samples (jitter off) with occupancy
// culling, the field of each sample's tile, render.  Failed rays give zeros.
int tfo_render_pixels(const tfg_field_config* cfg, const tfg_rpc* cam, double z_min, double z_max,
                      int n_tiles, const double* boxes6, const float* const* enc, const float* const* dnet,
                      const float* const* occupancy, const float* color, double spm, int cap,
                      double dcap, const float* bg, int n_px, const int32_t* px, float* rgb,
                      float* depth, float* opacity, int workers) {
    Shapes sh(*cfg);
    std::vector<double> frames(6 * size_t(n_tiles));
    for (int k = 0; k < n_tiles; ++k)
        for (int q = 0; q < 3; ++q) {
            frames[6 * k + q] = boxes6[6 * k + q];
            frames[6 * k + 3 + q] = 1.0 / (boxes6[6 * k + 3 + q] - boxes6[6 * k + q]);
        }
    par_for(size_t(n_px), workers < 1 ? 1 : workers, [&](size_t b, size_t e, int) {
        SampleActs a;
        std::vector<double> tt;
        std::vector<float> lc;
        std::vector<uint8_t> sl, ep;
        for (size_t i = b; i < e; ++i) {
            for (int c = 0; c < 3; ++c) rgb[3 * i + c] = 0.f;
            depth[i] = opacity[i] = 0.f;
            double o[3], d[3];
            if (ray_from_pixel(*cam, px[2 * i], px[2 * i + 1], z_min, z_max, o, d)) continue;
            int ss[16];
            double tn[16], tf[16];
            int ns = segments(o, d, boxes6, n_tiles, ss, tn, tf);
            tt.clear();
            lc.clear();
            sl.clear();
            ep.clear();
            int n = sample_ray(o, d, ns, ss, tn, tf, frames.data(), occupancy, sh.occ_res,
                               cfg->occupancy_threshold, spm, cap, z_min, dcap, 0, 0, tt, lc, sl, ep);
            std::vector<float> dl(n), tf32(n), sg(n), col(3 * size_t(n));
            deltas(tt.data(), n, o, d, z_min, dcap, dl.data());
            float d3[3] = {float(d[0]), float(d[1]), float(d[2])}, venc[64];
            encode_dir<float>(d3, cfg->view_freqs, venc);
            for (int k = 0; k < n; ++k) {
                tf32[k] = float(tt[k]);
                field_point(sh, enc[sl[k]], dnet[sl[k]], color, &lc[3 * size_t(k)], venc, a);
                sg[k] = a.sigma;
                for (int c = 0; c < 3; ++c) col[3 * k + c] = a.rgb[c];
            }
            render_ray(n, sg.data(), col.data(), tf32.data(), dl.data(), bg, rgb + 3 * i, depth + i,
                       opacity + i, nullptr, nullptr, nullptr);
        }
    });
    return 0;
}

void tfo_render_ray(int n, const float* sigma, const float* rgb, const float* t,
                    const float* delta, const float* bg, float* out_rgb, float* out_depth,
                    float* out_opacity, const float* g_rgb, float* d_sigma, float* d_rgb) {
    render_ray(n, sigma, rgb, t, delta, bg, out_rgb, out_depth, out_opacity, g_rgb, d_sigma,
               d_rgb);
}

int tfo_adam_step(float* params, const float* grads, float* m, float* v, uint64_t n,
                  uint64_t* step, double lr_base, double decay_rate, uint64_t decay_steps,
                  float beta1, float beta2, float eps, const char* group) {
    return adam(params, grads, m, v, n, step, lr_base, decay_rate, decay_steps, beta1, beta2, eps,
                group ? group : "?");
}

// TileField::create (field.hpp:93): per-tile streams from (seed, purpose, row, col).
int tfo_tile_create(const tfg_field_config* cfg, int row, int col, uint64_t seed, float* enc,
                    float* dnet, float* occupancy) {
    Shapes sh(*cfg);
    Rng re(hc(seed, kPurposeTileEnc, uint64_t(row), uint64_t(col)));
    for (size_t i = 0; i < sh.enc_params; ++i) enc[i] = float(re.uniform(-1e-4, 1e-4));
    Rng rd(hc(seed, kPurposeTileDnet, uint64_t(row), uint64_t(col)));
    mlp_init(sh.dw, rd, dnet);
    if (occupancy) {
        size_t nv = size_t(sh.occ_res) * sh.occ_res * sh.occ_res;
        for (size_t i = 0; i < nv; ++i) occupancy[i] = 1.0f;
    }
    return 0;
}
int tfo_color_create(const tfg_field_config* cfg, uint64_t seed, float* params) {
    Shapes sh(*cfg);
    Rng rc(hc(seed, kPurposeColor));
    mlp_init(sh.cw, rc, params);
    return 0;
}
int tfo_query_field(const tfg_field_config* cfg, const float* enc, const float* dnet,
                    const float* color, const float* local3, const float* dir3, float* sigma,
                    float* rgb) {
    Shapes sh(*cfg);
    float venc[64];
    encode_dir<float>(dir3, cfg->view_freqs, venc);
    SampleActs a;
    field_point(sh, enc, dnet, color, local3, venc, a);
    *sigma = a.sigma;
    if (rgb)
        for (int c = 0; c < 3; ++c) rgb[c] = a.rgb[c];
    return 0;
}

tfo_session* tfo_create(const tfg_field_config* fcfg, const tfg_train_config* tcfg,
                        const tfg_rpc* cams, int n_views, const uint8_t* const* images,
                        const tfg_roi* roi, int grid_rows, int grid_cols, int workers) {
    auto* s = new tfo_session(*fcfg);
    s->tc = *tcfg;
    s->cams.assign(cams, cams + n_views);
    s->images.resize(n_views);
    for (int v = 0; v < n_views; ++v) {
        size_t nb = size_t(cams[v].image_rows) * cams[v].image_cols * 3;
        s->images[v].assign(images[v], images[v] + nb);
    }
    s->roi = *roi;
    s->rows = grid_rows;
    s->cols = grid_cols;
    s->workers = workers < 1 ? 1 : workers;
    s->east.resize(grid_cols + 1);
    s->north.resize(grid_rows + 1);
    tfo_grid_edges(roi, grid_rows, grid_cols, s->east.data(), s->north.data());
    s->tiles.resize(size_t(grid_rows) * grid_cols);
    s->color.resize(s->sh.color_params);
    tfo_color_create(fcfg, tcfg->seed, s->color.data());
    s->color_m.assign(s->sh.color_params, 0.f);
    s->color_v.assign(s->sh.color_params, 0.f);
    return s;
}
void tfo_destroy(tfo_session* s) { delete s; }
int tfo_set_workers(tfo_session* s, int w) {
    s->workers = w < 1 ? 1 : w;
    return 0;
}

// SPEC 428-436 with the slot pin: the entering tile takes the slot of the
// leaving tile in the same row (east/west move) or column (north move).
int tfo_set_window(tfo_session* s, int pr, int pc) {
    if (s->rows == 1 && s->cols == 1) {
        s->nslots = 1;
        s->slot_tile[0] = 0;
        s->ensure_tile(0);
        s->pos_r = 0;
        s->pos_c = 0;
        return 0;
    }
    if (pr < 0 || pc < 0 || pr + 1 >= s->rows || pc + 1 >= s->cols) {
        g_err = "set_window: position outside the (H-1)x(W-1) lattice";
        return 1;
    }
    int want[4] = {pr * s->cols + pc, pr * s->cols + pc + 1, (pr + 1) * s->cols + pc,
                   (pr + 1) * s->cols + pc + 1};
    int next[4] = {-1, -1, -1, -1};
    if (s->nslots == 4) {
        // keep staying tiles in place
        bool used[4] = {false, false, false, false};
        for (int k = 0; k < 4; ++k)
            for (int sidx = 0; sidx < 4; ++sidx)
                if (s->slot_tile[sidx] == want[k]) {
                    next[sidx] = want[k];
                    used[k] = true;
                }
        for (int k = 0; k < 4; ++k) {
            if (used[k]) continue;
            int wr = want[k] / s->cols, wc = want[k] % s->cols;
            int best = -1;
            // leaving tile in the same row (horizontal move) or column (vertical move)
            for (int sidx = 0; sidx < 4; ++sidx) {
                if (next[sidx] != -1) continue;
                int lr = s->slot_tile[sidx] / s->cols, lc = s->slot_tile[sidx] % s->cols;
                bool horiz = (pr == s->pos_r);
                if ((horiz && lr == wr) || (!horiz && lc == wc)) {
                    best = sidx;
                    break;
                }
            }
            if (best < 0)
                for (int sidx = 0; sidx < 4; ++sidx)
                    if (next[sidx] == -1) {
                        best = sidx;
                        break;
                    }
            next[best] = want[k];
        }
    } else {
        for (int k = 0; k < 4; ++k) next[k] = want[k];
    }
    for (int k = 0; k < 4; ++k) {
        s->slot_tile[k] = next[k];
        s->ensure_tile(next[k]);
    }
    s->nslots = 4;
    s->pos_r = pr;
    s->pos_c = pc;
    s->accept.clear();
    return 0;
}
int tfo_window_tiles(tfo_session* s, int* r4, int* c4) {
    for (int k = 0; k < s->nslots; ++k) {
        r4[k] = s->slot_tile[k] / s->cols;
        c4[k] = s->slot_tile[k] % s->cols;
    }
    return s->nslots;
}

// accept_rays (SPEC 437-445) over the window's crop union, enumerated
// (view, row, col) ascending; rays whose localization throws are rejected.
int64_t tfo_build_accept(tfo_session* s) {
    s->accept.clear();
    std::vector<double> loaded(6 * s->nslots);
    for (int k = 0; k < s->nslots; ++k) s->box_of(s->slot_tile[k], &loaded[6 * k]);
    for (size_t v = 0; v < s->cams.size(); ++v) {
        const tfg_rpc& cam = s->cams[v];
        std::vector<std::array<int, 4>> rects;
        int u[4] = {INT32_MAX, INT32_MIN, INT32_MAX, INT32_MIN};
        for (int k = 0; k < s->nslots; ++k) {
            int r[4];
            if (crop_for_tile(cam, &loaded[6 * k], s->tc.margin_px, r) != 0) continue;
            rects.push_back({r[0], r[1], r[2], r[3]});
            u[0] = std::min(u[0], r[0]);
            u[1] = std::max(u[1], r[1]);
            u[2] = std::min(u[2], r[2]);
            u[3] = std::max(u[3], r[3]);
        }
        if (rects.empty()) continue;
        int nr = u[1] - u[0];
        std::vector<std::vector<uint64_t>> per_row(nr);
        par_for(size_t(nr), s->workers, [&](size_t b, size_t e, int) {
            for (size_t ri = b; ri < e; ++ri) {
                int row = u[0] + int(ri);
                for (int col = u[2]; col < u[3]; ++col) {
                    bool in = false;
                    for (auto& r : rects)
                        if (row >= r[0] && row < r[1] && col >= r[2] && col < r[3]) in = true;
                    if (!in) continue;
                    double o[3], d[3];
                    if (ray_from_pixel(cam, row, col, s->roi.z_min, s->roi.z_max, o, d)) continue;
                    int r0, r1, c0, c1;
                    if (!candidate_range(s->roi, s->east.data(), s->cols, s->north.data(),
                                         s->rows, o, d, &r0, &r1, &c0, &c1))
                        continue;
                    int hits = 0;
                    bool all_loaded = true;
                    for (int tr = r0; tr <= r1; ++tr)
                        for (int tcn = c0; tcn <= c1; ++tcn) {
                            int ti = tr * s->cols + tcn;
                            double b[6], a0, a1;
                            s->box_of(ti, b);
                            if (!intersect(o, d, b, &a0, &a1)) continue;
                            ++hits;
                            bool ld = false;
                            for (int k = 0; k < s->nslots; ++k)
                                if (s->slot_tile[k] == ti) ld = true;
                            if (!ld) all_loaded = false;
                        }
                    if (hits >= 1 && all_loaded)
                        per_row[ri].push_back((uint64_t(v) << 40) | (uint64_t(row) << 20) |
                                              uint64_t(col));
                }
            }
        });
        for (auto& r : per_row) s->accept.insert(s->accept.end(), r.begin(), r.end());
    }
    return int64_t(s->accept.size());
}
int64_t tfo_accept_export(tfo_session* s, uint64_t* out, uint64_t cap) {
    uint64_t n = std::min<uint64_t>(cap, s->accept.size());
    std::memcpy(out, s->accept.data(), n * 8);
    return int64_t(s->accept.size());
}

namespace {
int64_t build_batch(tfo_session* s, const std::vector<std::array<int, 3>>& px, uint64_t iter,
                    uint64_t ray_begin, int jitter) {
    int n = int(px.size());
    s->rays.assign(n, tfg_ray_entry{});
    s->venc.assign(size_t(n) * 6 * s->sh.cfg.view_freqs, 0.f);
    std::vector<double> boxes(6 * s->nslots), frames(6 * s->nslots);
    std::vector<const float*> occ(s->nslots);
    for (int k = 0; k < s->nslots; ++k) {
        s->box_of(s->slot_tile[k], &boxes[6 * k]);
        s->frame_of(s->slot_tile[k], &frames[6 * k]);
        occ[k] = s->tiles[s->slot_tile[k]].occ.data();
    }
    struct PerRay {
        std::vector<double> t;
        std::vector<float> lc;
        std::vector<uint8_t> sl, ep;
    };
    std::vector<PerRay> pr(n);
    std::vector<int> bad(n, 0);
    par_for(size_t(n), s->workers, [&](size_t b, size_t e, int) {
        for (size_t i = b; i < e; ++i) {
            int v = px[i][0], row = px[i][1], col = px[i][2];
            tfg_ray_entry& R = s->rays[i];
            R.image_id = v;
            R.row = row;
            R.col = col;
            const tfg_rpc& cam = s->cams[v];
            const uint8_t* pix = s->images[v].data() + 3 * (size_t(row) * cam.image_cols + col);
            for (int c = 0; c < 3; ++c) R.target[c] = float(pix[c]) / 255.0f; // u8_to_unit
            if (ray_from_pixel(cam, row, col, s->roi.z_min, s->roi.z_max, R.origin,
                               R.direction)) {
                bad[i] = 1;
                continue;
            }
            float d3[3] = {float(R.direction[0]), float(R.direction[1]), float(R.direction[2])};
            encode_dir<float>(d3, s->sh.cfg.view_freqs, &s->venc[i * 6 * s->sh.cfg.view_freqs]);
            int ss[16];
            double tn[16], tf[16];
            int m = segments(R.origin, R.direction, boxes.data(), s->nslots, ss, tn, tf);
            uint64_t key = hc(s->tc.seed, kPurposeJitter, iter, ray_begin + i);
            sample_ray(R.origin, R.direction, m, ss, tn, tf, frames.data(), occ.data(),
                       s->sh.occ_res, s->sh.cfg.occupancy_threshold, s->tc.samples_per_meter,
                       s->tc.max_samples_per_ray, s->roi.z_min, s->tc.delta_cap, jitter, key,
                       pr[i].t, pr[i].lc, pr[i].sl, pr[i].ep);
        }
    });
    for (int i = 0; i < n; ++i)
        if (bad[i]) {
            g_err = "sample: ray_from_pixel failed for a drawn pixel";
            return -1;
        }
    s->offsets.assign(n + 1, 0);
    for (int i = 0; i < n; ++i) s->offsets[i + 1] = s->offsets[i] + uint32_t(pr[i].t.size());
    size_t S = s->offsets[n];
    s->tdbl.resize(S);
    s->t.resize(S);
    s->delta.resize(S);
    s->local.resize(3 * S);
    s->slot.resize(S);
    s->endpoint.resize(S);
    for (int i = 0; i < n; ++i) {
        size_t o = s->offsets[i];
        int m = int(pr[i].t.size());
        for (int j = 0; j < m; ++j) {
            s->tdbl[o + j] = pr[i].t[j];
            s->t[o + j] = float(pr[i].t[j]);
            s->slot[o + j] = pr[i].sl[j];
            s->endpoint[o + j] = pr[i].ep[j];
            for (int c = 0; c < 3; ++c) s->local[3 * (o + j) + c] = pr[i].lc[3 * j + c];
        }
        deltas(&s->tdbl[o], m, s->rays[i].origin, s->rays[i].direction, s->roi.z_min,
               s->tc.delta_cap, &s->delta[o]);
    }
    s->sigma.clear();
    return int64_t(S);
}
} // namespace

// Trainer batch draw (SPEC 493): ray g of iteration `iter` takes accepted
// entry Rng(hash_combine(seed, PIXELS, iter, g)).next_below(|A|).
int64_t tfo_sample(tfo_session* s, uint64_t iter, uint64_t ray_begin, int n_rays, int jitter) {
    if (s->accept.empty()) {
        g_err = "sample: empty accepted-ray list (call build_accept)";
        return -1;
    }
    std::vector<std::array<int, 3>> px(n_rays);
    for (int i = 0; i < n_rays; ++i) {
        Rng r(hc(s->tc.seed, kPurposePixels, iter, ray_begin + uint64_t(i)));
        uint64_t e = s->accept[r.below(s->accept.size())];
        px[i] = {int(e >> 40), int((e >> 20) & 0xFFFFF), int(e & 0xFFFFF)};
    }
    return build_batch(s, px, iter, ray_begin, jitter);
}
int64_t tfo_sample_pixels(tfo_session* s, const int32_t* pixels, int n_rays) {
    std::vector<std::array<int, 3>> px(n_rays);
    for (int i = 0; i < n_rays; ++i) px[i] = {pixels[3 * i], pixels[3 * i + 1], pixels[3 * i + 2]};
    return build_batch(s, px, 0, 0, 0);
}
int tfo_batch_export(tfo_session* s, tfg_batch_view* out) {
    size_t n = s->rays.size(), S = s->t.size();
    if (out->capacity < S) return 1;
    if (out->rays) std::memcpy(out->rays, s->rays.data(), n * sizeof(tfg_ray_entry));
    if (out->offsets) std::memcpy(out->offsets, s->offsets.data(), (n + 1) * 4);
    if (out->t) std::memcpy(out->t, s->t.data(), S * 4);
    if (out->delta) std::memcpy(out->delta, s->delta.data(), S * 4);
    if (out->local) std::memcpy(out->local, s->local.data(), 3 * S * 4);
    if (out->slot) std::memcpy(out->slot, s->slot.data(), S);
    if (out->endpoint) std::memcpy(out->endpoint, s->endpoint.data(), S);
    return 0;
}

// forward_batch (field.hpp:186-188): per-sample sigma and rgb.
int tfo_forward(tfo_session* s, float* sigma_out, float* rgb_out) {
    size_t n = s->rays.size(), S = s->t.size();
    s->sigma.assign(S, 0.f);
    s->rgb.assign(3 * S, 0.f);
    int vd = 6 * s->sh.cfg.view_freqs;
    par_for(n, s->workers, [&](size_t b, size_t e, int) {
        SampleActs a;
        for (size_t i = b; i < e; ++i)
            for (uint32_t k = s->offsets[i]; k < s->offsets[i + 1]; ++k) {
                const TileRec& tr = s->tiles[s->slot_tile[s->slot[k]]];
                field_point(s->sh, tr.enc.data(), tr.dnet.data(), s->color.data(),
                            &s->local[3 * k], &s->venc[i * vd], a);
                s->sigma[k] = a.sigma;
                for (int c = 0; c < 3; ++c) s->rgb[3 * k + c] = a.rgb[c];
            }
    });
    if (sigma_out) std::memcpy(sigma_out, s->sigma.data(), S * 4);
    if (rgb_out) std::memcpy(rgb_out, s->rgb.data(), 3 * S * 4);
    return 0;
}

// render + color_loss + render backward (SPEC 361-378; loss convention of the
// example at SPEC 377: mean over rays and channels, grad 2(r-t)/(3B)).
int tfo_composite(tfo_session* s, float* ray_rgb, float* ray_depth, float* ray_op, float* dsig,
                  float* drgb, double* loss) {
    size_t n = s->rays.size(), S = s->t.size();
    if (s->sigma.size() != S) tfo_forward(s, nullptr, nullptr);
    s->dsig.assign(S, 0.f);
    s->drgb.assign(3 * S, 0.f);
    std::vector<double> lpart(n, 0.0);
    const float inv3b = 1.0f / (3.0f * float(s->tc.batch_rays));
    par_for(n, s->workers, [&](size_t b, size_t e, int) {
        for (size_t i = b; i < e; ++i) {
            uint32_t o = s->offsets[i], m = s->offsets[i + 1] - o;
            float rgb[3], dep, op;
            render_ray(int(m), &s->sigma[o], &s->rgb[3 * o], &s->t[o], &s->delta[o],
                       s->tc.background, rgb, &dep, &op, nullptr, nullptr, nullptr);
            float g[3];
            lpart[i] = color_loss_ray(rgb, s->rays[i].target, inv3b, g);
            render_ray(int(m), &s->sigma[o], &s->rgb[3 * o], &s->t[o], &s->delta[o],
                       s->tc.background, nullptr, nullptr, nullptr, g, &s->dsig[o],
                       &s->drgb[3 * o]);
            if (ray_rgb)
                for (int c = 0; c < 3; ++c) ray_rgb[3 * i + c] = rgb[c];
            if (ray_depth) ray_depth[i] = dep;
            if (ray_op) ray_op[i] = op;
        }
    });
    double L = 0;
    for (double x : lpart) L += x;
    if (loss) *loss = L / (3.0 * double(s->tc.batch_rays));
    if (dsig) std::memcpy(dsig, s->dsig.data(), S * 4);
    if (drgb) std::memcpy(drgb, s->drgb.data(), 3 * S * 4);
    return 0;
}

// backward_batch (field.hpp:190-197): privatized per worker, reduced in chunk order.
int tfo_backward(tfo_session* s) {
    size_t n = s->rays.size();
    int W = s->workers;
    if (size_t(W) > n) W = int(std::max<size_t>(n, 1));
    int ns = s->nslots;
    std::vector<std::vector<float>> ge(size_t(W) * ns), gd(size_t(W) * ns), gc(W);
    for (int w = 0; w < W; ++w) {
        for (int k = 0; k < ns; ++k) {
            ge[w * ns + k].assign(s->sh.enc_params, 0.f);
            gd[w * ns + k].assign(s->sh.dnet_params, 0.f);
        }
        gc[w].assign(s->sh.color_params, 0.f);
    }
    int vd = 6 * s->sh.cfg.view_freqs;
    int E = s->sh.cfg.embedding;
    par_for(n, W, [&](size_t b, size_t e, int w) {
        SampleActs a;
        for (size_t i = b; i < e; ++i)
            for (uint32_t k = s->offsets[i]; k < s->offsets[i + 1]; ++k) {
                int sl = s->slot[k];
                const TileRec& tr = s->tiles[s->slot_tile[sl]];
                field_point(s->sh, tr.enc.data(), tr.dnet.data(), s->color.data(),
                            &s->local[3 * k], &s->venc[i * vd], a);
                float dco[3];
                for (int c = 0; c < 3; ++c) {
                    float r = a.rgb[c];
                    dco[c] = s->drgb[3 * k + c] * r * (1.f - r);
                }
                float dcin[64];
                mlp_bwd<float>(s->sh.cw, s->color.data(), a.cacts, dco, gc[w].data(), dcin);
                float ddo[16];
                ddo[0] = s->dsig[k] * a.draw;
                for (int q = 0; q < E; ++q) ddo[1 + q] = dcin[q];
                float dfeat[16];
                mlp_bwd<float>(s->sh.dw, tr.dnet.data(), a.dacts, ddo, gd[w * ns + sl].data(),
                               dfeat);
                hash_backward<float>(s->sh, &s->local[3 * k], dfeat, ge[w * ns + sl].data());
            }
    });
    s->g_enc.assign(ns, std::vector<float>(s->sh.enc_params, 0.f));
    s->g_dnet.assign(ns, std::vector<float>(s->sh.dnet_params, 0.f));
    s->g_color.assign(s->sh.color_params, 0.f);
    for (int w = 0; w < W; ++w) {
        for (int k = 0; k < ns; ++k) {
            for (size_t i = 0; i < s->sh.enc_params; ++i) s->g_enc[k][i] += ge[w * ns + k][i];
            for (size_t i = 0; i < s->sh.dnet_params; ++i) s->g_dnet[k][i] += gd[w * ns + k][i];
        }
        for (size_t i = 0; i < s->sh.color_params; ++i) s->g_color[i] += gc[w][i];
    }
    for (int k = 0; k < ns; ++k) {
        int ti = s->slot_tile[k];
        char nm[64];
        std::snprintf(nm, sizeof nm, "tile(%d,%d).enc", ti / s->cols, ti % s->cols);
        if (!finite_all(s->g_enc[k])) {
            g_err = std::string("backward_batch: non-finite gradient in group ") + nm;
            return 1;
        }
        std::snprintf(nm, sizeof nm, "tile(%d,%d).dnet", ti / s->cols, ti % s->cols);
        if (!finite_all(s->g_dnet[k])) {
            g_err = std::string("backward_batch: non-finite gradient in group ") + nm;
            return 1;
        }
    }
    if (!finite_all(s->g_color)) {
        g_err = "backward_batch: non-finite gradient in group color";
        return 1;
    }
    return 0;
}
// color_loss over n rays (rgb, target: 3 per ray) with batch size B: the
// batch loss and, if grad != NULL, the per-ray gradient at rgb.
double tfo_color_loss(const float* rgb, const float* target, int n, int batch, float* grad) {
    const float inv3b = 1.0f / (3.0f * float(batch));
    double L = 0;
    for (int i = 0; i < n; ++i) {
        float g[3];
        L += color_loss_ray(rgb + 3 * i, target + 3 * i, inv3b, g);
        if (grad)
            for (int c = 0; c < 3; ++c) grad[3 * i + c] = g[c];
    }
    return L / (3.0 * double(batch));
}

// ---- backward primitives, exposed so tests pin them bit-for-bit against the
// reference's MlpT::backward_p (nn.hpp:116-157) and HashGridT::backward
// (nn.hpp:231-245) compiled verbatim into oracle/_ref.
int tfo_mlp_fwd_bwd(const int* widths, int nw, const float* params, const float* x, float* out,
                    const float* d_out, float* grad, float* d_in) {
    std::vector<int> w(widths, widths + nw);
    std::vector<float> acts(Shapes::mlp_acts(w));
    mlp_fwd<float>(w, params, x, acts.data());
    for (int i = 0; i < w.back(); ++i) out[i] = acts[acts.size() - w.back() + i];
    if (d_out) mlp_bwd<float>(w, params, acts.data(), d_out, grad, d_in);
    return 0;
}
int tfo_hash_lookup_bwd(const tfg_field_config* cfg, const float* tables, int n, const float* p3,
                        float* out, const float* d_out, float* grad) {
    Shapes sh(*cfg);
    for (int i = 0; i < n; ++i) {
        hash_lookup<float>(sh, tables, p3 + 3 * i, out + size_t(i) * sh.L * sh.F);
        if (d_out && grad) hash_backward<float>(sh, p3 + 3 * i, d_out + size_t(i) * sh.L * sh.F, grad);
    }
    return 0;
}

// ---- float64 shadow of the batch loss and its reverse-mode gradient (the
// finite-difference oracle of SPEC.md:289-291, 683; field.hpp:127-128 templates
// the batch operators on the scalar for exactly this).  Same math as the fp32
// path (field_point, render_ray, color_loss, tfo_backward) instantiated in
// double on the session's current batch; parameters per loaded slot.
// Returns the loss; gradients are written (zeroed first) when g_* != NULL.
double tfo_shadow_loss_grad(tfo_session* s, const double* const* enc, const double* const* dnet,
                            const double* color, double* const* g_enc, double* const* g_dnet,
                            double* g_color) {
    using S = double;
    const Shapes& sh = s->sh;
    const int ns = s->nslots, vd = 6 * sh.cfg.view_freqs, E = sh.cfg.embedding;
    const bool grad = g_enc && g_dnet && g_color;
    if (grad) {
        for (int k = 0; k < ns; ++k) {
            std::fill(g_enc[k], g_enc[k] + sh.enc_params, 0.0);
            std::fill(g_dnet[k], g_dnet[k] + sh.dnet_params, 0.0);
        }
        std::fill(g_color, g_color + sh.color_params, 0.0);
    }
    const S inv3b = 1.0 / (3.0 * double(s->tc.batch_rays));
    const S dmax = S(sh.cfg.density_max);
    double L = 0.0;
    const size_t nd = Shapes::mlp_acts(sh.dw), nc = Shapes::mlp_acts(sh.cw);
    for (size_t i = 0; i < s->rays.size(); ++i) {
        const uint32_t o = s->offsets[i], m = s->offsets[i + 1] - o;
        std::vector<S> feat(size_t(m) * 16), dacts(size_t(m) * nd), cacts(size_t(m) * nc), sg(m), draw(m), rgb(3 * size_t(m));
        S venc[64];
        for (int q = 0; q < vd; ++q) venc[q] = S(s->venc[i * vd + q]);
        for (uint32_t j = 0; j < m; ++j) {
            const uint32_t k = o + j;
            const int sl = s->slot[k];
            S loc[3] = {S(s->local[3 * k]), S(s->local[3 * k + 1]), S(s->local[3 * k + 2])};
            hash_lookup<S>(sh, enc[sl], loc, &feat[16 * j]);
            mlp_fwd<S>(sh.dw, dnet[sl], &feat[16 * j], &dacts[nd * j]);
            const S* dout = &dacts[nd * j] + sh.dw[0] + sh.dw[1];
            sg[j] = density_act<S>(dout[0], dmax, &draw[j]);
            S cin[64];
            for (int q = 0; q < E; ++q) cin[q] = dout[1 + q];
            for (int q = 0; q < vd; ++q) cin[E + q] = venc[q];
            mlp_fwd<S>(sh.cw, color, cin, &cacts[nc * j]);
            const S* co = &cacts[nc * j] + nc - 3;
            for (int c = 0; c < 3; ++c) rgb[3 * j + c] = sigm<S>(co[c]);
        }
        // render (SPEC 361-369) in S
        S T = 1, acc[3] = {0, 0, 0};
        std::vector<S> w(m), Tn(m);
        for (uint32_t j = 0; j < m; ++j) {
            const S a = 1 - std::exp(-(sg[j] * S(s->delta[o + j])));
            w[j] = T * a;
            for (int c = 0; c < 3; ++c) acc[c] += w[j] * rgb[3 * j + c];
            T = T * (1 - a);
            Tn[j] = T;
        }
        S g[3];
        for (int c = 0; c < 3; ++c) {
            const S out = acc[c] + T * S(s->tc.background[c]);
            const S df = out - S(s->rays[i].target[c]);
            L += df * df;
            g[c] = 2 * df * inv3b;
        }
        if (!grad) continue;
        S R[3] = {T * S(s->tc.background[0]), T * S(s->tc.background[1]), T * S(s->tc.background[2])};
        for (int j = int(m) - 1; j >= 0; --j) {
            const uint32_t k = o + uint32_t(j);
            const int sl = s->slot[k];
            S dsg = 0;
            for (int c = 0; c < 3; ++c) dsg += g[c] * (Tn[j] * rgb[3 * j + c] - R[c]);
            dsg *= S(s->delta[k]);
            S dco[3];
            for (int c = 0; c < 3; ++c) {
                const S r = rgb[3 * j + c];
                dco[c] = w[j] * g[c] * r * (1 - r);
                R[c] += w[j] * rgb[3 * j + c];
            }
            S dcin[64];
            mlp_bwd<S>(sh.cw, color, &cacts[nc * j], dco, g_color, dcin);
            S ddo[16];
            ddo[0] = dsg * draw[j];
            for (int q = 0; q < E; ++q) ddo[1 + q] = dcin[q];
            S dfeat[16];
            mlp_bwd<S>(sh.dw, dnet[sl], &dacts[nd * j], ddo, g_dnet[sl], dfeat);
            S loc[3] = {S(s->local[3 * k]), S(s->local[3 * k + 1]), S(s->local[3 * k + 2])};
            hash_backward<S>(sh, loc, dfeat, g_enc[sl]);
        }
    }
    return L * inv3b;
}

int tfo_get_grads(tfo_session* s, int slot, float* enc, float* dnet, float* color) {
    if (slot < 0 || slot >= int(s->g_enc.size())) return 1;
    if (enc) std::memcpy(enc, s->g_enc[slot].data(), s->sh.enc_params * 4);
    if (dnet) std::memcpy(dnet, s->g_dnet[slot].data(), s->sh.dnet_params * 4);
    if (color) std::memcpy(color, s->g_color.data(), s->sh.color_params * 4);
    return 0;
}

// TileField::update_occupancy (field.hpp:100-102; SPEC 301-310): EMA <-
// max(decay*EMA, sigma at a jittered voxel point), jitter from
// (seed, OCCUPANCY, row, col, dnet step, voxel).
int tfo_update_occupancy(tfo_session* s) {
    int R = s->sh.occ_res;
    size_t nv = size_t(R) * R * R;
    for (int k = 0; k < s->nslots; ++k) {
        int ti = s->slot_tile[k];
        TileRec& tr = s->tiles[ti];
        uint64_t base = hc(s->tc.seed, kPurposeOccupancy, uint64_t(ti / s->cols),
                           uint64_t(ti % s->cols), tr.dnet_step);
        par_for(nv, s->workers, [&](size_t b, size_t e, int) {
            for (size_t vi = b; vi < e; ++vi) {
                int x = int(vi % R), y = int((vi / R) % R), z = int(vi / (size_t(R) * R));
                Rng r(hc(base, uint64_t(vi)));
                float ux = r.flt(), uy = r.flt(), uz = r.flt();
                float p[3] = {(float(x) + ux) / float(R), (float(y) + uy) / float(R),
                              (float(z) + uz) / float(R)};
                float sg = sigma_point(s->sh, tr.enc.data(), tr.dnet.data(), p);
                float d = s->sh.cfg.occupancy_decay * tr.occ[vi];
                tr.occ[vi] = std::max(d, sg);
            }
        });
    }
    return 0;
}

// Adam over the window's groups in slot order (enc, dnet per slot), then the
// colour net; occupancy update when (iter+1) % interval == 0.
int tfo_optimizer_step(tfo_session* s, uint64_t iter) {
    const tfg_train_config& c = s->tc;
    for (int k = 0; k < s->nslots; ++k) {
        int ti = s->slot_tile[k];
        TileRec& tr = s->tiles[ti];
        char nm[64];
        std::snprintf(nm, sizeof nm, "tile(%d,%d).enc", ti / s->cols, ti % s->cols);
        if (adam(tr.enc.data(), s->g_enc[k].data(), tr.enc_m.data(), tr.enc_v.data(),
                 s->sh.enc_params, &tr.enc_step, c.lr_field, c.lr_decay_rate, c.lr_decay_steps,
                 c.beta1, c.beta2, c.eps, nm))
            return 1;
        std::snprintf(nm, sizeof nm, "tile(%d,%d).dnet", ti / s->cols, ti % s->cols);
        if (adam(tr.dnet.data(), s->g_dnet[k].data(), tr.dnet_m.data(), tr.dnet_v.data(),
                 s->sh.dnet_params, &tr.dnet_step, c.lr_field, c.lr_decay_rate,
                 c.lr_decay_steps, c.beta1, c.beta2, c.eps, nm))
            return 1;
    }
    if (adam(s->color.data(), s->g_color.data(), s->color_m.data(), s->color_v.data(),
             s->sh.color_params, &s->color_step, c.lr_color, c.lr_decay_rate, c.lr_decay_steps,
             c.beta1, c.beta2, c.eps, "color"))
        return 1;
    if (s->sh.cfg.occupancy_interval > 0 &&
        (iter + 1) % uint64_t(s->sh.cfg.occupancy_interval) == 0)
        tfo_update_occupancy(s);
    return 0;
}

int tfo_train_step(tfo_session* s, uint64_t iter, uint64_t ray_begin, int n_rays, double* loss) {
    if (tfo_sample(s, iter, ray_begin, n_rays, 1) < 0) return 1;
    tfo_forward(s, nullptr, nullptr);
    tfo_composite(s, nullptr, nullptr, nullptr, nullptr, nullptr, loss);
    if (tfo_backward(s)) return 1;
    return tfo_optimizer_step(s, iter);
}

int tfo_get_tile_state(tfo_session* s, int slot, tfg_tile_state* o) {
    if (slot < 0 || slot >= s->nslots) return 1;
    const TileRec& t = s->tiles[s->slot_tile[slot]];
    auto cp = [](float* dst, const std::vector<float>& v) {
        if (dst) std::memcpy(dst, v.data(), v.size() * 4);
    };
    cp(o->enc, t.enc);
    cp(o->dnet, t.dnet);
    cp(o->enc_m, t.enc_m);
    cp(o->enc_v, t.enc_v);
    cp(o->dnet_m, t.dnet_m);
    cp(o->dnet_v, t.dnet_v);
    cp(o->occupancy, t.occ);
    o->enc_step = t.enc_step;
    o->dnet_step = t.dnet_step;
    return 0;
}
int tfo_set_tile_state(tfo_session* s, int slot, const tfg_tile_state* in) {
    if (slot < 0 || slot >= s->nslots) return 1;
    TileRec& t = s->tiles[s->slot_tile[slot]];
    auto cp = [](std::vector<float>& v, const float* src) {
        if (src) std::memcpy(v.data(), src, v.size() * 4);
    };
    cp(t.enc, in->enc);
    cp(t.dnet, in->dnet);
    cp(t.enc_m, in->enc_m);
    cp(t.enc_v, in->enc_v);
    cp(t.dnet_m, in->dnet_m);
    cp(t.dnet_v, in->dnet_v);
    cp(t.occ, in->occupancy);
    t.enc_step = in->enc_step;
    t.dnet_step = in->dnet_step;
    return 0;
}
int tfo_get_color(tfo_session* s, float* p, float* m, float* v, uint64_t* step) {
    if (p) std::memcpy(p, s->color.data(), s->color.size() * 4);
    if (m) std::memcpy(m, s->color_m.data(), s->color.size() * 4);
    if (v) std::memcpy(v, s->color_v.data(), s->color.size() * 4);
    if (step) *step = s->color_step;
    return 0;
}
int tfo_set_color(tfo_session* s, const float* p, const float* m, const float* v,
                  uint64_t step) {
    if (p) std::memcpy(s->color.data(), p, s->color.size() * 4);
    if (m) std::memcpy(s->color_m.data(), m, s->color.size() * 4);
    if (v) std::memcpy(s->color_v.data(), v, s->color.size() * 4);
    s->color_step = step;
    return 0;
}

} // extern "C"
