// tf_common.cuh — shared host/device definitions of the B200 window hot path.
//
// Everything in this header that feeds the bit-exact contract (counter RNG,
// RPC projection, damped-Newton localisation, slab intersection, segment
// ordering, tile frames) is compiled with FMA contraction off (nvcc
// -fmad=false, host -ffp-contract=off) so each source operation rounds once,
// as in the reference's x86-64 build.  IEEE division and square root are the
// nvcc defaults (-prec-div/-prec-sqrt=true).
#pragma once

#include <cmath>
#include <cstdint>

#include "../../include/tilefield_gpu.h"

#ifdef __CUDACC__
#define TF_HD __host__ __device__ __forceinline__
#else
#define TF_HD inline
#endif

namespace tfg {

// ---------------------------------------------------------------- shapes
// The kernels are specialised for FieldConfig's defaults (nn.hpp:14-37).
constexpr int kLevels = 8;
constexpr int kFeat = 2;
constexpr int kTable = 1 << 15;
constexpr int kFeatDim = kLevels * kFeat;  // 16
constexpr int kDHidden = 64;
constexpr int kDOut = 16;                  // 1 + embedding(15)
constexpr int kEmb = 15;
constexpr int kViewFreqs = 4;
constexpr int kViewDim = 6 * kViewFreqs;   // 24
constexpr int kCIn = kEmb + kViewDim;      // 39
constexpr int kCHidden = 64;
constexpr int kOccRes = 32;
constexpr int kOccVox = kOccRes * kOccRes * kOccRes;
constexpr int kOccWords = kOccVox / 32;

// Flat parameter layouts of MlpT (nn.hpp:49-51): [W0(out x in), b0, W1, b1, ...].
constexpr int kDW1 = 0;                          // 64 x 16
constexpr int kDB1 = kDW1 + kDHidden * kFeatDim; // 1024
constexpr int kDW2 = kDB1 + kDHidden;            // 16 x 64
constexpr int kDB2 = kDW2 + kDOut * kDHidden;    // 2112
constexpr int kDnetParams = kDB2 + kDOut;        // 2128
constexpr int kCW1 = 0;                          // 64 x 39
constexpr int kCB1 = kCW1 + kCHidden * kCIn;     // 2496
constexpr int kCW2 = kCB1 + kCHidden;            // 64 x 64
constexpr int kCB2 = kCW2 + kCHidden * kCHidden; // 6656
constexpr int kCW3 = kCB2 + kCHidden;            // 3 x 64
constexpr int kCB3 = kCW3 + 3 * kCHidden;        // 6912
constexpr int kColorParams = kCB3 + 3;           // 6915

constexpr int kMaxSlots = 16;  // loaded tiles a batch may reference (render path)
constexpr int kTrainSlots = 4; // the 2x2 window
constexpr int kMaxSeg = 8;     // segments per ray (<= 3 in the configured regime)

// Stream purposes (rng.hpp:8-10: streams from (seed, purpose, counters)).
constexpr uint64_t kPurposePixels = 0x5049584Cull;
constexpr uint64_t kPurposeJitter = 0x4A495454ull;
constexpr uint64_t kPurposeTileEnc = 0x54454E43ull;
constexpr uint64_t kPurposeTileDnet = 0x54444E54ull;
constexpr uint64_t kPurposeColor = 0x434F4C52ull;
constexpr uint64_t kPurposeOccupancy = 0x4F434355ull;

// Programmatic dependent launch (launch_pdl): wait for the preceding grid's
// completion and memory before the first dependent access.
#ifdef __CUDACC__
__device__ __forceinline__ void pdl_wait() {
#ifndef TFG_NO_PDL
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
#endif
}
#endif

// ---------------------------------------------------------------- rng.hpp:11-48
TF_HD uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}
TF_HD uint64_t hash_combine(uint64_t a, uint64_t b) {
    return splitmix64(a ^ (b + 0x9e3779b97f4a7c15ull + (a << 6) + (a >> 2)));
}
TF_HD uint64_t mulhi64(uint64_t a, uint64_t b) {
#ifdef __CUDA_ARCH__
    return __umul64hi(a, b);
#else
    return uint64_t(((unsigned __int128)a * b) >> 64);
#endif
}
struct Rng {
    uint64_t s;
    TF_HD explicit Rng(uint64_t seed) : s(splitmix64(seed)) {}
    TF_HD uint64_t u64() { return s = splitmix64(s); }
    TF_HD double dbl() { return double(u64() >> 11) * 0x1.0p-53; }
    TF_HD float flt() { return float(u64() >> 40) * 0x1.0p-24f; }
    TF_HD uint64_t below(uint64_t n) { return mulhi64(u64(), n); }
    TF_HD double uniform(double lo, double hi) { return lo + (hi - lo) * dbl(); }
};

// ---------------------------------------------------------------- camera.cpp
// RPC00B rational cubic (camera.cpp:22-64).  Returns false where the
// reference's project() throws (|normalised coordinate| > 1.5).
// Coefficient load.  On the device it is a volatile load: the Newton loops
// would otherwise hoist all 80 loop-invariant coefficients into registers and
// spill (the camera is warp-uniform and L1-resident, so the reload is a
// broadcast).  The loaded value is the same either way.
TF_HD double rpc_coef(const double* p) {
#if defined(__CUDA_ARCH__) && !defined(TFG_RPC_HOIST)
    double v;
    asm volatile("ld.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
#else
    return *p;
#endif
}
TF_HD double rpc_poly(const double* c, double P, double L, double H) {
    // term order of rpc_terms (camera.cpp:22-43); left-to-right dot product
    // with each product formed in the reference's operand order.
    double s = 0;
    s += rpc_coef(c + 0) * 1.0;
    s += rpc_coef(c + 1) * L;
    s += rpc_coef(c + 2) * P;
    s += rpc_coef(c + 3) * H;
    s += rpc_coef(c + 4) * (L * P);
    s += rpc_coef(c + 5) * (L * H);
    s += rpc_coef(c + 6) * (P * H);
    s += rpc_coef(c + 7) * (L * L);
    s += rpc_coef(c + 8) * (P * P);
    s += rpc_coef(c + 9) * (H * H);
    s += rpc_coef(c + 10) * (P * L * H);
    s += rpc_coef(c + 11) * (L * L * L);
    s += rpc_coef(c + 12) * (L * P * P);
    s += rpc_coef(c + 13) * (L * H * H);
    s += rpc_coef(c + 14) * (L * L * P);
    s += rpc_coef(c + 15) * (P * P * P);
    s += rpc_coef(c + 16) * (P * H * H);
    s += rpc_coef(c + 17) * (L * L * H);
    s += rpc_coef(c + 18) * (P * P * H);
    s += rpc_coef(c + 19) * (H * H * H);
    return s;
}
// The four central-difference projections of a Newton iteration at once:
// every coefficient is loaded once and applied to the four points (the
// solve's bound is the L1 writeback of its coefficient loads).  Each point's
// arithmetic is exactly rpc_project's, in the same order.  Returns false if
// any point falls outside the valid cube (where project() would throw).
TF_HD void rpc_poly4(const double* c, const double* P, const double* L, double H, double* s) {
#pragma unroll
    for (int i = 0; i < 4; ++i) s[i] = 0;
    double k;
#define TFG_TERM4(n, expr)                                         \
    k = rpc_coef(c + n);                                           \
    _Pragma("unroll") for (int i = 0; i < 4; ++i) {                \
        const double Li = L[i], Pi = P[i];                         \
        (void)Li;                                                  \
        (void)Pi;                                                  \
        s[i] += k * (expr);                                        \
    }
    TFG_TERM4(0, 1.0)
    TFG_TERM4(1, Li)
    TFG_TERM4(2, Pi)
    TFG_TERM4(3, H)
    TFG_TERM4(4, Li * Pi)
    TFG_TERM4(5, Li * H)
    TFG_TERM4(6, Pi * H)
    TFG_TERM4(7, Li * Li)
    TFG_TERM4(8, Pi * Pi)
    TFG_TERM4(9, H * H)
    TFG_TERM4(10, Pi * Li * H)
    TFG_TERM4(11, Li * Li * Li)
    TFG_TERM4(12, Li * Pi * Pi)
    TFG_TERM4(13, Li * H * H)
    TFG_TERM4(14, Li * Li * Pi)
    TFG_TERM4(15, Pi * Pi * Pi)
    TFG_TERM4(16, Pi * H * H)
    TFG_TERM4(17, Li * Li * H)
    TFG_TERM4(18, Pi * Pi * H)
    TFG_TERM4(19, H * H * H)
#undef TFG_TERM4
}
TF_HD bool rpc_project4(const tfg_rpc& c, const double* x, const double* y, double z, double* row, double* col) {
    double L[4], P[4];
    const double H = (z - c.height_off) / c.height_scale;
    bool ok = fabs(H) <= 1.5;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        L[i] = (x[i] - c.long_off) / c.long_scale;
        P[i] = (y[i] - c.lat_off) / c.lat_scale;
        ok = ok && fabs(L[i]) <= 1.5 && fabs(P[i]) <= 1.5;
    }
    if (!ok) return false;
    double ln[4], ld[4], sn[4], sd[4];
    rpc_poly4(c.line_num, P, L, H, ln);
    rpc_poly4(c.line_den, P, L, H, ld);
    rpc_poly4(c.samp_num, P, L, H, sn);
    rpc_poly4(c.samp_den, P, L, H, sd);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        row[i] = c.line_off + c.line_scale * (ln[i] / ld[i]);
        col[i] = c.samp_off + c.samp_scale * (sn[i] / sd[i]);
    }
    return true;
}
TF_HD bool rpc_project(const tfg_rpc& c, double x, double y, double z, double* row, double* col) {
    double L = (x - c.long_off) / c.long_scale;
    double P = (y - c.lat_off) / c.lat_scale;
    double H = (z - c.height_off) / c.height_scale;
    if (!(fabs(L) <= 1.5 && fabs(P) <= 1.5 && fabs(H) <= 1.5)) return false;
    double rn = rpc_poly(c.line_num, P, L, H) / rpc_poly(c.line_den, P, L, H);
    double cn = rpc_poly(c.samp_num, P, L, H) / rpc_poly(c.samp_den, P, L, H);
    *row = c.line_off + c.line_scale * rn;
    *col = c.samp_off + c.samp_scale * cn;
    return true;
}

// 2x2 solve with Eigen FullPivLU's operation order (camera.cpp:84; see
// column-major first-maximum pivot, l = a/p, u = a - l*b, rank
// threshold |maxpivot| * 2 eps, forward then back substitution, Q permute).
TF_HD void lu2_solve(double a00, double a01, double a10, double a11, double b0, double b1,
                     double* x0, double* x1) {
    int pr = 0, pc = 0;
    double big = fabs(a00);
    double v = fabs(a10);
    if (v > big) { big = v; pr = 1; pc = 0; }
    v = fabs(a01);
    if (v > big) { big = v; pr = 0; pc = 1; }
    v = fabs(a11);
    if (v > big) { big = v; pr = 1; pc = 1; }
    if (big == 0.0) { *x0 = 0.0; *x1 = 0.0; return; }
    if (pr) { double t = a00; a00 = a10; a10 = t; t = a01; a01 = a11; a11 = t; }
    if (pc) { double t = a00; a00 = a01; a01 = t; t = a10; a10 = a11; a11 = t; }
    double l = a10 / a00;
    double u = a11 - l * a01;
    double maxp = big;
    int nonzero = 2;
    double bu = fabs(u);
    if (bu == 0.0) nonzero = 1;
    else if (bu > maxp) maxp = bu;
    double thr = fabs(maxp) * (2.220446049250313e-16 * 2.0);
    int rank = (fabs(a00) > thr) + (nonzero == 2 && fabs(u) > thr);
    if (rank == 0) { *x0 = 0.0; *x1 = 0.0; return; }
    double c0 = b0, c1 = b1;
    if (pr) { double t = c0; c0 = c1; c1 = t; }
    c1 = c1 - c0 * l;
    double r0, r1;
    if (rank == 2) {
        c1 = c1 / u;
        c0 = c0 - c1 * a01;
        c0 = c0 / a00;
        r0 = c0;
        r1 = c1;
    } else {
        r0 = c0 / a00;
        r1 = 0.0;
    }
    if (pc) { *x0 = r1; *x1 = r0; } else { *x0 = r0; *x1 = r1; }
}

TF_HD double hyp2(double a, double b) { return sqrt(a * a + b * b); }

// The pixel-independent head of localize at one height: every solve starts
// at the RPC centre, so the first projection and the first iteration's four
// Jacobian projections are the same for all pixels of a camera.  Computed
// once per (camera, height) with the same code, they are the same bits.
struct LocStart {
    int st;                  // 0; 1: the centre projection threw; 2: the first Jacobian's did
    double r, q;             // projection of the centre
    double pr4[4], pc4[4];   // the four central-difference points around it
};
TF_HD void rpc_loc_start(const tfg_rpc& c, double h, LocStart* s) {
    const double x = c.long_off, y = c.lat_off;
    const double hx = 1e-6 * c.long_scale;
    const double hy = 1e-6 * c.lat_scale;
    s->st = 0;
    if (!rpc_project(c, x, y, h, &s->r, &s->q)) {
        s->st = 1;
        return;
    }
    const double px[4] = {x + hx, x - hx, x + 0.0, x - 0.0};
    const double py[4] = {y + 0.0, y - 0.0, y + hy, y - hy};
    if (!rpc_project4(c, px, py, h, s->pr4, s->pc4)) s->st = 2;
}

// localize (camera.cpp:66-103): damped Newton at fixed height, central FD
// Jacobian (step 1e-6 * scale), <= 6 step halvings, tol 1e-4 px, <= 50 its.
// 0 ok, 1 project() threw, 2 no convergence.  `start` (optional): this
// camera's and height's rpc_loc_start, which replaces the first projection
// and the first iteration's Jacobian projections (same results, bit for bit).
TF_HD int rpc_localize(const tfg_rpc& c, double pr, double pc, double h, double* gx, double* gy,
                       const LocStart* start = nullptr) {
    double x = c.long_off, y = c.lat_off;
    const double hx = 1e-6 * c.long_scale;
    const double hy = 1e-6 * c.lat_scale;
    double r, q;
    if (start) {
        if (start->st == 1) return 1;
        r = start->r;
        q = start->q;
    } else if (!rpc_project(c, x, y, h, &r, &q)) {
        return 1;
    }
    double f0 = r - pr, f1 = q - pc;
    for (int it = 1; it <= 50; ++it) {
        double fn = hyp2(f0, f1);
        if (fn < 1e-4) { *gx = x; *gy = y; return 0; }
        double a0, a1, b0, b1, c0, c1, d0, d1;
        if (start && it == 1) {
            if (start->st == 2) return 1;
            a0 = start->pr4[0]; a1 = start->pc4[0];
            b0 = start->pr4[1]; b1 = start->pc4[1];
            c0 = start->pr4[2]; c1 = start->pc4[2];
            d0 = start->pr4[3]; d1 = start->pc4[3];
        } else {
            const double px[4] = {x + hx, x - hx, x + 0.0, x - 0.0};
            const double py[4] = {y + 0.0, y - 0.0, y + hy, y - hy};
            double pr4[4], pc4[4];
            if (!rpc_project4(c, px, py, h, pr4, pc4)) return 1;
            a0 = pr4[0]; a1 = pc4[0];
            b0 = pr4[1]; b1 = pc4[1];
            c0 = pr4[2]; c1 = pc4[2];
            d0 = pr4[3]; d1 = pc4[3];
        }
        // residual differences: (p_a - px) - (p_b - px)
        double j00 = ((a0 - pr) - (b0 - pr)) / (2 * hx);
        double j10 = ((a1 - pc) - (b1 - pc)) / (2 * hx);
        double j01 = ((c0 - pr) - (d0 - pr)) / (2 * hy);
        double j11 = ((c1 - pc) - (d1 - pc)) / (2 * hy);
        double s0, s1;
        lu2_solve(j00, j01, j10, j11, -f0, -f1, &s0, &s1);
        double lam = 1.0;
        double nx = x + s0, ny = y + s1;
        if (!rpc_project(c, nx, ny, h, &r, &q)) return 1;
        double n0 = r - pr, n1 = q - pc;
        for (int k = 0; k < 6 && hyp2(n0, n1) > hyp2(f0, f1); ++k) {
            lam *= 0.5;
            nx = x + lam * s0;
            ny = y + lam * s1;
            if (!rpc_project(c, nx, ny, h, &r, &q)) return 1;
            n0 = r - pr;
            n1 = q - pc;
        }
        x = nx;
        y = ny;
        f0 = n0;
        f1 = n1;
    }
    if (hyp2(f0, f1) < 1e-4) { *gx = x; *gy = y; return 0; }
    return 2;
}

// ray_from_pixel (camera.cpp:105-124) from the two localisations (top at
// z_max, bottom at z_min); |delta| summed as (x²+y²)+z².
TF_HD int rpc_ray_finish(double tx, double ty, double bx, double by, double zmin, double zmax,
                         double* o, double* d) {
    double dx = bx - tx, dy = by - ty, dz = zmin - zmax;
    double len = sqrt(dx * dx + dy * dy + dz * dz);
    if (!(len > 1e-12 && zmax > zmin)) return 3;
    o[0] = tx;
    o[1] = ty;
    o[2] = zmax;
    d[0] = dx / len;
    d[1] = dy / len;
    d[2] = dz / len;
    return 0;
}

TF_HD int rpc_ray(const tfg_rpc& c, int row, int col, double zmin, double zmax, double* o,
                  double* d) {
    double tx, ty, bx, by;
    int st = rpc_localize(c, double(row), double(col), zmax, &tx, &ty);
    if (st) return st;
    st = rpc_localize(c, double(row), double(col), zmin, &bx, &by);
    if (st) return st;
    double dx = bx - tx, dy = by - ty, dz = zmin - zmax;
    double len = sqrt(dx * dx + dy * dy + dz * dz);
    if (!(len > 1e-12 && zmax > zmin)) return 3;
    o[0] = tx;
    o[1] = ty;
    o[2] = zmax;
    d[0] = dx / len;
    d[1] = dy / len;
    d[2] = dz / len;
    return 0;
}

// ---------------------------------------------------------------- geometry.cpp:9-30
TF_HD bool slab(const double* o, const double* d, const double* box, double* t0o, double* t1o) {
    double t0 = 0.0, t1 = HUGE_VAL;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        if (d[k] == 0.0) {
            if (o[k] < box[k] || o[k] > box[3 + k]) return false;
            continue;
        }
        double inv = 1.0 / d[k];
        double ta = (box[k] - o[k]) * inv;
        double tb = (box[3 + k] - o[k]) * inv;
        if (ta > tb) { double t = ta; ta = tb; tb = t; }
        t0 = (t0 < ta) ? ta : t0;  // std::max(t0, ta) exactly (signed zeros included)
        t1 = (tb < t1) ? tb : t1;  // std::min(t1, tb)
        if (t0 > t1) return false;
    }
    if (t1 - t0 < 1e-6) return false;
    *t0o = t0;
    *t1o = t1;
    return true;
}

// OccupancyGrid::voxel_index (field.hpp:71-77), x fastest.
TF_HD int voxel_index(float x, float y, float z) {
    int ix = int(x * float(kOccRes)), iy = int(y * float(kOccRes)), iz = int(z * float(kOccRes));
    ix = ix < 0 ? 0 : (ix >= kOccRes ? kOccRes - 1 : ix);
    iy = iy < 0 ? 0 : (iy >= kOccRes ? kOccRes - 1 : iy);
    iz = iz < 0 ? 0 : (iz >= kOccRes ? kOccRes - 1 : iz);
    return ix + kOccRes * (iy + kOccRes * iz);
}

// ---------------------------------------------------------------- device structs
// Loaded tiles of one batch: boxes (min xyz, max xyz) and frames (origin,
// inv_size) in the scene frame, and the per-slot parameter pointers.
struct SlotTable {
    int n;
    double box[kMaxSlots][6];
    double frame[kMaxSlots][6];
};

struct FieldPtrs {
    const float* enc[kMaxSlots];
    // fp16 shadow of each slot's hash tables (__half2 per entry): what the
    // forward gather reads (as instant-ngp stores its tables); kept in step
    // with the fp32 master tables by Adam and by a conversion on reload
    const void* enc16[kMaxSlots];
    const float* dnet[kMaxSlots];
    const uint32_t* occ_bits[kMaxSlots];
    const float* color;
};

// One ray of a batch (RaySegmentBatch::RayEntry, ray_batch.hpp:14-20, plus
// its ordered segments).
struct RayRec {
    double o[3], d[3];
    double tn[kMaxSeg], tf[kMaxSeg];
    float target[3];
    int view, row, col;
    int nseg;
    int status;                 // 0 ok, else ray_from_pixel failure code
    uint8_t slot[kMaxSeg];
    uint16_t nint[kMaxSeg];     // intervals of the segment (n samples = nint+1 before culling)
    uint16_t cnt[kMaxSeg];      // kept samples of the segment
};

// What compositing needs of a ray, in one 64 B line (written by the sample
// writer once the bucket positions are known): the bucket position and kept
// count of each segment in ray order, the target colour; nseg < 0 marks a
// failed ray (no loss, no gradient).
struct alignas(16) RayHdr {
    uint32_t base[kMaxSeg];
    uint16_t cnt[kMaxSeg];
    float target[3];
    int32_t nseg;
};
static_assert(sizeof(RayHdr) == 64, "RayHdr is one 64 B line");

// Tile of <= 128 consecutive samples of one slot bucket (K2/K4 work unit).
struct TileDesc {  // 8 B: mlp_fwd_kernel loads it as one uint2
    uint32_t start;
    uint16_t n;
    uint16_t slot;
};
static_assert(sizeof(TileDesc) == 8, "TileDesc is loaded as one uint2");

// Status word bits (read back with the loss).
enum : uint32_t {
    kStatusRayFail = 1u << 0,
    kStatusSampleOverflow = 1u << 1,
    kStatusNonFinite = 1u << 2,
    kStatusSegOverflow = 1u << 3,
    kStatusBadBatch = 1u << 4,  // imported batch: a ray's samples are not <= 1 run per loaded slot
};

struct Status {
    uint32_t bits;
    uint32_t nonfinite_group;
    uint64_t n_samples;
    uint32_t n_tiles;
    uint32_t pad;
    double loss;
};

} // namespace tfg
