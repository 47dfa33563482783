// tf_kernels.h — launch interfaces of the hot-path kernels (internal to
// libtilefield_gpu.so; the public boundary is include/tilefield_gpu.h).
#pragma once

#include <cuda_runtime.h>

#include "tf_common.cuh"

namespace tfg {

// Per-sample arrays in slot-bucketed order (bucket s holds the samples of
// slot s, rays ascending, each ray's segment samples contiguous).
struct SampleArrays {
    float4* local;     // x, y, z (owning tile's [0,1]^3 frame), w = ray index bits
    float2* td;        // t (m along the ray), delta (m)
    uint8_t* endpoint; // 1 for segment endpoints
    float4* io;        // K2: (sigma, r, g, b); K3 overwrites with the pre-activation
                       // gradients (d raw sigma, d pre-sigmoid r, g, b) for K4
};

// Hash-grid level layout (HashGridT::init, nn.hpp:180-195).
struct HashLayout {
    int res[kLevels];
    uint32_t off[kLevels];  // entry offset of the level
    int dense[kLevels];     // 1 when (res+1)^3 <= T (direct indexing)
    uint32_t mask;          // T - 1
    // 0: the default FieldConfig's layout, which the kernels fold in as
    // constants (tf_hash.cuh); 1: another n_min / n_max / table_size, read
    // from this struct at run time
    int generic;
};

struct AcceptArgs {
    const tfg_rpc* cams;
    const LocStart* loc;         // per view: rpc_loc_start at z_max, then at z_min (or null)
    int n_views;
    const uint64_t* view_start;  // candidate offset of each view (n_views)
    const int* union_rect;       // r0, r1, c0, c1 per view
    const int* crop_rect;        // r0, r1, c0, c1 per (view, loaded slot); empty: r0 >= r1
    uint64_t n_candidates;
    const double* east;          // grid_cols + 1 shared edges (tiler.cpp:18-27)
    const double* north;         // grid_rows + 1
    int grid_rows, grid_cols;
    int loaded_tile[kTrainSlots];
    int n_loaded;
    double z_min, z_max;
    // Per-window pixel memo (indexed like the candidates: view_start[v] +
    // (row - r0) * ncols + (col - c0) over the union rect).  The RPC inversion
    // and the tile-incidence test of a pixel depend only on the scene, so a
    // pixel solved for the previous window position is copied, not re-solved:
    // info = done | hit | bbox of the hit tiles, rays = o[3], d[3].  Bounded by
    // the window's crop union (O(1) in the grid size).
    uint32_t* m_info;
    double* m_rays;
    // the previous window's memo (null: none / reuse off), its union rects
    // (r0, c0, cols, rows per view) and crop byte offsets (pixel offset x 3)
    const uint32_t* o_info;
    const double* o_rays;
    const int* o_rect;
    const uint64_t* o_off;
    int win_r0, win_r1, win_c0, win_c1;  // the loaded tiles' rectangle (inclusive)
    // pixels the memo does not settle: candidate indices + their count
    // (the list lives in the scan's output buffer, which is free until the scan)
    uint32_t* todo;
    uint32_t* todo_n;
    int sms;
};
constexpr uint32_t kMemoDone = 1u << 31, kMemoHit = 1u << 30;

struct RaygenArgs {
    const tfg_rpc* cams;
    const LocStart* loc;     // per view: rpc_loc_start at z_max, then at z_min (or null)
    const uint64_t* accept;  // draw mode: accepted list
    const uint32_t* n_accept_dev;  // its length, read on device (no host sync per move)
    const double* memo_rays;  // draw mode: the window's pixel-ray memo (accept pass), indexed like the crop pixels
    const int32_t* pixels;   // pixel mode (render/eval): view,row,col triplets
    int pixel_pairs;         // ... or (row, col) pairs of view 0 (the render camera)
    const uint8_t* crop_bytes;
    const int* crop_rect;        // r0, c0, cols, rows per view
    const uint64_t* crop_offset; // byte offset of each view's crop
    uint64_t seed, iter, ray_begin;
    int n_rays;
    int jitter;
    double z_min, z_max;
    double spm;
    int cap;
    double delta_cap;
    SlotTable slots;
    const uint32_t* occ_bits[kMaxSlots];
};

// A caller-built RaySegmentBatch (ray_batch.hpp:13-49) in ray order, on the
// device (tfg_batch_import).
struct ImportArgs {
    const tfg_ray_entry* rays;
    const uint32_t* offsets;  // n_rays + 1
    const float* t;
    const float* delta;
    const float* local;       // 3 per sample
    const uint8_t* slot;
    const uint8_t* endpoint;
    int n_rays;
    int nslots;
};

struct FieldArgs {
    FieldPtrs f;
    HashLayout hl;
    float density_max, density_lim;  // lim = log(density_max) (nn.hpp:272)
    const TileDesc* tiles;
    const Status* status;
    const float4* venc;  // 6 float4 per ray
    SampleArrays s;
};

struct FieldGradArgs {
    float* g_enc[kMaxSlots];
    float* g_dnet[kMaxSlots];
    float* g_color;
};

struct CompositeArgs {
    const RayHdr* hdr;   // per ray: segment positions / counts, target
    int n_rays;
    int sms;             // the persistent grid is sized from it
    SampleArrays s;
    const Status* status_in;
    Status* status;
    float3 bg;
    float inv3b;         // 1 / (3 B_global)
    int backward;
    float* ray_rgb;      // 3 per ray (may be null)
    float* ray_depth;
    float* ray_opacity;
    float density_max;   // sigma == density_max <=> clamped activation (zero grad)
    float4* export_io;   // optional: (d_sigma, d_rgb) per sample in reference semantics
    double* loss_parts;  // one partial loss per block, summed by loss_reduce_kernel
};

struct AdamGroup {
    uint64_t offset, count;
    float lr, bc1, bc2;
    int half_slot;  // >= 0: a slot's hash tables, also written to its fp16 shadow
};
constexpr int kMaxGroups = 2 * kTrainSlots + 1;
struct AdamArgs {
    float* params;
    const float* grads;
    float* m;
    float* v;
    AdamGroup g[kMaxGroups];
    int n_groups;
    float beta1, beta2, omb1, omb2, eps;
    uint32_t* group_flags;  // non-finite flag per group
    // sticky non-finite record {flag, group, seq}: not cleared by the next
    // batch, so a skipped step stays visible (and later steps stay skipped,
    // like the reference's throw) until the host reads it
    uint32_t* sticky;
    uint32_t seq;           // host sequence number of this optimizer step
    void* enc16;            // fp16 table shadows (slot k at k * enc16_stride halves)
    uint64_t enc16_stride;
};

struct OccArgs {
    HashLayout hl;
    float density_lim;
    const float* enc[kTrainSlots];
    const float* dnet[kTrainSlots];
    float* ema[kTrainSlots];
    uint32_t* bits[kTrainSlots];
    uint64_t base_key[kTrainSlots];  // hash_combine(seed, OCC, row, col, dnet_step)
    int n;
    float decay, threshold, density_max;
    int update;  // 0: only recompute bits from the EMA
    const uint32_t* sticky;  // non-null: skip the EMA update after a skipped (non-finite) Adam step
};

int scan_exclusive(const uint32_t* in, uint64_t n, uint32_t* out, uint32_t* block_sums,
                   uint32_t* grand_total, cudaStream_t st, uint64_t* launches);
int launch_accept(const AcceptArgs& a, uint32_t* flags, uint32_t* pos, uint32_t* block_sums,
                  uint32_t* n_out, uint64_t* out, cudaStream_t st, uint64_t* launches);
int launch_sampler(const RaygenArgs& a, RayRec* rays, RayHdr* hdr, float4* venc, uint32_t* counts,
                   uint32_t* P, uint32_t* block_sums, TileDesc* tiles, int max_tiles,
                   SampleArrays out, uint64_t capacity, Status* status, cudaStream_t st,
                   uint64_t* launches);
int launch_import(const ImportArgs& a, RayRec* rays, RayHdr* hdr, float4* venc, uint32_t* counts, uint32_t* P,
                  uint32_t* block_sums, TileDesc* tiles, int max_tiles, SampleArrays out, uint64_t capacity,
                  Status* status, cudaStream_t st, uint64_t* launches);
void launch_field_forward_tc(const FieldArgs& a, uint8_t* feat, int32_t* rays, int sms,
                             cudaStream_t st, uint64_t* launches);
void launch_field_backward_tc(const FieldArgs& a, const FieldGradArgs& g, uint8_t* feat,
                              int32_t* rays, int sms, cudaStream_t st, uint64_t* launches);
void launch_composite(const CompositeArgs& a, cudaStream_t st, uint64_t* launches);
void launch_adam(const AdamArgs& a, uint64_t total, cudaStream_t st, uint64_t* launches);
// fp32 hash tables of n slots (params + k * stride, enc_n floats) -> their fp16
// shadows (out + k * out_stride halves)
void launch_enc_half(const float* params, uint64_t stride, int n, uint64_t enc_n, uint64_t out_stride, void* out,
                     cudaStream_t st,
                     uint64_t* launches);
void launch_occupancy(const OccArgs& a, cudaStream_t st, uint64_t* launches);
// rpc_loc_start of n cameras at z_max and z_min -> out[2 v], out[2 v + 1]
void launch_loc_start(const tfg_rpc* cams, int n, double z_min, double z_max, LocStart* out, cudaStream_t st);


// Launch with programmatic stream serialization (the kernel calls
// pdl_wait() (tf_common.cuh) before reading its predecessor's outputs).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
#ifdef TFG_NO_PDL
    k<<<grid, block, smem, st>>>(static_cast<KArgs>(args)...);
    return cudaGetLastError();
#else
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
#endif
}

// evaluation metrics (k_eval.cu)
void launch_sq_diff(const float* a, const float* b, uint64_t n, double* out, int sms, cudaStream_t st);
void launch_abs_diff(const float* a, const float* b, const uint8_t* mask, uint64_t n, double* out, int sms,
                     cudaStream_t st);
void launch_ssim(const float* a, const float* b, int rows, int cols, const float* gw, double* out,
                 cudaStream_t st);
void launch_edge_band(const tfg_rpc* cam, const double* east, const double* north, int grid_rows,
                      int grid_cols, double z0, double z1, double step, uint64_t per_line, int band,
                      uint8_t* mask, cudaStream_t st);

} // namespace tfg
