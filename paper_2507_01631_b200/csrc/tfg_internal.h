// tfg_internal.h — host-side internals shared by the C-ABI translation units
// (tfg_api.cu: context, scene, window slide, training, render;
// tfg_io.cu: checkpoints + crop cache; tfg_eval.cu: evaluation metrics).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <memory>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "tf_common.cuh"
#include "tf_kernels.h"

namespace tfg {
namespace host {

// Records the thread-local message returned by tfg_last_error.
int fail(int code, const std::string& msg);
void comm_release(tfg_ctx* c);  // tfg_comm.cu

#define CK(call)                                                                            \
    do {                                                                                    \
        cudaError_t e_ = (call);                                                            \
        if (e_ != cudaSuccess)                                                              \
            return fail(TFG_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

struct TileHost {
    bool created = false;
    float* rec = nullptr;  // pinned: [params(stride) | m(stride) | v(stride) | ema(32^3)]
    uint64_t enc_step = 0, dnet_step = 0;
};

// Background TileField::create of the host records (the Rng stream of a tile
// is inherently sequential: 434k draws whose state is the previous output).
// Workers initialise tiles in snake first-visit order; ensure_record waits
// for a tile that is not ready yet.
struct InitPool {
    std::vector<std::thread> workers;
    std::vector<int> order;
    std::atomic<size_t> next{0};
    std::unique_ptr<std::atomic<int>[]> ready;
    std::atomic<bool> stop{false};
};

enum Phase { kPhSampler, kPhFieldFwd, kPhComposite, kPhFieldBwd, kPhAdam, kPhOccupancy,
             kPhAccept, kNumPhases };
inline const char* const kPhaseNames[kNumPhases] = {"sampler", "field_fwd", "composite", "field_bwd",
                                                    "adam", "occupancy", "accept"};

struct WinBuf {
    uint8_t* d_crops = nullptr;      // per-view union crop, u8 RGB
    int* d_crop_rect = nullptr;      // r0, c0, cols, rows per view
    uint64_t* d_crop_off = nullptr;  // byte offset of each view's crop
    uint64_t* d_accept = nullptr;    // packed (view, row, col)
    uint32_t* d_n = nullptr;         // accepted count (read by the ray draw on device)
    // pixel memo of this window's crop union (indexed like the crop pixels):
    // state (done | hit | hit-tile bbox) and the FP64 ray o[3], d[3]
    uint32_t* d_minfo = nullptr;
    double* d_mrays = nullptr;
    std::vector<int> h_crop_rect;
    std::vector<uint64_t> h_crop_off;
    int pos_r = -1, pos_c = -1;
    cudaEvent_t ready = nullptr;
};

struct Crop {
    int r0 = 0, r1 = 0, c0 = 0, c1 = 0;
    bool empty() const { return r0 >= r1 || c0 >= c1; }
};

} // namespace host
} // namespace tfg

using namespace tfg;
using namespace tfg::host;

struct tfg_ctx {
    int device = 0;
    void* comm = nullptr;  // ncclComm_t of tfg_comm_init (tfg_comm.cu)
    int comm_rank = 0, comm_ranks = 0;
    int sms = 148;
    cudaStream_t st = nullptr, side = nullptr;
    bool own_stream = true;
    cudaEvent_t ev_main = nullptr, ev_side = nullptr;
    tfg_field_config fc{};
    tfg_train_config tc{};
    HashLayout hl{};
    // floats per slot: hash tables (enc_n), density MLP (dn_n).  A slot's
    // record is [tables | pad | density MLP | pad]: the MLP at dn_off =
    // enc_n rounded up to 16 B, the next slot at stride = dn_off + dn_n
    // rounded up to 16 B (vector loads, reds and Adam's float4 groups need
    // aligned bases; the default FieldConfig needs no padding).
    // enc16_stride: halves per slot of the fp16 shadows (8 B aligned).
    uint64_t enc_n = 0, dn_n = 0, dn_off = 0, stride = 0, enc16_stride = 0, n_params = 0, color_off = 0;
    float density_lim = 0.f;
    int max_rays = 0;
    uint64_t sample_cap = 0;
    int max_tiles = 0;
    uint64_t launches = 0;

    // parameters / optimizer
    float *d_params = nullptr, *d_grads = nullptr, *d_m = nullptr, *d_v = nullptr;
    float* d_ema = nullptr;
    uint32_t* d_bits = nullptr;
    // fp16 shadows of the hash tables for the forward gather: training slots
    // [0, kTrainSlots), render slots after them; Adam keeps the training ones
    // current, any other write of the slot parameters marks them dirty
    void* d_enc16 = nullptr;
    bool enc16_dirty = true;
    uint32_t* d_group_flags = nullptr;
    Status* d_status = nullptr;
    Status* h_status = nullptr;
    uint64_t color_step = 0;
    // Optimizer steps whose Adam status the host has not read yet: their
    // step-count increments are rolled back (once) if the device reports a
    // non-finite gradient at or before them (sticky record {flag, group, seq}).
    struct StepRec {
        uint32_t seq;
        int tile[kTrainSlots];
        int nslots;
    };
    std::vector<StepRec> unverified;
    uint32_t step_seq = 0;
    uint32_t* d_sticky = nullptr;
    uint32_t* h_sticky = nullptr;  // pinned, 4 words
    std::string nonfinite_pending;  // message of a consumed record, raised by the next status check
    uint32_t sticky_done_seq = 0;   // failing step of the last consumed record (later snapshots repeat it)
    // pipelined status reads (tfg_loss_request / tfg_loss_poll): pinned
    // snapshots of the status + sticky record, one event each
    static constexpr int kRing = 4;
    Status* h_ring = nullptr;
    uint32_t* h_ring_sticky = nullptr;  // kRing x 4
    cudaEvent_t ev_ring[kRing] = {};
    uint32_t ring_seq[kRing] = {};
    uint32_t ring_head = 0, ring_tail = 0;

    // scene
    int n_views = 0;
    std::vector<tfg_rpc> cams;
    tfg_rpc* d_cams = nullptr;
    std::vector<uint8_t*> h_images;
    tfg_roi roi{};
    int rows = 0, cols = 0;
    std::vector<double> east, north;
    double *d_east = nullptr, *d_north = nullptr;
    std::vector<TileHost> tiles;

    // window
    int pos_r = -1, pos_c = -1;
    int nslots = 0;
    int slot_tile[kTrainSlots] = {-1, -1, -1, -1};
    SlotTable slots{};

    // per-window staging (crops + accepted-ray list), double buffered so the
    // next position can be staged on the side stream while this one trains
    WinBuf win[2];
    int front = 0;
    cudaEvent_t ev_swap = nullptr;  // main-stream point after which the back buffer is free
    // Tile records staged by prefetch_window (H2D ahead of the move) and the
    // evicted records awaiting their asynchronous D2H; record layout as the
    // host's: params | m | v (stride each) | occupancy EMA.
    float* d_stage_in = nullptr;
    float* d_stage_out = nullptr;
    int stage_tile[kTrainSlots] = {-1, -1, -1, -1};
    cudaEvent_t ev_stage_in = nullptr;   // side stream: staged H2D done
    cudaEvent_t ev_stage_read = nullptr; // main stream: staged records consumed
    cudaEvent_t ev_out_done = nullptr;   // side stream: evicted D2H done
    uint64_t crop_cap = 0, accept_cap = 0, cand_cap = 0;
    // accepted-list build scratch (one build at a time)
    uint32_t *d_flags = nullptr, *d_pos = nullptr, *d_block_sums = nullptr, *d_acc_sums = nullptr;
    uint32_t* d_todo_n = nullptr;  // accept: count of pixels the memo does not settle
    uint64_t* d_view_start = nullptr;
    bool memo_reuse = true;  // copy pixels solved for the previous window (TFG_NO_MEMO_REUSE=1: off)
    int *d_union = nullptr, *d_crop4 = nullptr;

    // batch
    RayRec* d_rays = nullptr;
    RayHdr* d_hdr = nullptr;  // per-ray composite header (written with the samples)
    float4* d_venc = nullptr;
    // rpc_loc_start per scene view (z_max, z_min) and for the render camera
    LocStart* d_loc = nullptr;
    LocStart* d_rloc = nullptr;
    uint32_t *d_counts = nullptr, *d_P = nullptr;
    double* d_loss_parts = nullptr;  // per-block partial losses of K3
    TileDesc* d_tiles = nullptr;
    SampleArrays s{};
    float* d_ray_out = nullptr;  // rgb(3) | depth | opacity per ray
    // render pipeline: pinned double buffers (pixels in, outputs + status out)
    int32_t* h_rpix = nullptr;   // 2 x max_rays x (row, col)
    float* h_rout = nullptr;     // 2 x max_rays x 5
    Status* h_rstat = nullptr;   // 2
    cudaEvent_t ev_rdone[2] = {nullptr, nullptr};
    int32_t* d_pixels = nullptr;
    uint8_t* d_feat = nullptr;    // bf16 feature tiles (4 KB per 128-sample tile)
    int32_t* d_tile_rays = nullptr;
    float4* d_export = nullptr;   // parity export of (d_sigma, d_rgb) in ray semantics
    int cur_rays = 0;
    bool have_batch = false;
    bool fwd_done = false;  // feature tiles of the current batch are resident
    bool io_fwd = false;    // io holds the forward's (sigma, rgb) (not yet K3's gradients)
    uint8_t* d_imp = nullptr;  // batch import staging (ray-order arrays of a caller batch)

    bool render_mode = false;

    // render
    float* d_rparams = nullptr;  // kMaxSlots * stride
    uint32_t* d_rbits = nullptr;
    float* d_rcolor = nullptr;
    int rn = 0;
    SlotTable rslots{};
    tfg_rpc* d_rcam = nullptr;

    uint64_t bytes_total = 0;
    std::unordered_map<void*, uint64_t> alloc_bytes;  // device allocations (memory_report)
    uint64_t h2d_bytes = 0, d2h_bytes = 0;
    float* h_records = nullptr;  // one pinned block for every tile record
    InitPool init;

    // per-phase device timing (CUDA events on the context stream)
    bool prof = false;
    std::vector<cudaEvent_t> ev_pool;
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev_open;
    double prof_ms[kNumPhases] = {};
    uint64_t prof_n[kNumPhases] = {};
    uint64_t prof_launch[kNumPhases] = {};
};

namespace tfg {
namespace host {

// Every device buffer of a context goes through dalloc/dfree, so
// memory_report's total_device is the live HBM footprint.
template <typename T>
int dalloc(tfg_ctx* c, T** p, uint64_t n) {
    if (n == 0) n = 1;
    CK(cudaMalloc(reinterpret_cast<void**>(p), n * sizeof(T)));
    c->bytes_total += n * sizeof(T);
    c->alloc_bytes[*p] = n * sizeof(T);
    return 0;
}
template <typename T>
void dfree(tfg_ctx* c, T*& p) {
    if (!p) return;
    auto it = c->alloc_bytes.find(static_cast<void*>(p));
    if (it != c->alloc_bytes.end()) {
        c->bytes_total -= it->second;
        c->alloc_bytes.erase(it);
    }
    cudaFree(static_cast<void*>(p));
    p = nullptr;
}

// shared helpers (defined in tfg_api.cu)
void tile_box(const tfg_ctx* c, int ti, double* b);
bool crop_for_tile(const tfg_rpc& cam, const double* box, int margin, Crop* out);
std::vector<int> window_tiles(const tfg_ctx* c, int pr, int pc);
int ensure_record(tfg_ctx* c, int ti);
int slot_copy(tfg_ctx* c, int slot, int ti, bool to_host);
int settle_steps(tfg_ctx* c);

} // namespace host
} // namespace tfg
