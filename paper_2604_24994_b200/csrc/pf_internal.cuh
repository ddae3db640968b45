// pf_internal.cuh -- internal declarations of libpowerfoam (B200 / sm_100a).
// Nothing here is shared with oracle/ (the CPU oracle is independent code).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/powerfoam.h"

namespace pf {

constexpr int kTile = 16;           // 16x16-pixel tiles
constexpr int kTilePix = kTile * kTile;
constexpr float kTStop = 1e-4f;     // early termination threshold

// Per-view camera constants handed to kernels by value.
struct CamParams {
    int W, H, tiles_x, tiles_y;
    float fx, fy, cx, cy;
    float M[12];     // c2w row-major
    float near_plane;
    int model;       // PF_PINHOLE / PF_FISHEYE
    double ifx, ify; // 1 / fx, 1 / fy (fp64, host-computed; K6/K7 pixel rays)
};

// Device-side records built by K0 from the caller's arrays.
//   cellA[i] = (p.x, p.y, p.z, r)      cellB[i] = (sigma, R, G, B)
//   cellE[i] = (first edge, degree)    edges[q] = (n.x, n.y, n.z, k)
// with n = p_j - p_i and k = 0.5 * (|n|^2 - (w_j - w_i)) for edge q = (i -> j):
// the bounded cell of i keeps the side  a t' <= k + n.e  of the radical plane,
// a = d.n, in the cell-local ray frame (P:577-585 with the
// weight sign of SURVEY C1).
struct DeviceScene {
    int64_t N = 0, E = 0;
    const float *sites = nullptr, *weights = nullptr, *radii = nullptr, *density = nullptr,
                *rgb = nullptr;
    const int64_t *nbr_off = nullptr;
    const int32_t *nbr_idx = nullptr;
    float bg[3] = {0, 0, 0};
    float4 *cellA = nullptr, *cellB = nullptr, *edges = nullptr;
    uint2 *cellE = nullptr;
    const float *normals = nullptr;   // caller's dipole normals [N,3] or null
    float4 *cellN = nullptr;          // (n_i, 0) when dipoles are present
    // detail sites (NEXT-2)
    int K = 0;                        // detail sites per cell (0 = none)
    float sv_gamma = 0.0f, sv_tau = 0.0f;
    float sv_axes[24] = {};
    const float *duv = nullptr, *ddisp = nullptr, *dsv = nullptr;
    double *cellF = nullptr;          // per cell: m(3) u(3) v(3) 1/|n| 1/|e_k x m| k  (fp64)
    float *g_uv = nullptr, *g_disp = nullptr, *g_sv = nullptr;   // backward outputs (+=)
};
constexpr int kMaxDetail = 8;
constexpr int64_t kNoColCap = 0x7fffff0ll;   // colour slots per view (27-bit record field)
constexpr int kCellF = 12;

// grow-only device buffer
struct DevBuf {
    void *ptr = nullptr;
    size_t bytes = 0;
    cudaError_t reserve(size_t n);
    void release();
    template <class T> T *as() const { return static_cast<T *>(ptr); }
};

struct ViewState {
    CamParams cam{};
    int64_t P = 0;                           // tile/cell pairs of this view
    int64_t nvis = 0;                        // visible cells (count > 0)
    DevBuf rect, count, keybits;             // binning of this view (N-sized)
    DevBuf tdir;                             // fisheye: tile-centre rays (3T doubles) + cos/sin(th)
    uint32_t *vals_p = nullptr;              // sorted cell ids (the call's shared array)
    uint2 *ranges_p = nullptr;               // this view's per-tile [start,end) into vals_p
    int64_t pair_off = 0;                    // first pair of this view in the shared arrays
    uint32_t *order = nullptr;               // tiles by decreasing list length (K6/K7 grid order)
    uint32_t *chunk_off = nullptr;           // first 32-entry chunk of each tile
    // K6 -> K7 segment records (see pf_raster.cu): per (warp, chunk) descriptor
    // (first record, count | kOverflow), chunks walked per warp, the record arena
    DevBuf desc, wdone, rec;
    int64_t rec_cap = 0;                     // records the arena holds
    DevBuf saved;                            // float4[H*W] final (C + T bg, T)
    int64_t nseg = 0;                        // detail: segments of the last recording K6
    DevBuf col;                              // detail: colour slots (float4 rgb + delta)
    int64_t col_cap = 0;
};

struct BallBVH;   // pf_bvh.cuh

// Per-view arguments of the fused multi-view K6 / K7 launches (a device array,
// one entry per view; CTA b works on view b / T, tile order[b % T]).
struct ViewArgs {
    CamParams cam;
    const uint2 *ranges;
    const uint32_t *order, *vals, *chunk_off;
    float4 *out, *saved;
    const float4 *grad_out;
    uint2 *desc;
    uint32_t *wdone, *rec, *rec_used;
    uint32_t *seg_used;   // detail scenes: segments the recording K6 composited (sizes K7D items)
    float4 *col;          // detail scenes: per-segment colour + displacement slots (K6 -> K7)
    uint32_t *col_used;
    uint32_t rec_cap, col_cap;
};

// Items of the split detail backward (NEXT-2, pf_raster.cu): one per composited
// detail segment with a gradient, {cell, view << 25 | pixel, wa bits, g_ts bits},
// plus the parallel-ray chart parameter; written by K7, consumed by K7D.
struct DetailItems {
    uint4 *it;
    float *tpar;
    uint32_t *used;
    uint32_t cap;
};

// one sort batch of up to kBatchViews views (kernel parameter of the binning)
constexpr int kBatchViews = 8;
struct BatchViews {
    const int *count[kBatchViews];
    const uint32_t *keybits[kBatchViews];
    const int4 *rect[kBatchViews];
    const double *tdir[kBatchViews];
    CamParams cam[kBatchViews];
    int n;       // views in the batch
    int first;   // index of the batch's first view in the call
};

struct StageEvent {
    int stage;
    cudaEvent_t a, b;
    int launches;   // kernels launched between a and b
};

}  // namespace pf

struct pf_scene {
    int device = 0;
    uint32_t flags = 0;
    pf::DeviceScene ds;
    pf::DevBuf cellA, cellB, cellE, edges, cellN, cellF;
    bool edges_built = false;
    // sort / emit scratch
    pf::DevBuf keys0, keys1, vals1, sort_hist, scan_tmp, scan_totals;
    pf::DevBuf sort_status;         // onesweep: digit histograms, tickets, look-back status
    pf::DevBuf vals_all, ranges_all;   // sorted pairs of all views of the last call
    pf::DevBuf bvis, bvis_off, ptot;   // visible-cell counts per (view, block), pair totals
    pf::DevBuf ckeys0, ckeys1, cvals0, cvals1, ccnt, coffs;   // visible cells sorted by depth
    pf::DevBuf order_all, chunk_off_all;  // per-view tile orders / chunk offsets (V x T)
    pf::DevBuf acc;                 // backward packed accumulators
    pf::DevBuf rec_used;            // u32[2V] records used, then detail segments, per view (K6 atomics)
    pf::DevBuf items, item_tpar, item_cnt;   // split detail backward: K7 -> K7D items, counters
    uint32_t *pinned_seg = nullptr; // host readback of the segment counts (backward)
    int pinned_seg_n = 0;
    double rec_ratio = 3.0;         // arena capacity in records per (tile, cell) pair
    double col_ratio = 16.0;        // detail colour slots per pair (adapts like rec_ratio)
    bool col_ratio_fixed = false;   // PF_COL_RATIO set (tests of the recompute path)
    uint32_t *pinned_rec = nullptr; // host copy of rec_used from the previous forward
    int pinned_rec_n = 0, rec_seen_views = 0;
    std::vector<int64_t> rec_prev_P; // per-view pair counts of the forward pinned_rec came from
    bool rec_ratio_fixed = false;   // PF_REC_RATIO set (tests of the overflow path)
    std::vector<pf::ViewState> views;
    pf::ViewState debug_view;       // pf_debug_* scratch (leaves the forward state intact)
    std::vector<pf_camera> fwd_cams;
    int32_t fwd_views = 0;          // views saved by the last forward
    int64_t *pinned = nullptr;      // pinned host readback of pair totals
    int pinned_n = 0;
    int *pinned_hb = nullptr;       // pinned host readback of the per-block visible counts
    size_t pinned_hb_n = 0;
    int64_t launches = 0;
    bool profiling = false;
    cudaStream_t side = nullptr;    // K0 of a training forward runs here, beside K1-K5
    cudaEvent_t side_fork = nullptr, side_join = nullptr;
    // per-view K6 / K7 launches alternate between the call's stream and this one, so
    // one view's tail overlaps the next view's start (pf_raster.cu, view_streams)
    cudaStream_t pair = nullptr;
    cudaEvent_t pair_fork = nullptr, pair_join = nullptr;
    std::vector<pf::StageEvent> events;
    int64_t stage_l0 = 0;   // s->launches at the open stage's begin
    std::vector<cudaEvent_t> event_pool;
    // NEXT-4 tracer: the ball BVH (built per call; once for PF_STATIC_SCENE) and stats
    pf::BallBVH *bvh = nullptr;
    bool bvh_built = false;
    pf::DevBuf trace_stats, trace_nodes;   // stats; BVH nodes in the tracer's layout
    pf::DevBuf vargs;               // ViewArgs of the fused K6 / K7 launches
    pf::ViewArgs *pinned_args = nullptr;
    std::vector<pf::ViewArgs> host_args;
    int pinned_args_n = 0;
    int cull_on = -1;               // PF_PLANE_CULL (debug knob), read once per handle
    bool attrs_k6 = false, attrs_k7 = false;   // dynamic shared-memory attributes set
    int k6_per_view = -1;           // PF_K6_PER_VIEW (A/B knob): one K6 launch per view
};

namespace pf {

// ---- launch wrappers (defined in the .cu files); return cudaGetLastError() ----
cudaError_t launch_edge_records(pf_scene *s, cudaStream_t st);
cudaError_t launch_validate(pf_scene *s, int *d_flag, cudaStream_t st);
cudaError_t launch_preprocess(pf_scene *s, ViewState &v, cudaStream_t st);
// K1 of up to kBatchViews pinhole views in one launch (cells read once)
cudaError_t launch_preprocess_batch(pf_scene *s, const BatchViews &bv, cudaStream_t st);
cudaError_t radix_sort_pairs(pf_scene *s, uint64_t *keys, uint32_t *vals, uint64_t *keys_alt,
                             uint32_t *vals_alt, int64_t n, int end_bit, bool *result_in_alt,
                             cudaStream_t st);
cudaError_t radix_sort_pairs32(pf_scene *s, uint32_t *keys, uint32_t *vals, uint32_t *keys_alt,
                               uint32_t *vals_alt, int64_t n, int end_bit, bool *result_in_alt,
                               cudaStream_t st);
int vis_blocks(int64_t N);
cudaError_t launch_count_visible(pf_scene *s, const BatchViews &bv, int nbx, int *bvis,
                                 long long *ptot, cudaStream_t st);
cudaError_t launch_compact_visible(pf_scene *s, const BatchViews &bv, int nbx, const int *bvis,
                                   uint32_t *boff, long long *d_nvis, unsigned long long *keys,
                                   uint32_t *vals, cudaStream_t st);
cudaError_t launch_emit_sorted(pf_scene *s, const BatchViews &bv, int tile_bits,
                               const unsigned long long *skeys, const uint32_t *svals, int64_t n,
                               int *cnt_sorted, uint32_t *offs, long long *d_tot,
                               uint32_t *keys, uint32_t *vals, cudaStream_t st);
cudaError_t launch_full_keys(pf_scene *s, const uint32_t *tkeys, const uint32_t *vals,
                             const uint32_t *keybits, int64_t P, int tile_bits, uint64_t *out,
                             cudaStream_t st);
cudaError_t launch_ranges(pf_scene *s, const uint32_t *keys, int64_t P, int T, int tile_bits,
                          uint2 *ranges_all, int V, cudaStream_t st);
cudaError_t launch_tile_order(pf_scene *s, const uint2 *ranges_all, int T, int V,
                              uint32_t *order_all, uint32_t *chunk_off_all, cudaStream_t st);
// K6 over views [0, V) in ONE launch (args: the views' ViewArgs, device); counters
// (debug counting build) only with V == 1
cudaError_t launch_forward(pf_scene *s, const ViewState *views, int V, const ViewArgs *args,
                           int64_t *counters, bool record, float *st_contrib, float *st_normal,
                           cudaStream_t st);
cudaError_t launch_backward(pf_scene *s, const ViewState *views, int V, const ViewArgs *args,
                            cudaStream_t st);
// detail scenes: items the split backward's arena must hold (0: no split)
int64_t detail_items_needed(const pf_scene *s, const ViewState *views, int V);
cudaError_t pack_trace_nodes(pf_scene *s, BallBVH &bvh, DevBuf &nodes, cudaStream_t st);
cudaError_t launch_trace(pf_scene *s, const BallBVH &bvh, const CamParams &cam, float *out,
                         unsigned long long *stats, cudaStream_t st);
cudaError_t launch_unpack(pf_scene *s, float *gs, float *gw, float *gr, float *gd, float *gc,
                          float *gn, cudaStream_t st);

// small transfers without the copy engines: a one-block kernel copying 4-byte words
// between device and pinned host memory (pf_api.cu)
cudaError_t small_copy(pf_scene *s, void *dst, const void *src, size_t bytes, cudaStream_t st);

// stage timing helpers (pf_api.cu)
void stage_begin(pf_scene *s, int stage, cudaStream_t st, cudaEvent_t *ev);
void stage_end(pf_scene *s, int stage, cudaStream_t st, cudaEvent_t ev);

inline int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

}  // namespace pf
