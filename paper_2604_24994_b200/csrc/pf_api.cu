// pf_api.cu -- host side of the C ABI (include/powerfoam.h): handle, argument
// checks, grow-only workspaces, per-view saved state, error strings, stage timing.
#include <cuda_runtime.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <new>
#include <string>

#include <nvtx3/nvToolsExt.h>

#include "pf_bvh.cuh"
#include "pf_internal.cuh"

namespace {

thread_local std::string g_err;

int fail(int code, const std::string &msg)
{
    g_err = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char *what)
{
    return fail(e == cudaErrorMemoryAllocation ? PF_ERR_OUT_OF_MEMORY : PF_ERR_CUDA,
                std::string(what) + ": " + cudaGetErrorString(e));
}

#define PF_CUDA(expr)                                        \
    do {                                                     \
        cudaError_t _e = (expr);                             \
        if (_e != cudaSuccess) return cuda_fail(_e, #expr);  \
    } while (0)

// restores the caller's current device on scope exit
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev)
    {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard()
    {
        int cur;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

bool finitef(float v) { return isfinite(v); }

int check_camera(const pf_camera &c)
{
    if (c.width < 1 || c.height < 1 || c.width > 32768 || c.height > 32768)
        return fail(PF_ERR_INVALID_ARGUMENT, "camera width/height must be in [1, 32768]");
    if (!(c.fx > 0.0f) || !(c.fy > 0.0f) || !finitef(c.fx) || !finitef(c.fy))
        return fail(PF_ERR_INVALID_ARGUMENT, "camera fx/fy must be finite and > 0");
    if (!finitef(c.cx) || !finitef(c.cy))
        return fail(PF_ERR_INVALID_ARGUMENT, "camera cx/cy must be finite");
    for (int k = 0; k < 12; ++k)
        if (!finitef(c.c2w[k])) return fail(PF_ERR_INVALID_ARGUMENT, "camera c2w not finite");
    if (!(c.near_plane > 0.0f) || !finitef(c.near_plane))
        return fail(PF_ERR_INVALID_ARGUMENT, "camera near_plane must be finite and > 0");
    if (c.model != PF_PINHOLE && c.model != PF_FISHEYE)
        return fail(PF_ERR_INVALID_ARGUMENT, "camera model must be PF_PINHOLE or PF_FISHEYE");
    return PF_OK;
}

pf::CamParams cam_params(const pf_camera &c)
{
    pf::CamParams p;
    p.W = c.width;
    p.H = c.height;
    p.tiles_x = (c.width + pf::kTile - 1) / pf::kTile;
    p.tiles_y = (c.height + pf::kTile - 1) / pf::kTile;
    p.fx = c.fx;
    p.fy = c.fy;
    p.cx = c.cx;
    p.cy = c.cy;
    for (int k = 0; k < 12; ++k) p.M[k] = c.c2w[k];
    p.near_plane = c.near_plane;
    p.model = c.model;
    p.ifx = 1.0 / (double)c.fx;
    p.ify = 1.0 / (double)c.fy;
    return p;
}

int tile_bits(int T)
{
    int b = 0;
    while ((1 << b) < T) ++b;
    return b;
}

int reserve_view_bins(pf_scene *s, pf::ViewState &v)
{
    size_t N = (size_t)s->ds.N;
    PF_CUDA(v.rect.reserve(16 * N));
    PF_CUDA(v.count.reserve(4 * N));
    PF_CUDA(v.keybits.reserve(4 * N));
    if (v.cam.model == PF_FISHEYE)
        PF_CUDA(v.tdir.reserve(sizeof(double) * (3 * (size_t)v.cam.tiles_x * v.cam.tiles_y + 2)));
    return PF_OK;
}

// The views of one sort batch as a kernel parameter.
pf::BatchViews batch_views(pf::ViewState *views, int b0, int b1)
{
    pf::BatchViews bv;
    memset(&bv, 0, sizeof(bv));
    bv.n = b1 - b0;
    bv.first = b0;
    for (int v = b0; v < b1; ++v) {
        bv.count[v - b0] = views[v].count.as<int>();
        bv.keybits[v - b0] = views[v].keybits.as<uint32_t>();
        bv.rect[v - b0] = views[v].rect.as<int4>();
        bv.tdir[v - b0] = views[v].tdir.as<double>();
        bv.cam[v - b0] = views[v].cam;
    }
    return bv;
}

pf::ViewArgs view_args(pf::ViewState &vs, float *out, const float *grad_out, bool record)
{
    pf::ViewArgs a;
    memset(&a, 0, sizeof(a));
    a.cam = vs.cam;
    a.ranges = vs.ranges_p;
    a.order = vs.order;
    a.vals = vs.vals_p;
    a.chunk_off = vs.chunk_off;
    a.out = (float4 *)out;
    a.saved = record ? vs.saved.as<float4>() : nullptr;
    a.grad_out = (const float4 *)grad_out;
    a.desc = record ? vs.desc.as<uint2>() : nullptr;
    a.wdone = record ? vs.wdone.as<uint32_t>() : nullptr;
    a.rec = record ? vs.rec.as<uint32_t>() : nullptr;
    a.rec_cap = (uint32_t)vs.rec_cap;
    a.col = (record && vs.col_cap) ? vs.col.as<float4>() : nullptr;   // detail scenes
    a.col_cap = (uint32_t)vs.col_cap;
    return a;
}

// The ViewArgs of a fused K6 / K7 launch: staged in pinned memory (slot 0 forward,
// slot 1 backward; every reuse of a slot follows a host sync of the call that used
// it) and copied to the handle's device array on the call's stream.
int upload_view_args(pf_scene *s, const pf::ViewArgs *a, int V, int slot, cudaStream_t st,
                     const pf::ViewArgs **dev)
{
    const int per = V + 8;
    if (s->pinned_args_n < per) {
        if (s->pinned_args) cudaFreeHost(s->pinned_args);
        s->pinned_args = nullptr;
        s->pinned_args_n = 0;
        PF_CUDA(cudaMallocHost(&s->pinned_args, sizeof(pf::ViewArgs) * 2 * (size_t)per));
        s->pinned_args_n = per;
    }
    PF_CUDA(s->vargs.reserve(sizeof(pf::ViewArgs) * 2 * (size_t)s->pinned_args_n));
    pf::ViewArgs *h = s->pinned_args + (size_t)slot * s->pinned_args_n;
    memcpy(h, a, sizeof(pf::ViewArgs) * (size_t)V);
    pf::ViewArgs *d = s->vargs.as<pf::ViewArgs>() + (size_t)slot * s->pinned_args_n;
    PF_CUDA(pf::small_copy(s, d, h, sizeof(pf::ViewArgs) * (size_t)V, st));
    *dev = d;
    return PF_OK;
}

// Sorting and ranges for views [0, V) of this call (K1 and the visible-cell
// counts ran, every v.P is known), in batches of up to kBatchViews views:
//   K2: compact the visible cells of the batch (view-major, cell order);
//   K4a: radix-sort them by (view, depth key) -- 32 + view bits, ~N_vis items;
//   K3: emit their tile pairs in that order, key = view << tile_bits | tile;
//   K4b: stable radix sort of the pairs by (view, tile) (tile_bits + view bits);
//   K5: per-tile ranges, LPT tile order.
// Inside a tile the pairs are then ordered by (depth key, cell): the order of the
// stable (tile << 32 | key) sort of cell-major pairs.  Leaves the
// sorted (view, tile) keys in *keys_out (scratch) and the cell ids in s->vals_all.
int emit_sort_ranges(pf_scene *s, pf::ViewState *views, int V, cudaStream_t st,
                     uint32_t **keys_out)
{
    constexpr int kSortViews = pf::kBatchViews;
    const int T = views[0].cam.tiles_x * views[0].cam.tiles_y;
    const int tb = tile_bits(T);
    const int Vb = V < kSortViews ? V : kSortViews;
    int vb = 0;
    while ((1 << vb) < Vb) ++vb;
    if (tb + vb > 32) return fail(PF_ERR_INVALID_ARGUMENT, "too many tiles for the sort keys");
    int64_t Ptot = 0;
    for (int v = 0; v < V; ++v) {
        views[v].pair_off = Ptot;
        Ptot += views[v].P;
    }
    if (Ptot >= (int64_t)0xFFFFFFFFll)
        return fail(PF_ERR_OUT_OF_MEMORY, "pair count of one call exceeds 2^32");
    const size_t p = (size_t)(Ptot > 0 ? Ptot : 1);
    const size_t N = (size_t)s->ds.N;
    const size_t nv = N * (size_t)Vb + 1;   // visible cells of one batch, at most
    PF_CUDA(s->keys0.reserve(4 * p));
    PF_CUDA(s->keys1.reserve(4 * p));
    PF_CUDA(s->vals1.reserve(4 * p));
    PF_CUDA(s->vals_all.reserve(4 * p));
    PF_CUDA(s->ranges_all.reserve(sizeof(uint2) * (size_t)T * V));
    PF_CUDA(s->ckeys0.reserve(8 * nv));
    PF_CUDA(s->ckeys1.reserve(8 * nv));
    PF_CUDA(s->cvals0.reserve(4 * nv));
    PF_CUDA(s->cvals1.reserve(4 * nv));
    PF_CUDA(s->ccnt.reserve(4 * nv));
    PF_CUDA(s->coffs.reserve(4 * nv + 16));
    const int nbx = pf::vis_blocks((int64_t)N);
    PF_CUDA(s->bvis_off.reserve(4 * ((size_t)nbx * Vb + 16)));
    uint32_t *k0 = s->keys0.as<uint32_t>(), *k1 = s->keys1.as<uint32_t>();
    uint32_t *v0 = s->vals_all.as<uint32_t>(), *v1 = s->vals1.as<uint32_t>();
    uint2 *rall = s->ranges_all.as<uint2>();
    long long *d_tmp = s->scan_totals.as<long long>() + V;   // two scratch totals (bin_views)
    for (int b0 = 0; b0 < V; b0 += kSortViews) {
        const int b1 = (b0 + kSortViews < V) ? b0 + kSortViews : V;
        const int64_t off = views[b0].pair_off;
        const int64_t Pb = views[b1 - 1].pair_off + views[b1 - 1].P - off;
        const pf::BatchViews bv = batch_views(views, b0, b1);
        int64_t nvis = 0;
        for (int v = b0; v < b1; ++v) nvis += views[v].nvis;
        if (Pb > 0) {
            PF_CUDA(pf::launch_compact_visible(s, bv, nbx, s->bvis.as<int>(), s->bvis_off.as<uint32_t>(),
                                               d_tmp, s->ckeys0.as<unsigned long long>(),
                                               s->cvals0.as<uint32_t>(), st));
            bool alt = false;   // (radix_sort_pairs times itself as stage 4)
            PF_CUDA(pf::radix_sort_pairs(s, s->ckeys0.as<uint64_t>(), s->cvals0.as<uint32_t>(),
                                         s->ckeys1.as<uint64_t>(), s->cvals1.as<uint32_t>(), nvis,
                                         32 + vb, &alt, st));
            const unsigned long long *sk = (alt ? s->ckeys1 : s->ckeys0).as<unsigned long long>();
            const uint32_t *sv = (alt ? s->cvals1 : s->cvals0).as<uint32_t>();
            PF_CUDA(pf::launch_emit_sorted(s, bv, tb, sk, sv, nvis, s->ccnt.as<int>(),
                                           s->coffs.as<uint32_t>(), d_tmp + 1,
                                           k0 + off, v0 + off, st));
            PF_CUDA(pf::radix_sort_pairs32(s, k0 + off, v0 + off, k1 + off, v1 + off, Pb, tb + vb,
                                           &alt, st));
            if (alt) {
                PF_CUDA(cudaMemcpyAsync(v0 + off, v1 + off, 4 * (size_t)Pb, cudaMemcpyDeviceToDevice, st));
                PF_CUDA(cudaMemcpyAsync(k0 + off, k1 + off, 4 * (size_t)Pb, cudaMemcpyDeviceToDevice, st));
            }
        }
        // ranges of this batch's views, relative to the batch's first pair
        PF_CUDA(pf::launch_ranges(s, k0 + off, Pb, T, tb, rall + (size_t)b0 * T, b1 - b0, st));
        for (int v = b0; v < b1; ++v) {
            views[v].vals_p = v0 + off;
            views[v].ranges_p = rall + (size_t)v * T;
        }
    }
    PF_CUDA(s->order_all.reserve(sizeof(uint32_t) * (size_t)T * V));
    PF_CUDA(s->chunk_off_all.reserve(sizeof(uint32_t) * (size_t)T * V));
    for (int v = 0; v < V; ++v) {
        views[v].order = s->order_all.as<uint32_t>() + (size_t)v * T;
        views[v].chunk_off = s->chunk_off_all.as<uint32_t>() + (size_t)v * T;
    }
    PF_CUDA(pf::launch_tile_order(s, rall, T, V, s->order_all.as<uint32_t>(),
                                  s->chunk_off_all.as<uint32_t>(), st));
    *keys_out = k0;
    return PF_OK;
}

// K1 for views [0, V), the visible-cell and pair counts of every view (one
// kernel per sort batch), then one readback of all pair totals and visible
// counts (the call's only host sync before K6).
int bin_views_of(pf_scene *s, pf::ViewState *views, int V, cudaStream_t st)
{
    PF_CUDA(s->scan_totals.reserve(sizeof(int64_t) * (size_t)(V + 4)));
    PF_CUDA(s->ptot.reserve(sizeof(long long) * (size_t)V));
    long long *ptot = s->ptot.as<long long>();
    PF_CUDA(cudaMemsetAsync(ptot, 0, sizeof(long long) * (size_t)V, st));
    const int nbx = pf::vis_blocks(s->ds.N);
    PF_CUDA(s->bvis.reserve(sizeof(int) * ((size_t)nbx * V + 16)));
    for (int v = 0; v < V; ++v) {
        int rc = reserve_view_bins(s, views[v]);
        if (rc) return rc;
    }
    for (int b0 = 0; b0 < V; b0 += pf::kBatchViews) {
        const int b1 = (b0 + pf::kBatchViews < V) ? b0 + pf::kBatchViews : V;
        bool fish = false;
        for (int v = b0; v < b1; ++v) fish = fish || views[v].cam.model == PF_FISHEYE;
        if (fish || b1 - b0 == 1) {   // fisheye K1 (tile tests per view), or a single view
            for (int v = b0; v < b1; ++v) PF_CUDA(pf::launch_preprocess(s, views[v], st));
        } else {
            PF_CUDA(pf::launch_preprocess_batch(s, batch_views(views, b0, b1), st));
        }
    }
    for (int b0 = 0; b0 < V; b0 += pf::kBatchViews) {
        const int b1 = (b0 + pf::kBatchViews < V) ? b0 + pf::kBatchViews : V;
        PF_CUDA(pf::launch_count_visible(s, batch_views(views, b0, b1), nbx, s->bvis.as<int>(),
                                         ptot, st));
    }
    if ((int)s->pinned_n < 2 * V) {
        if (s->pinned) cudaFreeHost(s->pinned);
        s->pinned = nullptr;
        s->pinned_n = 0;
        PF_CUDA(cudaMallocHost(&s->pinned, sizeof(int64_t) * (size_t)(2 * V + 16)));
        s->pinned_n = 2 * V + 16;
    }
    // per view: the pair total, and the visible cells (a sum over its blocks)
    const size_t nhb = (size_t)nbx * V;
    if (s->pinned_hb_n < nhb) {
        if (s->pinned_hb) cudaFreeHost(s->pinned_hb);
        s->pinned_hb = nullptr;
        s->pinned_hb_n = 0;
        PF_CUDA(cudaMallocHost(&s->pinned_hb, sizeof(int) * nhb));
        s->pinned_hb_n = nhb;
    }
    const int *hb = s->pinned_hb;
    PF_CUDA(pf::small_copy(s, s->pinned, ptot, sizeof(int64_t) * (size_t)V, st));
    PF_CUDA(pf::small_copy(s, s->pinned_hb, s->bvis.ptr, sizeof(int) * nhb, st));
    PF_CUDA(cudaStreamSynchronize(st));
    for (int v = 0; v < V; ++v) {
        const int64_t P = s->pinned[v];
        if (P < 0 || P >= (int64_t)0xFFFFFFFFll)
            return fail(PF_ERR_OUT_OF_MEMORY, "tile/cell pair count exceeds 2^32");
        views[v].P = P;
        int64_t c = 0;
        for (int b = 0; b < nbx; ++b) c += hb[(size_t)v * nbx + b];
        views[v].nvis = c;
    }
    return PF_OK;
}

int bin_views(pf_scene *s, int V, cudaStream_t st)
{
    return bin_views_of(s, s->views.data(), V, st);
}

}  // namespace

// ---------------------------------------------------------------------------
namespace pf {

// Small host <-> device transfers of the call (ViewArgs up; pair / visible / record
// counts down) as a one-block kernel reading or writing pinned host memory directly
// (UVA maps cudaMallocHost memory), NOT as cudaMemcpyAsync: a training loop keeps the
// copy engines busy with its own transfers (the next dL/dimage up, the last gradients
// down), and a 2 KB copy queued behind a 265 MB one stalls the whole forward.
__global__ void k_small_copy(const uint32_t *__restrict__ src, uint32_t *__restrict__ dst, int n)
{
    for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
}

cudaError_t small_copy(pf_scene *s, void *dst, const void *src, size_t bytes, cudaStream_t st)
{
    if (!bytes) return cudaSuccess;
    ++s->launches;
    k_small_copy<<<1, 256, 0, st>>>(static_cast<const uint32_t *>(src), static_cast<uint32_t *>(dst),
                                    (int)(bytes / 4));
    return cudaGetLastError();
}

cudaError_t DevBuf::reserve(size_t n)
{
    if (n <= bytes && ptr) return cudaSuccess;
    size_t want = n + n / 4 + 256;
    if (ptr) {
        cudaError_t e = cudaDeviceSynchronize();  // the old buffer may still be in use
        if (e != cudaSuccess) return e;
        cudaFree(ptr);
        ptr = nullptr;
        bytes = 0;
    }
    cudaError_t e = cudaMalloc(&ptr, want);
    if (e != cudaSuccess) {
        ptr = nullptr;
        return e;
    }
    bytes = want;
    return cudaSuccess;
}

void DevBuf::release()
{
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
}

// NVTX range names of the stages (SURVEY §5 tracing): visible in nsys / ncu --nvtx
static const char *const kStageNames[PF_NUM_STAGES] = {
    "pf K0 edge records", "pf K1 preprocess", "pf K2 visible/compact", "pf K3 emit",
    "pf K4 sort", "pf K5 ranges", "pf K6 forward", "pf K7 backward", "pf K8 unpack"};

void stage_begin(pf_scene *s, int stage, cudaStream_t st, cudaEvent_t *ev)
{
    *ev = nullptr;
    nvtxRangePushA(kStageNames[stage]);   // host-side range around the stage's launches
    s->stage_l0 = s->launches;
    if (!s->profiling) return;
    if (s->event_pool.empty()) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) return;
        s->event_pool.push_back(e);
    }
    *ev = s->event_pool.back();
    s->event_pool.pop_back();
    cudaEventRecord(*ev, st);
}

void stage_end(pf_scene *s, int stage, cudaStream_t st, cudaEvent_t ev)
{
    nvtxRangePop();
    if (!ev) return;
    cudaEvent_t e2;
    if (s->event_pool.empty()) {
        if (cudaEventCreate(&e2) != cudaSuccess) return;
    } else {
        e2 = s->event_pool.back();
        s->event_pool.pop_back();
    }
    cudaEventRecord(e2, st);
    s->events.push_back(StageEvent{stage, ev, e2, (int)(s->launches - s->stage_l0)});
}

}  // namespace pf

// ---------------------------------------------------------------------------
extern "C" {

const char *pf_last_error(void) { return g_err.c_str(); }

int pf_create_scene(const pf_scene_desc *d, pf_scene **out, pf_stream_t stream)
{
    if (!out) return fail(PF_ERR_INVALID_ARGUMENT, "out handle pointer is NULL");
    *out = nullptr;
    if (!d) return fail(PF_ERR_INVALID_ARGUMENT, "scene descriptor is NULL");
    if (d->num_cells < 1) return fail(PF_ERR_INVALID_ARGUMENT, "num_cells must be >= 1");
    if (d->num_cells >= (int64_t)1 << 31)
        return fail(PF_ERR_INVALID_ARGUMENT, "num_cells must be < 2^31");
    if (d->num_edges < 0 || d->num_edges >= (int64_t)1 << 32)
        return fail(PF_ERR_INVALID_ARGUMENT, "num_edges must be in [0, 2^32)");
    if (!d->sites || !d->weights || !d->radii || !d->density || !d->rgb || !d->nbr_offsets ||
        (d->num_edges > 0 && !d->nbr_indices))
        return fail(PF_ERR_INVALID_ARGUMENT, "a scene array pointer is NULL");
    for (int c = 0; c < 3; ++c)
        if (!isfinite(d->background[c]))
            return fail(PF_ERR_INVALID_ARGUMENT, "background not finite");
    if (d->num_detail != 0) {
        if (d->num_detail < 0 || d->num_detail > pf::kMaxDetail)
            return fail(PF_ERR_INVALID_ARGUMENT, "num_detail must be 0 or 1..8");
        if (!d->normals)
            return fail(PF_ERR_INVALID_ARGUMENT, "detail sites need dipole normals");
        if (!d->detail_uv || !d->detail_disp || !d->detail_sv)
            return fail(PF_ERR_INVALID_ARGUMENT, "a detail array pointer is NULL");
        if (((uintptr_t)d->detail_uv & 7) || ((uintptr_t)d->detail_sv & 15))
            return fail(PF_ERR_INVALID_ARGUMENT,
                        "detail_uv must be 8-byte and detail_sv 16-byte aligned");
        if (!(d->sv_tau > 0.0f) || !isfinite(d->sv_tau) || !isfinite(d->sv_gamma))
            return fail(PF_ERR_INVALID_ARGUMENT, "sv_tau must be finite and > 0, sv_gamma finite");
        for (int a = 0; a < 24; ++a)
            if (!isfinite(d->sv_axes[a / 3][a % 3]))
                return fail(PF_ERR_INVALID_ARGUMENT, "sv_axes not finite");
    }
    cudaStream_t st = (cudaStream_t)stream;
    pf_scene *s = new (std::nothrow) pf_scene();
    if (!s) return fail(PF_ERR_OUT_OF_MEMORY, "host allocation failed");
    if (cudaGetDevice(&s->device) != cudaSuccess) {
        delete s;
        return fail(PF_ERR_CUDA, "no current CUDA device");
    }
    s->flags = d->flags;
    if (const char *r = getenv("PF_REC_RATIO")) {   // debug knob: K6->K7 record arena size
        const double v = atof(r);
        if (v > 0.0) s->rec_ratio = v;
        s->rec_ratio_fixed = v > 0.0;
    }
    if (const char *r = getenv("PF_COL_RATIO")) {   // debug knob: detail colour slots per pair
        const double v = atof(r);
        if (v >= 0.0) {
            s->col_ratio = v;
            s->col_ratio_fixed = true;
        }
    }
    pf::DeviceScene &ds = s->ds;
    ds.N = d->num_cells;
    ds.E = d->num_edges;
    ds.sites = d->sites;
    ds.weights = d->weights;
    ds.radii = d->radii;
    ds.density = d->density;
    ds.rgb = d->rgb;
    ds.nbr_off = d->nbr_offsets;
    ds.nbr_idx = d->nbr_indices;
    ds.normals = d->normals;
    for (int c = 0; c < 3; ++c) ds.bg[c] = d->background[c];
    if (d->num_detail > 0) {
        ds.K = d->num_detail;
        ds.sv_gamma = d->sv_gamma;
        ds.sv_tau = d->sv_tau;
        for (int a = 0; a < 24; ++a) ds.sv_axes[a] = d->sv_axes[a / 3][a % 3];
        ds.duv = d->detail_uv;
        ds.ddisp = d->detail_disp;
        ds.dsv = d->detail_sv;
    }
    int rc = PF_OK;
    do {
        size_t N = (size_t)ds.N, E = (size_t)(ds.E > 0 ? ds.E : 1);
        cudaError_t e;
        if ((e = s->cellA.reserve(16 * N)) != cudaSuccess) { rc = cuda_fail(e, "alloc cellA"); break; }
        if ((e = s->cellB.reserve(16 * N)) != cudaSuccess) { rc = cuda_fail(e, "alloc cellB"); break; }
        if ((e = s->cellE.reserve(8 * N)) != cudaSuccess) { rc = cuda_fail(e, "alloc cellE"); break; }
        if ((e = s->edges.reserve(16 * E)) != cudaSuccess) { rc = cuda_fail(e, "alloc edges"); break; }
        if (ds.normals) {
            if ((e = s->cellN.reserve(16 * N)) != cudaSuccess) { rc = cuda_fail(e, "alloc cellN"); break; }
            ds.cellN = s->cellN.as<float4>();
        }
        if (ds.K) {
            if ((e = s->cellF.reserve(sizeof(double) * pf::kCellF * N)) != cudaSuccess) { rc = cuda_fail(e, "alloc cellF"); break; }
            ds.cellF = s->cellF.as<double>();
        }
        ds.cellA = s->cellA.as<float4>();
        ds.cellB = s->cellB.as<float4>();
        ds.cellE = s->cellE.as<uint2>();
        ds.edges = s->edges.as<float4>();
        if (d->flags & PF_VALIDATE) {
            int *flag = nullptr;
            if ((e = cudaMalloc(&flag, sizeof(int))) != cudaSuccess) { rc = cuda_fail(e, "alloc"); break; }
            int host = 0;
            e = cudaMemsetAsync(flag, 0, sizeof(int), st);
            if (e == cudaSuccess) e = pf::launch_validate(s, flag, st);
            if (e == cudaSuccess) e = cudaMemcpyAsync(&host, flag, sizeof(int), cudaMemcpyDeviceToHost, st);
            if (e == cudaSuccess) e = cudaStreamSynchronize(st);
            cudaFree(flag);
            if (e != cudaSuccess) { rc = cuda_fail(e, "validation"); break; }
            if (host) {
                std::string why = "scene validation failed:";
                if (host & 1) why += " non-finite site;";
                if (host & 2) why += " non-finite rgb;";
                if (host & 4) why += " non-finite weight;";
                if (host & 8) why += " radius not finite/positive;";
                if (host & 16) why += " density not finite/non-negative;";
                if (host & 32) why += " bad neighbour offsets;";
                if (host & 64) why += " neighbour index out of range or self loop;";
                if (host & 128) why += " dipole normal zero or non-finite;";
                if (host & 256) why += " non-finite detail-site value;";
                rc = fail(PF_ERR_INVALID_ARGUMENT, why);
                break;
            }
        }
        if (d->flags & PF_STATIC_SCENE) {
            if ((e = pf::launch_edge_records(s, st)) != cudaSuccess) { rc = cuda_fail(e, "K0"); break; }
            s->edges_built = true;
        }
    } while (0);
    if (rc != PF_OK) {
        pf_destroy(s);
        return rc;
    }
    *out = s;
    return PF_OK;
}

int pf_destroy(pf_scene *s)
{
    if (!s) return PF_OK;
    DeviceGuard g(s->device);
    cudaDeviceSynchronize();
    if (s->bvh) {
        s->bvh->release();
        delete s->bvh;
        s->bvh = nullptr;
    }
    s->trace_stats.release();
    s->trace_nodes.release();
    s->cellA.release();
    s->cellB.release();
    s->cellE.release();
    s->edges.release();
    s->cellN.release();
    s->cellF.release();
    s->keys0.release();
    s->keys1.release();
    s->vals1.release();
    s->sort_hist.release();
    s->sort_status.release();
    s->scan_tmp.release();
    s->scan_totals.release();
    s->acc.release();
    for (auto &v : s->views) {
        v.rect.release();
        v.count.release();
        v.keybits.release();
        v.tdir.release();
        v.saved.release();
        v.desc.release();
        v.wdone.release();
        v.rec.release();
        v.col.release();
    }
    s->debug_view.rect.release();
    s->debug_view.count.release();
    s->debug_view.keybits.release();
    s->debug_view.tdir.release();
    s->vals_all.release();
    pf::DevBuf *cbufs[] = {&s->bvis, &s->bvis_off, &s->ptot, &s->ckeys0, &s->ckeys1,
                           &s->cvals0, &s->cvals1, &s->ccnt, &s->coffs};
    for (auto *b : cbufs) b->release();
    s->ranges_all.release();
    s->order_all.release();
    s->chunk_off_all.release();
    s->rec_used.release();
    s->items.release();
    s->item_tpar.release();
    s->item_cnt.release();
    if (s->pinned_seg) cudaFreeHost(s->pinned_seg);
    if (s->pinned) cudaFreeHost(s->pinned);
    if (s->pinned_rec) cudaFreeHost(s->pinned_rec);
    if (s->pinned_hb) cudaFreeHost(s->pinned_hb);
    if (s->pinned_args) cudaFreeHost(s->pinned_args);
    s->vargs.release();
    for (auto &e : s->events) {
        cudaEventDestroy(e.a);
        cudaEventDestroy(e.b);
    }
    for (auto e : s->event_pool) cudaEventDestroy(e);
    if (s->side) cudaStreamDestroy(s->side);
    if (s->pair) cudaStreamDestroy(s->pair);
    if (s->pair_fork) cudaEventDestroy(s->pair_fork);
    if (s->pair_join) cudaEventDestroy(s->pair_join);
    if (s->side_fork) cudaEventDestroy(s->side_fork);
    if (s->side_join) cudaEventDestroy(s->side_join);
    delete s;
    return PF_OK;
}

int pf_render_forward(pf_scene *s, const pf_camera *cams, int32_t V, float *out,
                      pf_stream_t stream)
{
    return pf_render_forward_ex(s, cams, V, out, nullptr, stream);
}

int pf_render_forward_ex(pf_scene *s, const pf_camera *cams, int32_t V, float *out,
                         const pf_forward_extras *ex, pf_stream_t stream)
{
    if (!s) return fail(PF_ERR_INVALID_ARGUMENT, "scene handle is NULL");
    if (!cams || V < 1) return fail(PF_ERR_INVALID_ARGUMENT, "need >= 1 camera");
    if (!out) return fail(PF_ERR_INVALID_ARGUMENT, "out is NULL");
    for (int v = 0; v < V; ++v) {
        int rc = check_camera(cams[v]);
        if (rc) return rc;
        if (cams[v].width != cams[0].width || cams[v].height != cams[0].height)
            return fail(PF_ERR_INVALID_ARGUMENT, "all views of one call must share width/height");
    }
    DeviceGuard g(s->device);
    cudaStream_t st = (cudaStream_t)stream;
    s->fwd_views = 0;
    bool k0_side = false;
    if (!(s->flags & PF_STATIC_SCENE) || !s->edges_built) {
        // K0 (edge records, read only by K6/K7) on a side stream, concurrent with the
        // binning and sort of K1-K5; joined before the first K6
        if (!s->side) {
            if (cudaStreamCreateWithFlags(&s->side, cudaStreamNonBlocking) != cudaSuccess ||
                cudaEventCreateWithFlags(&s->side_fork, cudaEventDisableTiming) != cudaSuccess ||
                cudaEventCreateWithFlags(&s->side_join, cudaEventDisableTiming) != cudaSuccess) {
                cudaGetLastError();
                if (s->side) cudaStreamDestroy(s->side);
    if (s->pair) cudaStreamDestroy(s->pair);
    if (s->pair_fork) cudaEventDestroy(s->pair_fork);
    if (s->pair_join) cudaEventDestroy(s->pair_join);
                s->side = nullptr;
            }
        }
        if (s->side) {
            PF_CUDA(cudaEventRecord(s->side_fork, st));
            PF_CUDA(cudaStreamWaitEvent(s->side, s->side_fork, 0));
            PF_CUDA(pf::launch_edge_records(s, s->side));
            PF_CUDA(cudaEventRecord(s->side_join, s->side));
            k0_side = true;
        } else {
            PF_CUDA(pf::launch_edge_records(s, st));
        }
        s->edges_built = true;
    }
    if ((int)s->views.size() < V) s->views.resize(V);
    for (int v = 0; v < V; ++v) s->views[v].cam = cam_params(cams[v]);
    int rc = bin_views(s, V, st);
    if (rc) return rc;
    const size_t npix = (size_t)cams[0].width * cams[0].height;
    const bool record = !(s->flags & PF_INFERENCE);
    if (record) {
        // adapt the record-arena size to what the previous forward used (records per
        // pair of THAT forward: bin_views has already overwritten views[v].P)
        if (s->rec_seen_views > 0 && !s->rec_ratio_fixed) {
            const int pv = s->rec_seen_views;
            for (int v = 0; v < pv; ++v) {
                const int64_t prevP = s->rec_prev_P[v];
                const uint32_t used = s->pinned_rec[v], segs = s->pinned_rec[pv + v];
                if (prevP > 0 && used > 0)
                    s->rec_ratio = fmax(s->rec_ratio * 0.98, 1.3 * (double)used / (double)prevP);
                const uint32_t cols = s->pinned_rec[2 * pv + v];   // slots claimed (warp blocks)
                if (prevP > 0 && (segs > 0 || cols > 0) && !s->col_ratio_fixed)
                    s->col_ratio = fmax(s->col_ratio * 0.98,
                                        1.2 * (double)(segs > cols ? segs : cols) / (double)prevP);
            }
        }
        // per view: records used, detail segments, detail colour slots used
        PF_CUDA(s->rec_used.reserve(sizeof(uint32_t) * 3 * (size_t)V));
        PF_CUDA(cudaMemsetAsync(s->rec_used.ptr, 0, sizeof(uint32_t) * 3 * (size_t)V, st));
    }
    uint32_t *ks_all = nullptr;
    rc = emit_sort_ranges(s, s->views.data(), V, st, &ks_all);
    if (rc) return rc;
    if (k0_side) PF_CUDA(cudaStreamWaitEvent(st, s->side_join, 0));
    s->host_args.resize(V);
    for (int v = 0; v < V; ++v) {
        pf::ViewState &vs = s->views[v];
        uint32_t *used = nullptr;
        if (record) {
            const int T = vs.cam.tiles_x * vs.cam.tiles_y;
            PF_CUDA(vs.saved.reserve(16 * npix));
            const size_t chunks = (size_t)(vs.P / 32 + T + 1);
            PF_CUDA(vs.desc.reserve(sizeof(uint2) * 8 * chunks));
            PF_CUDA(vs.wdone.reserve(sizeof(uint32_t) * 8 * (size_t)T));
            vs.rec_cap = (int64_t)(s->rec_ratio * (double)vs.P) + (s->rec_ratio_fixed ? 0 : 1024);
            if (vs.rec_cap > (int64_t)0xFFFFFFF0ll) vs.rec_cap = 0xFFFFFFF0ll;
            PF_CUDA(vs.rec.reserve(72 * (size_t)vs.rec_cap));
            used = s->rec_used.as<uint32_t>() + v;
            if (s->ds.K) {   // K6 -> K7 segment colours (a full arena: K7 recomputes)
                vs.col_cap = (int64_t)(s->col_ratio * (double)vs.P) + (s->col_ratio_fixed ? 0 : 1024);
                if (vs.col_cap > (int64_t)pf::kNoColCap) vs.col_cap = pf::kNoColCap;
                PF_CUDA(vs.col.reserve(16 * (size_t)vs.col_cap));
            }
        }
        pf::ViewArgs a = view_args(vs, out + 4 * npix * (size_t)v, nullptr, record);
        a.rec_used = used;
        a.seg_used = record ? s->rec_used.as<uint32_t>() + V + v : nullptr;
        if (record && s->ds.K) a.col_used = s->rec_used.as<uint32_t>() + 2 * V + v;
        s->host_args[v] = a;
    }
    {   // K6 of every view in one launch
        const pf::ViewArgs *dargs = nullptr;
        rc = upload_view_args(s, s->host_args.data(), V, 0, st, &dargs);
        if (rc) return rc;
        PF_CUDA(pf::launch_forward(s, s->views.data(), V, dargs, nullptr, record,
                                   ex ? ex->contrib : nullptr, ex ? ex->normal_term : nullptr, st));
    }
    if (record) {
        if (s->pinned_rec_n < 3 * V) {
            if (s->pinned_rec) cudaFreeHost(s->pinned_rec);
            s->pinned_rec = nullptr;
            s->pinned_rec_n = 0;
            PF_CUDA(cudaMallocHost(&s->pinned_rec, sizeof(uint32_t) * (size_t)(3 * V + 16)));
            s->pinned_rec_n = 3 * V + 16;
        }
        // (read at the next forward; a copy-engine transfer is fine here: nothing waits on it)
        PF_CUDA(cudaMemcpyAsync(s->pinned_rec, s->rec_used.ptr, sizeof(uint32_t) * 3 * (size_t)V,
                                cudaMemcpyDeviceToHost, st));
        s->rec_prev_P.resize(V);
        for (int v = 0; v < V; ++v) s->rec_prev_P[v] = s->views[v].P;
        s->rec_seen_views = V;   // read at the next forward, after its sync
    }
    s->fwd_cams.assign(cams, cams + V);
    s->fwd_views = record ? V : 0;
    return PF_OK;
}

int pf_render_backward(pf_scene *s, const pf_camera *cams, int32_t V, const float *grad_out,
                       float *grad_sites, float *grad_weights, float *grad_radii,
                       float *grad_density, float *grad_rgb, pf_stream_t stream)
{
    pf_grads g = {grad_sites, grad_weights, grad_radii, grad_density, grad_rgb, nullptr,
                  nullptr, nullptr, nullptr};
    return pf_render_backward_ex(s, cams, V, grad_out, &g, stream);
}

int pf_render_backward_ex(pf_scene *s, const pf_camera *cams, int32_t V, const float *grad_out,
                          const pf_grads *g, pf_stream_t stream)
{
    if (!s) return fail(PF_ERR_INVALID_ARGUMENT, "scene handle is NULL");
    if (!cams || V < 1 || !grad_out || !g)
        return fail(PF_ERR_INVALID_ARGUMENT, "need cameras, grad_out and gradient arrays");
    if (!g->sites || !g->weights || !g->radii || !g->density || !g->rgb)
        return fail(PF_ERR_INVALID_ARGUMENT, "a gradient array pointer is NULL");
    if (V != s->fwd_views || (int)s->fwd_cams.size() < V ||
        memcmp(cams, s->fwd_cams.data(), sizeof(pf_camera) * (size_t)V) != 0)
        return fail(PF_ERR_STATE, "backward needs the immediately preceding forward with the same cameras");
    DeviceGuard dg(s->device);
    cudaStream_t st = (cudaStream_t)stream;
    const size_t N = (size_t)s->ds.N;
    PF_CUDA(s->acc.reserve(N * 48));   // 12 floats per cell (pf_raster.cu)
    PF_CUDA(cudaMemsetAsync(s->acc.ptr, 0, N * 48, st));
    const size_t npix = (size_t)cams[0].width * cams[0].height;
    if (s->ds.K && g->detail_sv && ((uintptr_t)g->detail_sv & 7))
        return fail(PF_ERR_INVALID_ARGUMENT, "grads.detail_sv must be 8-byte aligned");
    s->ds.g_uv = g->detail_uv;        // detail-site gradients go straight to the caller (+=)
    s->ds.g_disp = g->detail_disp;
    s->ds.g_sv = g->detail_sv;
    int brc = PF_OK;
    if (s->ds.K && (npix >= ((size_t)1 << 25) || V > 128))
        return fail(PF_ERR_INVALID_ARGUMENT, "detail backward: at most 2^25 pixels per view and 128 views per call");
    if (s->ds.K) {
        // split detail backward: the item arena holds every segment the recording K6
        // composited (one host sync: the counts of the forward just issued)
        if (s->pinned_seg_n < V) {
            if (s->pinned_seg) cudaFreeHost(s->pinned_seg);
            s->pinned_seg = nullptr;
            s->pinned_seg_n = 0;
            PF_CUDA(cudaMallocHost(&s->pinned_seg, sizeof(uint32_t) * (size_t)(V + 16)));
            s->pinned_seg_n = V + 16;
        }
        PF_CUDA(pf::small_copy(s, s->pinned_seg, s->rec_used.as<uint32_t>() + V,
                               sizeof(uint32_t) * (size_t)V, st));
        PF_CUDA(cudaStreamSynchronize(st));
        for (int v = 0; v < V; ++v) s->views[v].nseg = s->pinned_seg[v];
        const int64_t cap = pf::detail_items_needed(s, s->views.data(), V);
        if (cap > (int64_t)0xFFFFFF00ll)
            return fail(PF_ERR_OUT_OF_MEMORY, "detail segments of one backward launch exceed 2^32");
        if (cap > 0) {
            PF_CUDA(s->items.reserve(16 * (size_t)cap));
            PF_CUDA(s->item_tpar.reserve(4 * (size_t)cap));
        }
        PF_CUDA(s->item_cnt.reserve(sizeof(uint32_t) * (size_t)V));
        PF_CUDA(cudaMemsetAsync(s->item_cnt.ptr, 0, sizeof(uint32_t) * (size_t)V, st));
    }
    s->host_args.resize(V);
    for (int v = 0; v < V; ++v)
        s->host_args[v] = view_args(s->views[v], nullptr, grad_out + 4 * npix * (size_t)v, true);
    const pf::ViewArgs *dargs = nullptr;
    brc = upload_view_args(s, s->host_args.data(), V, 1, st, &dargs);
    if (brc == PF_OK) {   // K7 of every view in one launch
        cudaError_t e = pf::launch_backward(s, s->views.data(), V, dargs, st);
        if (e != cudaSuccess) brc = cuda_fail(e, "K7");
    }
    s->ds.g_uv = s->ds.g_disp = s->ds.g_sv = nullptr;
    if (brc != PF_OK) return brc;
    if (s->ds.K && (s->flags & PF_VALIDATE) && pf::detail_items_needed(s, s->views.data(), V) > 0) {
        // every K7 item must have fitted the arena sized from the forward's segment
        // count (the replay finds exactly the recorded segments)
        PF_CUDA(pf::small_copy(s, s->pinned_seg, s->item_cnt.ptr, sizeof(uint32_t) * (size_t)V, st));
        PF_CUDA(cudaStreamSynchronize(st));
        const int64_t cap = pf::detail_items_needed(s, s->views.data(), V);
        for (int v = 0; v < V; ++v)
            if ((int64_t)s->pinned_seg[v] > cap)
                return fail(PF_ERR_STATE, "detail backward: more K7 items than the forward recorded segments");
    }
    PF_CUDA(pf::launch_unpack(s, g->sites, g->weights, g->radii, g->density, g->rgb,
                              s->ds.cellN ? g->normals : nullptr, st));
    return PF_OK;
}

int pf_trace_forward(pf_scene *s, const pf_camera *cams, int32_t V, float *out, int64_t *stats,
                     pf_stream_t stream)
{
    if (!s) return fail(PF_ERR_INVALID_ARGUMENT, "scene handle is NULL");
    if (!cams || V < 1) return fail(PF_ERR_INVALID_ARGUMENT, "need >= 1 camera");
    if (!out) return fail(PF_ERR_INVALID_ARGUMENT, "out is NULL");
    for (int v = 0; v < V; ++v) {
        int rc = check_camera(cams[v]);
        if (rc) return rc;
        if (cams[v].width != cams[0].width || cams[v].height != cams[0].height)
            return fail(PF_ERR_INVALID_ARGUMENT, "all views of one call must share width/height");
    }
    DeviceGuard g(s->device);
    cudaStream_t st = (cudaStream_t)stream;
    const bool stat = (s->flags & PF_STATIC_SCENE) != 0;
    if (!stat || !s->edges_built) {
        PF_CUDA(pf::launch_edge_records(s, st));
        s->edges_built = true;
    }
    if (!s->bvh) {
        s->bvh = new (std::nothrow) pf::BallBVH();
        if (!s->bvh) return fail(PF_ERR_OUT_OF_MEMORY, "host allocation failed");
    }
    if (!stat || !s->bvh_built) {
        PF_CUDA(pf::build_ball_bvh(s, *s->bvh, s->ds.N, s->ds.sites, s->ds.radii, st));
        PF_CUDA(pf::pack_trace_nodes(s, *s->bvh, s->trace_nodes, st));
        s->bvh_built = true;
    }
    PF_CUDA(s->trace_stats.reserve(8 * 8));
    unsigned long long *dst = s->trace_stats.as<unsigned long long>();
    if (stats) PF_CUDA(cudaMemsetAsync(dst, 0, 8 * 5, st));
    const size_t npix = (size_t)cams[0].width * cams[0].height;
    for (int v = 0; v < V; ++v)
        PF_CUDA(pf::launch_trace(s, *s->bvh, cam_params(cams[v]), out + 4 * npix * (size_t)v,
                                 stats ? dst : nullptr, st));
    if (stats) {
        unsigned long long h[5];
        PF_CUDA(cudaMemcpyAsync(h, dst, sizeof(h), cudaMemcpyDeviceToHost, st));
        PF_CUDA(cudaStreamSynchronize(st));
        for (int k = 0; k < 5; ++k) stats[k] = (int64_t)h[k];
    }
    return PF_OK;
}

int pf_debug_binning(pf_scene *s, const pf_camera *cam, int32_t *rect, int32_t *count,
                     uint32_t *keybits, uint64_t *keys, uint32_t *vals, uint32_t *ranges,
                     int64_t *num_pairs, pf_stream_t stream)
{
    if (!s || !cam || !num_pairs) return fail(PF_ERR_INVALID_ARGUMENT, "NULL argument");
    int rc = check_camera(*cam);
    if (rc) return rc;
    DeviceGuard g(s->device);
    cudaStream_t st = (cudaStream_t)stream;
    pf::ViewState &vs = s->debug_view;
    s->fwd_views = 0;   // the debug pass reuses the call's sorted-pair arrays
    vs.cam = cam_params(*cam);
    rc = bin_views_of(s, &vs, 1, st);
    if (rc) return rc;
    const int64_t P = vs.P;
    *num_pairs = P;
    const size_t N = (size_t)s->ds.N;
    if (rect) PF_CUDA(cudaMemcpyAsync(rect, vs.rect.ptr, 16 * N, cudaMemcpyDeviceToDevice, st));
    if (count) PF_CUDA(cudaMemcpyAsync(count, vs.count.ptr, 4 * N, cudaMemcpyDeviceToDevice, st));
    if (keybits) PF_CUDA(cudaMemcpyAsync(keybits, vs.keybits.ptr, 4 * N, cudaMemcpyDeviceToDevice, st));
    if (keys) {
        uint32_t *ks = nullptr;
        rc = emit_sort_ranges(s, &vs, 1, st, &ks);
        if (rc) return rc;
        if (P > 0) {
            // the sort's keys hold the tile only: export the full (tile << 32 | keybits)
            PF_CUDA(pf::launch_full_keys(s, ks, vs.vals_p, vs.keybits.as<uint32_t>(), P,
                                         tile_bits(vs.cam.tiles_x * vs.cam.tiles_y), keys, st));
            if (vals) PF_CUDA(cudaMemcpyAsync(vals, vs.vals_p, 4 * (size_t)P, cudaMemcpyDeviceToDevice, st));
        }
        if (ranges)
            PF_CUDA(cudaMemcpyAsync(ranges, vs.ranges_p,
                                    sizeof(uint2) * (size_t)vs.cam.tiles_x * vs.cam.tiles_y,
                                    cudaMemcpyDeviceToDevice, st));
    }
    PF_CUDA(cudaStreamSynchronize(st));
    return PF_OK;
}

int pf_debug_counters(pf_scene *s, const pf_camera *cam, int64_t *counters, pf_stream_t stream)
{
    if (!s || !cam || !counters) return fail(PF_ERR_INVALID_ARGUMENT, "NULL argument");
    int rc = check_camera(*cam);
    if (rc) return rc;
    DeviceGuard g(s->device);
    cudaStream_t st = (cudaStream_t)stream;
    if (!(s->flags & PF_STATIC_SCENE) || !s->edges_built) {
        PF_CUDA(pf::launch_edge_records(s, st));
        s->edges_built = true;
    }
    pf::ViewState &vs = s->debug_view;
    s->fwd_views = 0;   // the debug pass reuses the call's sorted-pair arrays
    vs.cam = cam_params(*cam);
    rc = bin_views_of(s, &vs, 1, st);
    if (rc) return rc;
    uint32_t *ks;
    rc = emit_sort_ranges(s, &vs, 1, st, &ks);
    if (rc) return rc;
    PF_CUDA(cudaMemsetAsync(counters, 0, 32 * (size_t)cam->width * cam->height, st));
    s->host_args.assign(1, view_args(vs, nullptr, nullptr, false));
    const pf::ViewArgs *dargs = nullptr;
    rc = upload_view_args(s, s->host_args.data(), 1, 0, st, &dargs);
    if (rc) return rc;
    PF_CUDA(pf::launch_forward(s, &vs, 1, dargs, counters, false, nullptr, nullptr, st));
    PF_CUDA(cudaStreamSynchronize(st));
    return PF_OK;
}

int64_t pf_launch_count(const pf_scene *s) { return s ? s->launches : -1; }

int pf_set_profiling(pf_scene *s, int enable)
{
    if (!s) return fail(PF_ERR_INVALID_ARGUMENT, "NULL handle");
    s->profiling = enable != 0;
    return PF_OK;
}

int pf_stage_times(pf_scene *s, double *ms, int64_t *launches)
{
    if (!s || !ms) return fail(PF_ERR_INVALID_ARGUMENT, "NULL argument");
    DeviceGuard g(s->device);
    for (int k = 0; k < PF_NUM_STAGES; ++k) {
        ms[k] = 0.0;
        if (launches) launches[k] = 0;
    }
    for (auto &e : s->events) {
        PF_CUDA(cudaEventSynchronize(e.b));
        float t = 0.0f;
        PF_CUDA(cudaEventElapsedTime(&t, e.a, e.b));
        if (e.stage >= 0 && e.stage < PF_NUM_STAGES) {
            ms[e.stage] += t;
            if (launches) launches[e.stage] += e.launches;
        }
        s->event_pool.push_back(e.a);
        s->event_pool.push_back(e.b);
    }
    s->events.clear();
    return PF_OK;
}

int pf_last_pair_counts(const pf_scene *s, int64_t *pairs, int32_t V)
{
    if (!s || !pairs) return fail(PF_ERR_INVALID_ARGUMENT, "NULL argument");
    for (int v = 0; v < V; ++v) pairs[v] = v < (int)s->views.size() ? s->views[v].P : 0;
    return PF_OK;
}

}  // extern "C"
