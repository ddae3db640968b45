// pf_raster.cu -- K6 forward blend, K7 backward replay, K8 gradient unpack.
//
// One CTA per 16x16 tile (256 threads); warp w covers an 8x4 pixel block and
// walks the tile's sorted cell list independently (no CTA barriers), 32
// entries at a time: lane-parallel fp64 cull of the entries against the warp's
// ray cone + staging of the survivors with the warp-centred ray frame
// (SURVEY C18), then all 32 lanes (pixels) in lockstep on each survivor:
//   sphere test (a8) -> __any_sync cull -> half-space clipping against the
//   cell's neighbour planes (a9, division free, branch free) -> front-to-back
//   compositing (a10) -> warp vote early termination.
// The backward (K7) replays the identical walk front to back (bit-identical
// intervals and transmittances, same inlined math with explicit IEEE
// intrinsics), recovers S_k = out_rgb - C_k from the saved final colour, and
// scatters gradients: own-cell terms warp-reduced by shuffles then one float4
// atomic per warp, neighbour terms as float4 atomics.
#include <cuda_runtime.h>
#include <math.h>
#include <stdlib.h>

#include "pf_internal.cuh"
#include "pf_pixel.cuh"

namespace pf {


// ------------------------------------------------------------------------
// K6 forward
// ------------------------------------------------------------------------
#ifndef PF_K6_MINB
#define PF_K6_MINB 4
#endif
#ifndef PF_K6I_MINB   // K6 without records (inference, counting): 5 CTAs/SM measured faster
#define PF_K6I_MINB 5
#endif
#ifndef PF_K6_CULL_MIN_REC   // recording K6: cells with fewer list planes are clipped by
#define PF_K6_CULL_MIN_REC 6u  // all of them (the cull costs more than it saves there;
#endif                         // measured: 6 best of {0, 6, 9, 12}; inference K6: always cull)
#ifndef PF_K6_PCULL   // warp-level plane cull in K6 (cull_planes)
#define PF_K6_PCULL 1
#endif
#ifndef PF_K7_MINB
#define PF_K7_MINB 4
#endif
#ifndef PF_K7_DIRECT_MAX   // up to this many segment lanes: per-lane atomics, no warp reduction
#define PF_K7_DIRECT_MAX 10
#endif
#ifndef PF_K7_NBR_PREFETCH   // K7: L1 prefetch of a binding plane's neighbour id
#define PF_K7_NBR_PREFETCH 1
#endif
#ifndef PF_K7_PREFETCH   // K7: L2 prefetch of the next chunk's K6 records
#define PF_K7_PREFETCH 1
#endif
#ifndef PF_K7_AGG   // K7: neighbour REDs aggregated over lanes with the same j (match_any);
                    // measured 9.32 -> 14.09 ms per 8 views (train8_1m): off
#define PF_K7_AGG 0
#endif
#ifndef PF_K7_GROUP   // K7: up to this many consecutive disjoint-mask records per pass
#define PF_K7_GROUP 4
#endif
constexpr int kFuseTiles = 4096;   // views with fewer tiles: one fused K6 / K7 launch
#ifndef PF_K7D_GROUP   // detail K7: records per pass (per-record column reductions inside)
#define PF_K7D_GROUP 4
#endif
#ifndef PF_K7D_MINB
#define PF_K7D_MINB 2
#endif
#ifndef PF_K6D_MINB
#define PF_K6D_MINB 3
#endif
// kWide: the non-recording launch for wide-cone (fisheye) views, at 4 CTAs/SM
// (measured: 5 CTAs/SM is faster for pinhole views, slower for fisheye ones)
// kFused: all views of the call in one launch, this CTA's ViewArgs read from the
// device array into shared memory (small views: no per-view launch tails); else
// one launch per view with its ViewArgs by value (constant-bank operands; measured
// faster for 1080p views, whose launches are ~14 waves long)
// detail K6: the chart's soft-Voronoi weights spread over the warp (detail_plane_warp).
// Bit-identical, but measured slower (nerfsynth200k+detail8 K6 15.8 -> 20.4 ms): a hit
// cell holds ~18 of the warp's 32 rays, so the lockstep chart is half-used already and
// the spread version needs ~5 rounds of shuffles per cell. Off.
#ifndef PF_K6D_WARPSV
#define PF_K6D_WARPSV 0
#endif
#ifndef PF_K6D_QUEUE   // detail K6: segment colours evaluated 32 at a time (ColQueue)
#define PF_K6D_QUEUE 1
#endif
// Detail K6: the colour of a composited segment (Eq. svrad: soft-Voronoi weights at
// the displaced-face hit and the 8 x 8 x 3 SV blend) does not change the
// transmittance, so it need not be evaluated in the cell-by-cell lockstep, where a
// cell holds a few of the warp's 32 rays.  The warp queues (chart parameter, cell,
// weight T_k alpha_k) per segment and evaluates 32 queued colours at once, one per
// lane; each pixel then adds its own entries in queue (= list) order with the same
// fmaf as composite_step, so the image is bit-identical to the in-line evaluation.
struct ColQueue {
    double t[64];                // Q + t d: the displaced-face hit (or the parallel entry)
    uint32_t cell[64], slot[64]; // slot: the K6 -> K7 colour slot (kNoCol: none)
    float w[64], delta[64];      // T_k alpha_k, the clamped displacement
    float cr[32], cg[32], cb[32];
    uint8_t lane[64];            // the segment's pixel (lane of the warp)
};

template <bool kCount, bool kRecord, bool kDipole, int kDetail, bool kWide = false,
          bool kFused = false>
__global__ void __launch_bounds__(256, kDetail ? PF_K6D_MINB
                                               : (kRecord || kWide ? PF_K6_MINB : PF_K6I_MINB))
k6_forward(DeviceScene ds, const ViewArgs one, const ViewArgs *__restrict__ va, int ntiles,
           long long *__restrict__ counters, float *__restrict__ st_contrib,
           float *__restrict__ st_normal, int cull_on)
{
    __shared__ ViewArgs VAs[kFused ? 1 : 1];
    if (kFused) load_view_args(va, ntiles, VAs[0]);
    const ViewArgs &VA = kFused ? VAs[0] : one;
    const CamParams &cam = VA.cam;
    const uint2 *__restrict__ ranges = VA.ranges;
    const uint32_t *__restrict__ vals = VA.vals;
    float4 *__restrict__ out = VA.out;
    float4 *__restrict__ saved = VA.saved;
    const uint32_t *__restrict__ chunk_off = VA.chunk_off;
    uint2 *__restrict__ desc = VA.desc;
    uint32_t *__restrict__ wdone = VA.wdone;
    uint32_t *__restrict__ rec = VA.rec;
    uint32_t *__restrict__ rec_used = VA.rec_used;
    const uint32_t rec_cap = VA.rec_cap;
    __shared__ WarpStage WS[kWarps];
    __shared__ PixelRays PR;
    __shared__ WarpCtx WC[kWarps];
    __shared__ WarpRec WR[kRecord ? kWarps : 1];
    __shared__ float4 WN[kDipole ? kWarps * 32 : 1];
    // warp plane cull (cull_planes); the counting build evaluates every list plane
    // so its X_p stays the SURVEY 8(d) work count
    constexpr bool kCull = PF_K6_PCULL && !kCount;
    extern __shared__ PlaneBuf PB[];   // kWarps entries when kCull (dynamic: static smem is full)
    const int tile = (int)VA.order[kFused ? blockIdx.x % ntiles : blockIdx.x], lane = threadIdx.x & 31,
              warp = threadIdx.x >> 5;
    WarpStage &S = WS[warp];
    if (lane == 0) S.nrm = kDipole ? WN + warp * 32 : nullptr;
    WarpCtx &W = WC[warp];
    WarpRec &Rb = WR[kRecord ? warp : 0];
    PixelSetup P;
    setup_pixel(cam, tile, P, PR, W);
    const uint2 rg = ranges[tile];
    float T = 1.0f, Cr = 0.0f, Cg = 0.0f, Cb = 0.0f;
    bool done = !P.valid;
    float om[8];
    if (kDetail) sv_axis_weights(ds, P.R, om);
    constexpr bool kQueue = kDetail && PF_K6D_QUEUE;
    // the queue follows the plane-cull buffers in dynamic shared memory
    ColQueue &Q = reinterpret_cast<ColQueue *>(PB + (kCull ? kWarps : 0))[warp];
    int qn = 0;                  // queued entries (warp-uniform)
    unsigned long long qmine = 0;   // this lane's entries
    auto flush = [&](int n) {
        __syncwarp();
        const int pl = lane < n ? (int)Q.lane[lane] : lane;
        float omq[8];
#pragma unroll
        for (int a = 0; a < 8; ++a) omq[a] = __shfl_sync(0xffffffffu, om[a], pl);
        if (lane < n) {
            const uint32_t cell = Q.cell[lane];
            const int ti = (threadIdx.x & ~31) + pl;
            const double dq[3] = {PR.dx[ti], PR.dy[ti], PR.dz[ti]};
            double cq[3];
            cell_c(ds, cam, cell, cq);
            float cr, cg, cb;
            detail_color<kDetail>(ds, cell, dq, cq, Q.t[lane], omq, cr, cg, cb);
            Q.cr[lane] = cr;
            Q.cg[lane] = cg;
            Q.cb[lane] = cb;
            if (kRecord && Q.slot[lane] != kNoCol)
                VA.col[Q.slot[lane]] = make_float4(cr, cg, cb, Q.delta[lane]);
        }
        __syncwarp();
        const unsigned mine = (unsigned)qmine & (n == 32 ? 0xffffffffu : ((1u << n) - 1u));
        for (unsigned mm = mine; mm; mm &= mm - 1) {
            const int p = __ffs(mm) - 1;
            const float w = Q.w[p];
            Cr = fmaf(w, Q.cr[p], Cr);
            Cg = fmaf(w, Q.cg[p], Cg);
            Cb = fmaf(w, Q.cb[p], Cb);
        }
        const int rest = qn - n;   // entries n.. move to the front (n = 32 > rest)
        if (lane < rest) {
            Q.t[lane] = Q.t[n + lane];
            Q.cell[lane] = Q.cell[n + lane];
            Q.slot[lane] = Q.slot[n + lane];
            Q.w[lane] = Q.w[n + lane];
            Q.delta[lane] = Q.delta[n + lane];
            Q.lane[lane] = Q.lane[n + lane];
        }
        qmine = n == 32 ? (qmine >> 32) : 0ull;
        qn = rest;
        __syncwarp();
    };
    long long xs = 0, xh = 0, xp = 0, xc = 0;
    uint32_t chunks = 0, nseg = 0;   // nseg: composited segments (detail: K7D item count)
    uint32_t cnext = 0, cend = 0;    // detail: the warp's block of colour slots
    for (uint32_t base = rg.x; base < rg.y; base += 32, ++chunks) {
        if (__all_sync(0xffffffffu, done)) break;
        unsigned m = stage_chunk<kDipole, kCull>(S, ds, cam, vals, base + lane, rg.y, W, lane);
        int nrec = 0;
        while (m) {
            const int j = __ffs(m) - 1;
            m &= m - 1;
            Seg g;
            bool hit = false;
            if (!done) hit = sphere_hit(P.R, S, j, g, ds, cam, PR);
            if (!__any_sync(0xffffffffu, hit)) continue;
            if (kCount && hit) {
                ++xh;
                xp += S.deg[j];
            }
            int kept = 0;
            const bool culled = kCull && cull_on && S.deg[j] <= 32u &&
                                S.deg[j] >= (kRecord ? PF_K6_CULL_MIN_REC : 0u);
            if (culled) {
                kept = cull_planes(S, j, W, ds.edges, PB[warp], lane);
                if (kept < 0) continue;   // the warp's beam misses cell i: every interval is empty
            }
            float4 dpl = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
            DetailGeo G;
            double dd[3], dc[3];
            if (kDetail) {
                // neighbour planes first; the displaced face (its chart evaluation is
                // the expensive part) only where the interval is still non-empty
                if (culled)
                    clip_interval_kept<kRecord, false>(P.R, PB[warp], kept, g, hit, dpl);
                else
                    clip_interval<kRecord, false>(P.R, ds.edges, S.eb[j], S.deg[j], g, hit, dpl);
                const bool pre = g.dt > 0.0f;
                if (__any_sync(0xffffffffu, pre)) {
                    if (PF_K6D_WARPSV) {   // the chart's soft-Voronoi spread over the warp
                        dd[0] = PR.dx[threadIdx.x]; dd[1] = PR.dy[threadIdx.x]; dd[2] = PR.dz[threadIdx.x];
                        cell_c(ds, cam, S.cell[j], dc);
                        const float4 f = detail_plane_warp<kDetail>(ds, S.cell[j], pre, dd, dc, S.r[j], G, lane);
                        if (pre) dpl = f;
                    } else if (pre) {
                        dd[0] = PR.dx[threadIdx.x]; dd[1] = PR.dy[threadIdx.x]; dd[2] = PR.dz[threadIdx.x];
                        cell_c(ds, cam, S.cell[j], dc);
                        dpl = detail_plane<kDetail>(ds, S.cell[j], dd, dc, S.r[j], G);
                    }
                    clip_plane<kRecord>(P.R, dpl, kEndDipole, g);
                    const float dt = __fsub_rn(g.hi, g.lo);
                    g.dt = (pre && dt > 0.0f) ? dt : 0.0f;
                }
            } else {
                if (kDipole) dpl = S.nrm[j];
                if (culled)
                    clip_interval_kept<kRecord, kDipole>(P.R, PB[warp], kept, g, hit, dpl);
                else
                    clip_interval<kRecord, kDipole>(P.R, ds.edges, S.eb[j], S.deg[j], g, hit, dpl);
            }
            const bool seg = g.dt > 0.0f;
            float4 *colp = nullptr;   // detail: this lane's colour slot (K7 reads it back)
            if (kRecord) {
                const unsigned sm = __ballot_sync(0xffffffffu, seg);
                if (sm) {
                    const uint32_t c = seg ? (end_code<kDipole>(g.lo_q) | (end_code<kDipole>(g.hi_q) << 8)) : 0u;
                    reinterpret_cast<uint16_t *>(Rb.w + nrec * kRecWords + 2)[lane] = (uint16_t)c;
                    uint32_t cslot = kNoCol;
                    if (kDetail && VA.col) {
                        // colour slots of the record's segments, contiguous, from the
                        // warp's current block of kColBlock slots (one atomic per block,
                        // not per record: the counter is shared by the whole view)
                        const uint32_t n = (uint32_t)__popc(sm);
                        if (cnext + n > cend) {
                            uint32_t b = 0;
                            if (lane == 0) b = atomicAdd(VA.col_used, kColBlock);
                            cnext = __shfl_sync(0xffffffffu, b, 0);
                            cend = cnext + kColBlock;
                        }
                        cslot = cnext;
                        cnext += n;
                        if (cslot >= kNoCol || cslot + n > VA.col_cap) cslot = kNoCol;
                        if (seg && cslot != kNoCol)
                            colp = VA.col + cslot + __popc(sm & ((1u << lane) - 1u));
                    }
                    if (lane == 0) {
                        Rb.w[nrec * kRecWords] = sm;
                        // plain scenes: the cell id itself (K7 skips the list gather);
                        // detail scenes: the chunk slot and the first colour slot
                        Rb.w[nrec * kRecWords + 1] = kDetail ? ((uint32_t)j | (cslot << 5)) : S.cell[j];
                    }
                    ++nrec;
                    nseg += __popc(sm);
                }
            }
            float wk = 0.0f;
            if (seg) {
                float alpha;
                const float Tk = T;
                float cr = S.cr[j], cg = S.cg[j], cb = S.cb[j];
                if (kQueue) {
                    // composite_step without the colour (it is added at the flush)
                    const float ex = __expf(-__fmul_rn(S.sig[j], g.dt));
                    alpha = __fsub_rn(1.0f, ex);
                    T = __fmul_rn(T, ex);
                } else {
                    if (kDetail) {
                        detail_color<kDetail>(ds, S.cell[j], dd, dc,
                                     G.parallel ? (double)__fadd_rn(g.tc, g.lo) : G.ts, om, cr, cg, cb);
                        if (kRecord && colp) *colp = make_float4(cr, cg, cb, G.delta);
                    }
                    composite_step(S.sig[j], g.dt, cr, cg, cb, T, Cr, Cg, Cb, alpha);
                }
                wk = __fmul_rn(Tk, alpha);
                if (kCount) ++xc;
                if (T < kTStop) {
                    done = true;
                    if (kCount) xs = (long long)(base + j - rg.x) + 1;
                }
            }
            if (kQueue) {
                const unsigned pm = __ballot_sync(0xffffffffu, seg);
                if (pm) {
                    if (seg) {
                        const int pos = qn + __popc(pm & ((1u << lane) - 1u));
                        Q.t[pos] = G.parallel ? (double)__fadd_rn(g.tc, g.lo) : G.ts;
                        Q.cell[pos] = S.cell[j];
                        Q.slot[pos] = (kRecord && colp) ? (uint32_t)(colp - VA.col) : kNoCol;
                        Q.w[pos] = wk;
                        Q.delta[pos] = G.delta;
                        Q.lane[pos] = (uint8_t)lane;
                        qmine |= 1ull << pos;
                    }
                    qn += __popc(pm);
                    if (qn >= 32) flush(32);
                }
            }
            if (st_contrib && __any_sync(0xffffffffu, seg)) {
                // NEXT-1 by-products: sum T_k alpha_k (pruning / L_sparse) and
                // sum T_k alpha_k max(n.d, 0)^2 (L_normal), warp-reduced per cell
                float wn = 0.0f;
                if (kDipole && seg) {
                    const float4 Nn = S.nrm[j];
                    const float nd = fmaxf(fmaf(P.R.dx, Nn.x, fmaf(P.R.dy, Nn.y, __fmul_rn(P.R.dz, Nn.z))), 0.0f);
                    wn = wk * nd * nd;
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    wk += __shfl_xor_sync(0xffffffffu, wk, o);
                    if (kDipole) wn += __shfl_xor_sync(0xffffffffu, wn, o);
                }
                if (lane == 0) {
                    atomicAdd(st_contrib + S.cell[j], wk);
                    if (kDipole && st_normal) atomicAdd(st_normal + S.cell[j], wn);
                }
            }
            if (__all_sync(0xffffffffu, done)) break;
        }
        if (kRecord) {
            __syncwarp();
            uint2 d = make_uint2(0u, 0u);
            if (nrec) {
                uint32_t b0 = 0;
                if (lane == 0) b0 = atomicAdd(rec_used, (uint32_t)nrec);
                b0 = __shfl_sync(0xffffffffu, b0, 0);
                if ((uint64_t)b0 + nrec <= rec_cap) {
                    uint32_t *dst = rec + (size_t)b0 * kRecWords;
                    for (int w = lane; w < nrec * kRecWords; w += 32) dst[w] = Rb.w[w];
                    d = make_uint2(b0, (uint32_t)nrec);
                } else {
                    d = make_uint2(0u, kOverflow);
                }
            }
            if (lane == 0) desc[(size_t)(chunk_off[tile] + chunks) * kWarps + warp] = d;
            __syncwarp();
        }
        __syncwarp();
    }
    if (kQueue && qn) flush(qn);
    if (kRecord && lane == 0) {
        wdone[(size_t)tile * kWarps + warp] = chunks;
        if (kDetail && nseg) atomicAdd(VA.seg_used, nseg);
    }
    if (P.in_image) {   // pixels without a ray keep T = 1: the background
        const float4 o = make_float4(fmaf(T, ds.bg[0], Cr), fmaf(T, ds.bg[1], Cg),
                                     fmaf(T, ds.bg[2], Cb), T);
        const size_t pix = (size_t)P.y * cam.W + P.x;
        if (out) out[pix] = o;
        if (saved) saved[pix] = o;
        if (kCount) {
            if (!done) xs = (long long)(rg.y - rg.x);
            counters[4 * pix + 0] = xs;
            counters[4 * pix + 1] = xh;
            counters[4 * pix + 2] = xp;
            counters[4 * pix + 3] = xc;
        }
    }
}

#ifndef PF_VIEW_STREAMS   // per-view K6 / K7 launches on two alternating streams
#define PF_VIEW_STREAMS 1
#endif
// The stream of view v's per-view launch: even views on the call's stream, odd ones on
// the handle's second stream (forked from / joined back into the call's stream by
// view_streams_begin / _end), so a view's last wave overlaps the next view's first.
static bool view_streams_begin(pf_scene *s, cudaStream_t st, int V)
{
    if (!PF_VIEW_STREAMS || V < 2) return false;
    if (!s->pair) {
        if (cudaStreamCreateWithFlags(&s->pair, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&s->pair_fork, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&s->pair_join, cudaEventDisableTiming) != cudaSuccess) {
            cudaGetLastError();
            if (s->pair) cudaStreamDestroy(s->pair);
            s->pair = nullptr;
            return false;
        }
    }
    cudaEventRecord(s->pair_fork, st);
    cudaStreamWaitEvent(s->pair, s->pair_fork, 0);
    return true;
}

static void view_streams_end(pf_scene *s, cudaStream_t st, bool on)
{
    if (!on) return;
    cudaEventRecord(s->pair_join, s->pair);
    cudaStreamWaitEvent(st, s->pair_join, 0);
}

template <bool kDipole, int kDetail>
static int launch_forward_t(pf_scene *s, const ViewState *views, int V, const ViewArgs *args,
                            int64_t *counters, bool record, float *stc, float *stn,
                            cudaStream_t st)
{
    const int T = views[0].cam.tiles_x * views[0].cam.tiles_y;
    // the plane-cull buffers are dynamic shared memory (static + dynamic may pass 48 KB)
    // (+ the detail colour queues, ColQueue, after them)
    const size_t dynq = (kDetail && PF_K6D_QUEUE) ? kWarps * sizeof(ColQueue) : 0;
    const size_t dyn = (PF_K6_PCULL ? kWarps * sizeof(PlaneBuf) : 0) + dynq;
    if (s->cull_on < 0) {   // debug knob, read once per handle: 0 clips by every list plane
        const char *e = getenv("PF_PLANE_CULL");
        s->cull_on = (e && e[0] == '0') ? 0 : 1;
    }
    bool wide = false;
    for (int v = 0; v < V; ++v) wide = wide || views[v].cam.model == PF_FISHEYE;
    if (dyn && !s->attrs_k6) {   // once per handle (the attribute is per device)
        cudaFuncSetAttribute(k6_forward<true, false, kDipole, kDetail>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
        cudaFuncSetAttribute(k6_forward<true, false, kDipole, kDetail, false, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
        cudaFuncSetAttribute(k6_forward<false, true, kDipole, kDetail>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
        cudaFuncSetAttribute(k6_forward<false, false, kDipole, kDetail>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
        cudaFuncSetAttribute(k6_forward<false, true, kDipole, kDetail, false, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
        cudaFuncSetAttribute(k6_forward<false, false, kDipole, kDetail, false, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
        if constexpr (!kDetail) {
            cudaFuncSetAttribute(k6_forward<false, false, kDipole, kDetail, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
            cudaFuncSetAttribute(k6_forward<false, false, kDipole, kDetail, true, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
        }
    }
    s->attrs_k6 = true;
    // fused for small views (few waves per launch), per view otherwise (PF_K6_PER_VIEW=1
    // forces per-view launches, =0 the fused one; A/B knob)
    if (s->k6_per_view < 0) {
        const char *e = getenv("PF_K6_PER_VIEW");
        s->k6_per_view = e ? (e[0] == '1' ? 1 : 0) : 2;
    }
    const bool fused = s->k6_per_view == 0 || (s->k6_per_view == 2 && T < kFuseTiles);
    const ViewArgs *h = s->host_args.data();
    if (fused) {
        const unsigned grid = (unsigned)(T * V);
        if (counters)
            k6_forward<true, false, kDipole, kDetail, false, true><<<grid, 256, dynq, st>>>(
                s->ds, h[0], args, T, (long long *)counters, nullptr, nullptr, 0);
        else if (record)
            k6_forward<false, true, kDipole, kDetail, false, true><<<grid, 256, dyn, st>>>(
                s->ds, h[0], args, T, nullptr, stc, stn, s->cull_on);
        else {
            auto kern = k6_forward<false, false, kDipole, kDetail, false, true>;
            if constexpr (!kDetail)
                if (wide) kern = k6_forward<false, false, kDipole, kDetail, true, true>;
            kern<<<grid, 256, dyn, st>>>(s->ds, h[0], args, T, nullptr, stc, stn, s->cull_on);
        }
        return 1;
    }
    const bool two = !counters && view_streams_begin(s, st, V);
    for (int v = 0; v < V; ++v) {
        cudaStream_t sv = (two && (v & 1)) ? s->pair : st;
        if (counters)
            k6_forward<true, false, kDipole, kDetail><<<T, 256, dynq, sv>>>(
                s->ds, h[v], nullptr, T, (long long *)counters, nullptr, nullptr, 0);
        else if (record)
            k6_forward<false, true, kDipole, kDetail><<<T, 256, dyn, sv>>>(
                s->ds, h[v], nullptr, T, nullptr, stc, stn, s->cull_on);
        else {
            auto kern = k6_forward<false, false, kDipole, kDetail>;
            if constexpr (!kDetail)
                if (wide) kern = k6_forward<false, false, kDipole, kDetail, true>;
            kern<<<T, 256, dyn, sv>>>(s->ds, h[v], nullptr, T, nullptr, stc, stn, s->cull_on);
        }
    }
    view_streams_end(s, st, two);
    return V;
}

cudaError_t launch_forward(pf_scene *s, const ViewState *views, int V, const ViewArgs *args,
                           int64_t *counters, bool record, float *st_contrib, float *st_normal,
                           cudaStream_t st)
{
    cudaEvent_t ev;
    stage_begin(s, 6, st, &ev);
    int n;
    if (s->ds.K == 8)
        n = launch_forward_t<true, 8>(s, views, V, args, counters, record, st_contrib, st_normal, st);
    else if (s->ds.K)
        n = launch_forward_t<true, 1>(s, views, V, args, counters, record, st_contrib, st_normal, st);
    else if (s->ds.cellN)
        n = launch_forward_t<true, 0>(s, views, V, args, counters, record, st_contrib, st_normal, st);
    else
        n = launch_forward_t<false, 0>(s, views, V, args, counters, record, st_contrib, st_normal, st);
    s->launches += n;
    stage_end(s, 6, st, ev);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------
// K7 backward
// ------------------------------------------------------------------------
namespace {

// d t_end / d theta times  w = +-dL/ddt  for one interval end:
//   sphere end at t' = +-s:  dt/dp_i = (t' d - e)/t',  dt/dr = r/t'
//   plane end (i,j), a = d.n: dt/dp_i = (t' d - e)/a, dt/dp_j = (n - t' d + e)/a,
//                             dt/dw_i = 1/(2a), dt/dw_j = -1/(2a)
//   near end: 0
struct OwnGrad {
    float px, py, pz, w, r, nx, ny, nz;
};

// Accumulator layout: 12 floats per cell, acc[12 i + k]:
//   k = 0..3 (p.x, p.y, p.z, w)  4..7 (r, sigma, R, G)  8 (B)  9..11 dipole normal.
// With nj != nullptr the neighbour term is returned in (*nj, *nv) for a warp-aggregated
// scatter (red_nbr_agg) instead of being issued here.
template <bool kDipole, bool kDetail>
__device__ __forceinline__ void end_grad(const Ray &R, const Seg &g, int q, float tprime,
                                         float wgt, float rad, const float4 *__restrict__ edges,
                                         const int32_t *__restrict__ nbr, float *acc, OwnGrad &o,
                                         const float4 &dnrm, uint32_t eb, float &g_ts,
                                         int *nj = nullptr, float4 *nv = nullptr)
{
    if (q == kEndNear) return;
    if (kDetail && q == kEndDipole) {   // the displaced face: through the detail chain
        g_ts += wgt;
        return;
    }
    const float xpx = fmaf(tprime, R.dx, -g.ex), xpy = fmaf(tprime, R.dy, -g.ey),
                xpz = fmaf(tprime, R.dz, -g.ez);   // x* - p_i
    if (kDipole && q == kEndDipole) {
        // dipole face t* = (p - Q).n / (d.n): dt/dp_i = n/a, dt/dn_i = (p_i - x*)/a
        const float nx = dnrm.x, ny = dnrm.y, nz = dnrm.z;
        const float a = fmaf(R.dx, nx, fmaf(R.dy, ny, __fmul_rn(R.dz, nz)));
        const float f = __fdividef(wgt, a);
        o.px = fmaf(f, nx, o.px);
        o.py = fmaf(f, ny, o.py);
        o.pz = fmaf(f, nz, o.pz);
        o.nx = fmaf(-f, xpx, o.nx);
        o.ny = fmaf(-f, xpy, o.ny);
        o.nz = fmaf(-f, xpz, o.nz);
        return;
    }
    if (q == kEndSphere) {
        const float f = __fdividef(wgt, tprime);
        o.px = fmaf(f, xpx, o.px);
        o.py = fmaf(f, xpy, o.py);
        o.pz = fmaf(f, xpz, o.pz);
        o.r = fmaf(f, rad, o.r);
        return;
    }
    const uint32_t qe = eb + (uint32_t)q - 2u;   // global edge of the binding plane
    const float4 E = __ldg(edges + qe);
    const float a = fmaf(R.dx, E.x, fmaf(R.dy, E.y, __fmul_rn(R.dz, E.z)));
    const float f = __fdividef(wgt, a);
    o.px = fmaf(f, xpx, o.px);
    o.py = fmaf(f, xpy, o.py);
    o.pz = fmaf(f, xpz, o.pz);
    o.w = fmaf(0.5f, f, o.w);
    const int j = __ldg(nbr + qe);
    const float4 t = make_float4(f * (E.x - xpx), f * (E.y - xpy), f * (E.z - xpz), -0.5f * f);
    if (nj) {
        *nj = j;
        *nv = t;
        return;
    }
    atomicAdd(reinterpret_cast<float4 *>(acc + 12 * (size_t)j), t);
}

// Warp-aggregated neighbour scatter (every lane calls it; j < 0: nothing to add).
// Lanes with the same neighbour j (neighbouring pixels leaving cell i through the
// same face) are found by __match_any_sync; their float4 terms are summed by a
// log-step tree over each group's lanes (uniform shuffles) and the group's lowest
// lane issues ONE REDG.F32x4.  If no two lanes share a j the REDs go out directly.
__device__ __forceinline__ void red_nbr_agg(float *acc, int j, float4 v, int lane)
{
    const int key = j >= 0 ? j : -1 - lane;   // idle lanes: singleton groups
    const unsigned peers = __match_any_sync(0xffffffffu, key);
    const bool multi = __any_sync(0xffffffffu, __popc(peers) > 1);
    if (multi) {
        const unsigned below = peers & ((1u << lane) - 1u);
        unsigned up = peers & ~(below | (1u << lane));
        int rel = __popc(below);
        while (__any_sync(0xffffffffu, up != 0u)) {
            const int nxt = up ? __ffs(up) - 1 : lane;
            const float tx = __shfl_sync(0xffffffffu, v.x, nxt),
                        ty = __shfl_sync(0xffffffffu, v.y, nxt),
                        tz = __shfl_sync(0xffffffffu, v.z, nxt),
                        tw = __shfl_sync(0xffffffffu, v.w, nxt);
            const bool even = !(rel & 1);
            if (even && up) {
                v.x += tx;
                v.y += ty;
                v.z += tz;
                v.w += tw;
            }
            up &= __ballot_sync(0xffffffffu, even);
            rel >>= 1;
        }
        if (j >= 0 && below == 0u) atomicAdd(reinterpret_cast<float4 *>(acc + 12 * (size_t)j), v);
    } else if (j >= 0) {
        atomicAdd(reinterpret_cast<float4 *>(acc + 12 * (size_t)j), v);
    }
}

// Sum of 9 per-lane values over the warp by a transposing reduction (12 shuffles
// instead of 45): after it, the lane with (lane & 1) == 0 and a valid slot holds
// the warp total of one value and issues one atomic; 9 lanes, one instruction.
__device__ __forceinline__ void warp_reduce9_atomic(float v[10], float *acc_cell, int lane)
{
    const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4, b1 = lane & 2;
    float u[6];
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const float send = b4 ? v[k] : v[k + 5], keep = b4 ? v[k + 5] : v[k];
        u[k] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
    u[5] = 0.0f;
    float w[4];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const float send = b3 ? u[k] : u[k + 3], keep = b3 ? u[k + 3] : u[k];
        w[k] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
    w[3] = 0.0f;
    float x[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const float send = b2 ? w[k] : w[k + 2], keep = b2 ? w[k + 2] : w[k];
        x[k] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
    const float send = b1 ? x[0] : x[1], keep = b1 ? x[1] : x[0];
    float y = keep + __shfl_xor_sync(0xffffffffu, send, 2);
    y += __shfl_xor_sync(0xffffffffu, y, 1);
    const int j = (b3 ? 3 : 0) + (b2 ? 2 : 0) + (b1 ? 1 : 0);
    const int idx = (b4 ? 5 : 0) + j;
    const bool valid = !(lane & 1) && (b3 ? j <= 4 : j <= 2) && idx < 9;
    if (valid) atomicAdd(acc_cell + idx, y);
}

// Same for up to 16 values (slots padded to 16): 16 shuffles; lane (lane & 1) == 0
// ends with the total of value ((lane >> 1) & 15).
template <int K>
__device__ __forceinline__ void warp_reduce16_atomic(float v[16], float *acc_cell, int lane)
{
#pragma unroll
    for (int half = 8; half >= 1; half >>= 1) {
        const bool up = lane & (2 * half);   // lane bit log2(2*half): keeps the upper half
#pragma unroll
        for (int k = 0; k < half; ++k) {
            const float send = up ? v[k] : v[k + half], keep = up ? v[k + half] : v[k];
            v[k] = keep + __shfl_xor_sync(0xffffffffu, send, 2 * half);
        }
    }
    float y = v[0] + __shfl_xor_sync(0xffffffffu, v[0], 1);
    const int idx = (lane >> 1) & 15;
    if (!(lane & 1) && idx < K) atomicAdd(acc_cell + idx, y);
}

// value of one interval end from its recorded constraint code (see end_code)
template <bool kDipole>
__device__ __forceinline__ float coded_end(const Ray &R, const float4 *__restrict__ edges,
                                           const int32_t *__restrict__ nbr, uint32_t eb,
                                           uint32_t code, bool lo, const Seg &g, int &q,
                                           const float4 &dplane)
{
    if (code == 0u) {
        q = kEndSphere;
        return lo ? -g.s : g.s;
    }
    if (lo && code == 1u) {
        q = kEndNear;
        return __fsub_rn(R.tnear, g.tc);
    }
    float4 E;
    if (kDipole && code == 254u) {
        q = kEndDipole;
        E = dplane;
    } else {
        q = (int)code;                      // 2 + local plane index
        E = __ldg(edges + eb + code - 2u);
#if PF_K7_NBR_PREFETCH   // end_grad reads the neighbour id after the replay math
        asm volatile("prefetch.global.L1 [%0];" ::"l"(nbr + eb + code - 2u));
#endif
    }
    const float a = fmaf(R.dx, E.x, fmaf(R.dy, E.y, __fmul_rn(R.dz, E.z)));
    const float b = fmaf(E.x, g.ex, fmaf(E.y, g.ey, fmaf(E.z, g.ez, E.w)));
    return __fmul_rn(b, rcp_approx(a));
}

// Backward of one detail segment (NEXT-2), fused: radiance at the displaced-face
// hit (Eq. svrad; colour and c_k . G in one pass over the SV values), the
// compositing replay of the segment, the interval-end derivatives, then the
// chain of P:284-293 run backwards in the order of the oracle's
// detail_backward.  Every lane of the warp calls it (seg lanes carry values).
// dL/dv_{k,a,c} = sum over the warp's pixels of w'_k (om_a gC_c), an outer
// product: both factors go to a [32][33] smem tile and each lane forms 6 of the
// K*24 sums over the seg lanes (float2 atomics); dL/ds_k and dL/dd_k are
// column sums of the same tile refilled.
//
// The geometric part runs in fp64: at grazing incidence the chart point is far
// from the sites and moves radially with t*, the softmax gradient's radial
// components cancel (sum_k dL/drho_k = 0) and what is left is multiplied by
// |x - p| / |d.m| ~ 1/|d.m|^2; fp32 residuals of that cancellation would
// dominate the normal's gradient.  So the weights are renormalised in fp64
// (the zero sum then holds to 1e-16) and the unit vectors, adjoints and the
// frame terms are fp64 too.
struct DetailCtx {
    double d[3], c[3];   // the exact ray direction and p - Q
    DetailGeo G;
};

// unit vectors (q - s_k)/rho_k: fp64 (rsqrt + one Newton step, ~1e-14) or fp32
template <typename T>
__device__ __forceinline__ void sv_units(const float2 s[kMaxDetail], int K, double q0, double q1,
                                         T ux[kMaxDetail], T uy[kMaxDetail])
{
#pragma unroll
    for (int k = 0; k < kMaxDetail; ++k) {
        ux[k] = uy[k] = (T)0;
        if (k < K) {
            const float2 sk = s[k];
            const T dx = (T)(q0 - (double)sk.x), dy = (T)(q1 - (double)sk.y);
            const T r2 = dx * dx + dy * dy;
            if (r2 > (T)0) {
                T ri = (T)rsqrtf((float)r2);
                if (sizeof(T) == 8) ri = ri * ((T)1.5 - (T)0.5 * r2 * ri * ri);
                ux[k] = dx * ri;
                uy[k] = dy * ri;
            }
        }
    }
}

// one unit vector (q - s)/|q - s| (as sv_units for one site)
template <typename T>
__device__ __forceinline__ void sv_unit(const float2 sk, double q0, double q1, T &ux, T &uy)
{
    ux = uy = (T)0;
    const T dx = (T)(q0 - (double)sk.x), dy = (T)(q1 - (double)sk.y);
    const T r2 = dx * dx + dy * dy;
    if (r2 > (T)0) {
        T ri = (T)rsqrtf((float)r2);
        if (sizeof(T) == 8) ri = ri * ((T)1.5 - (T)0.5 * r2 * ri * ri);
        ux = dx * ri;
        uy = dy * ri;
    }
}

struct BwdPixel {
    float T, Cr, Cg, Cb;
    float4 fin, G;
    float GT_Tfin;
};

#ifdef PF_DETAIL_NOINLINE   // A/B knob (inlined measured 20% faster: no call-boundary spills)
#define PF_DETAIL_FN __noinline__
#else
#define PF_DETAIL_FN __forceinline__
#endif
// The reverse chain of P:284-293 for one detail segment (after the compositing
// replay gave wa = T_k alpha_k and g_ts = dL/dt_s of the displaced-face hit):
// writes the lane's row of the dL/dv outer-product tile (brow: w_k, om_a wa G_c)
// and of the site / displacement gradient tile (grow: dL/ds_k 2K, dL/dd_k K) and
// adds the own-cell normal / position / radius terms to o.
template <typename T, int KT>
__device__ __forceinline__ void detail_reverse(const DeviceScene &ds, uint32_t cell, const DetailCtx &X,
                                               double ys0, double ys1, double ys2, double qs0,
                                               double qs1, const float ws[kMaxDetail],
                                               const float dG[kMaxDetail], float wa, float g_ts,
                                               float rad, const float4 &Gp, const float *om,
                                               float *brow, float *grow, OwnGrad &o)
{
    const int K = KT == 8 ? 8 : ds.K;
    const float tau = ds.sv_tau;
    const double *F = ds.cellF + (size_t)kCellF * cell;
    const double m0 = __ldg(F), m1 = __ldg(F + 1), m2 = __ldg(F + 2);
    const double u0 = __ldg(F + 3), u1 = __ldg(F + 4), u2 = __ldg(F + 5);
    const double v0 = __ldg(F + 6), v1 = __ldg(F + 7), v2 = __ldg(F + 8);
    const double d0 = X.d[0], d1 = X.d[1], d2 = X.d[2];
    const float2 *uv = reinterpret_cast<const float2 *>(ds.duv) + (size_t)K * cell;
    // ---- reverse of Eq. svrad: dL/dc = wa G
#pragma unroll
    for (int k = 0; k < kMaxDetail; ++k) brow[k] = ws[k];
#pragma unroll
    for (int a = 0; a < 8; ++a) {
        const float oa = om[a] * wa;
        brow[8 + 3 * a] = oa * Gp.x;
        brow[9 + 3 * a] = oa * Gp.y;
        brow[10 + 3 * a] = oa * Gp.z;
    }
    const T tm0 = (T)m0, tm1 = (T)m1, tm2 = (T)m2, tu0 = (T)u0, tu1 = (T)u1, tu2 = (T)u2;
    const T tv0 = (T)v0, tv1 = (T)v1, tv2 = (T)v2, td0 = (T)d0, td1 = (T)d1, td2 = (T)d2;
    const T tA = (T)X.G.A, ttau = (T)tau;
    T wsum = 0, sw = 0;
#pragma unroll
    for (int k = 0; k < kMaxDetail; ++k) {
        wsum += (T)ws[k];
        sw += (T)ws[k] * (T)dG[k];
    }
    const T iwsum = (T)1 / wsum;
    sw *= iwsum;   // renormalised: sum_k w_k (dG_k - sw) = 0 to working-precision rounding
    T gq0 = 0, gq1 = 0;
    const T cq = -ttau * (T)wa * iwsum;
#pragma unroll
    for (int k = 0; k < kMaxDetail; ++k) {
        float gx = 0.0f, gy = 0.0f;
        if (k < K) {
            T ux, uy;
            sv_unit<T>(__ldg(uv + k), qs0, qs1, ux, uy);
            const T grho = cq * (T)ws[k] * ((T)dG[k] - sw);
            gq0 += grho * ux;
            gq1 += grho * uy;
            gx = -(float)(grho * ux);
            gy = -(float)(grho * uy);
        }
        grow[2 * k] = gx;
        grow[2 * k + 1] = gy;
        grow[16 + k] = 0.0f;
    }
    T gm0 = 0, gm1 = 0, gm2 = 0, gc0 = 0, gc1 = 0, gc2 = 0;
    T gu0 = 0, gu1 = 0, gu2 = 0, gv0 = 0, gv1 = 0, gv2 = 0;
    if (!X.G.parallel) {
        const T s0 = (T)ys0, s1 = (T)ys1, s2 = (T)ys2;
        // qs = (ys.u, ys.v)
        const T gy0 = gq0 * tu0 + gq1 * tv0, gy1 = gq0 * tu1 + gq1 * tv1,
                gy2 = gq0 * tu2 + gq1 * tv2;
        gu0 = gq0 * s0; gu1 = gq0 * s1; gu2 = gq0 * s2;
        gv0 = gq1 * s0; gv1 = gq1 * s1; gv2 = gq1 * s2;
        // ys = ts d - c
        const T gts = (T)g_ts + gy0 * td0 + gy1 * td1 + gy2 * td2;
        gc0 = -gy0; gc1 = -gy1; gc2 = -gy2;
        // ts = (c.m + delta) / (d.m)
        const T iA = (T)1 / tA;
        const T f = gts * iA;
        gc0 += f * tm0; gc1 += f * tm1; gc2 += f * tm2;
        gm0 = -f * s0; gm1 = -f * s1; gm2 = -f * s2;
        T gdr = 0;
        const float r = rad;
        if (X.G.dr > r) o.r += (float)f;            // delta = r
        else if (X.G.dr < -r) o.r -= (float)f;      // delta = -r
        else gdr = f;
        // Eq. svdisp at the base-face hit (the chart point in fp64 as in the forward)
        // detail_plane's explicit op sequence, so x_bar (and the unit vectors taken
        // there) is bit-identical to the forward's
        const double B = dot3d(X.c, m0, m1, m2);
        const double tb = __dmul_rn(B, __drcp_rn(X.G.A));
        const double y0 = __fma_rn(tb, d0, -X.c[0]), y1 = __fma_rn(tb, d1, -X.c[1]),
                     y2 = __fma_rn(tb, d2, -X.c[2]);
        const double qb0 = __fma_rn(y0, u0, __fma_rn(y1, u1, __dmul_rn(y2, u2)));
        const double qb1 = __fma_rn(y0, v0, __fma_rn(y1, v1, __dmul_rn(y2, v2)));
        const float *wb = X.G.w;   // detail_plane's weights at x_bar
        const float *dk = ds.ddisp + (size_t)K * cell;
        T dr = 0, bsum = 0;
#pragma unroll
        for (int k = 0; k < kMaxDetail; ++k) {
            bsum += (T)wb[k];
            if (k < K) dr += (T)wb[k] * (T)__ldg(dk + k);
        }
        const T ibsum = (T)1 / bsum;
        dr *= ibsum;
        T gb0 = 0, gb1 = 0;
#pragma unroll
        for (int k = 0; k < kMaxDetail; ++k) {
            if (k < K) {
                T ux, uy;
                sv_unit<T>(__ldg(uv + k), qb0, qb1, ux, uy);
                const T wk = (T)wb[k] * ibsum;
                grow[16 + k] = (float)(wk * gdr);
                const T grho = -ttau * wk * gdr * ((T)__ldg(dk + k) - dr);
                gb0 += grho * ux;
                gb1 += grho * uy;
                grow[2 * k] -= (float)(grho * ux);
                grow[2 * k + 1] -= (float)(grho * uy);
            }
        }
        const T b0 = (T)y0, b1 = (T)y1, b2 = (T)y2;
        const T hy0 = gb0 * tu0 + gb1 * tv0, hy1 = gb0 * tu1 + gb1 * tv1,
                hy2 = gb0 * tu2 + gb1 * tv2;
        gu0 += gb0 * b0; gu1 += gb0 * b1; gu2 += gb0 * b2;
        gv0 += gb1 * b0; gv1 += gb1 * b1; gv2 += gb1 * b2;
        const T f2 = (hy0 * td0 + hy1 * td1 + hy2 * td2) * iA;
        gc0 += f2 * tm0 - hy0; gc1 += f2 * tm1 - hy1; gc2 += f2 * tm2 - hy2;
        gm0 -= f2 * b0; gm1 -= f2 * b1; gm2 -= f2 * b2;
    }
    // frame: v = m x u, u = w/|w|, w = e_k x m, m = n/|n|
    gm0 += tu1 * gv2 - tu2 * gv1;           // u x gv
    gm1 += tu2 * gv0 - tu0 * gv2;
    gm2 += tu0 * gv1 - tu1 * gv0;
    gu0 += gv1 * tm2 - gv2 * tm1;           // gv x m
    gu1 += gv2 * tm0 - gv0 * tm2;
    gu2 += gv0 * tm1 - gv1 * tm0;
    const T iwl = (T)__ldg(F + 10), inn = (T)__ldg(F + 9);   // stored as reciprocals
    const int kax = (int)__ldg(F + 11);
    const T ug = tu0 * gu0 + tu1 * gu1 + tu2 * gu2;
    const T gw0 = (gu0 - tu0 * ug) * iwl, gw1 = (gu1 - tu1 * ug) * iwl,
            gw2 = (gu2 - tu2 * ug) * iwl;
    // + gw x e_k
    if (kax == 0) { gm1 += gw2; gm2 -= gw1; }
    else if (kax == 1) { gm0 -= gw2; gm2 += gw0; }
    else { gm0 += gw1; gm1 -= gw0; }
    const T mg = tm0 * gm0 + tm1 * gm1 + tm2 * gm2;
    o.nx += (float)((gm0 - tm0 * mg) * inn);
    o.ny += (float)((gm1 - tm1 * mg) * inn);
    o.nz += (float)((gm2 - tm2 * mg) * inn);
    o.px += (float)gc0;
    o.py += (float)gc1;
    o.pz += (float)gc2;
}

template <typename T, int KT>
__device__ PF_DETAIL_FN void detail_segment(const Ray &R, const Seg &g, bool seg,
                                            const WarpStage &S, int j, BwdPixel &px,
                                            const DeviceScene &ds, float *acc, int lane,
                                            const DetailCtx &X, const float *om, float (*buf)[33],
                                            float (*gbuf)[25], bool grouped)
{
    const int K = KT == 8 ? 8 : ds.K;   // K == 8 (the paper's setting) known at compile time
    const uint32_t cell = S.cell[j];
    const float tau = ds.sv_tau;
    OwnGrad o = {0, 0, 0, 0, 0, 0, 0, 0};
    float gs = 0.0f;
    // dL/ds_k (2K) and dL/dd_k (K) of this lane's segment go straight to its row of the
    // warp's gbuf tile (column sums below): no per-lane register arrays for them, and
    // the per-site unit vectors, weights and displacements are recomputed / re-read per
    // k instead of held in fp64 arrays (register pressure: 2 CTAs/SM)
    if (seg) {
        const double *F = ds.cellF + (size_t)kCellF * cell;
        const double m0 = __ldg(F), m1 = __ldg(F + 1), m2 = __ldg(F + 2);
        const double u0 = __ldg(F + 3), u1 = __ldg(F + 4), u2 = __ldg(F + 5);
        const double v0 = __ldg(F + 6), v1 = __ldg(F + 7), v2 = __ldg(F + 8);
        const double d0 = X.d[0], d1 = X.d[1], d2 = X.d[2];
        const float2 *uv = reinterpret_cast<const float2 *>(ds.duv) + (size_t)K * cell;
        // ---- forward: Eq. svrad at x (the interval entry for a parallel ray)
        const double tcol = X.G.parallel ? (double)__fadd_rn(g.tc, g.lo) : X.G.ts;
        // the chart point by detail_color's explicit op sequence (bit-identical weights)
        const double ys0 = __fma_rn(tcol, d0, -X.c[0]), ys1 = __fma_rn(tcol, d1, -X.c[1]),
                     ys2 = __fma_rn(tcol, d2, -X.c[2]);
        const double qs0 = __fma_rn(ys0, u0, __fma_rn(ys1, u1, __dmul_rn(ys2, u2)));
        const double qs1 = __fma_rn(ys0, v0, __fma_rn(ys1, v1, __dmul_rn(ys2, v2)));
        float ws[kMaxDetail], dG[kMaxDetail];
        float2 st[kMaxDetail];
        load_sites(uv, K, st);
        soft_voronoi(st, K, qs0, qs1, tau, ws);
        const float4 *sv = reinterpret_cast<const float4 *>(ds.dsv) + (size_t)6 * K * cell;
        float cr = 0.0f, cg = 0.0f, cb = 0.0f;
#pragma unroll
        for (int k = 0; k < kMaxDetail; ++k) {
            dG[k] = 0.0f;
            if (k < K) {
                float v[24];
#pragma unroll
                for (int q = 0; q < 6; ++q) {
                    const float4 x = __ldg(sv + 6 * k + q);
                    v[4 * q] = x.x; v[4 * q + 1] = x.y; v[4 * q + 2] = x.z; v[4 * q + 3] = x.w;
                }
                float kr = 0.0f, kg = 0.0f, kb = 0.0f;
#pragma unroll
                for (int a = 0; a < 8; ++a) {
                    kr = fmaf(om[a], v[3 * a], kr);
                    kg = fmaf(om[a], v[3 * a + 1], kg);
                    kb = fmaf(om[a], v[3 * a + 2], kb);
                }
                cr = fmaf(ws[k], kr, cr);
                cg = fmaf(ws[k], kg, cg);
                cb = fmaf(ws[k], kb, cb);
                dG[k] = fmaf(kr, px.G.x, fmaf(kg, px.G.y, kb * px.G.z));   // c_k . G
            }
        }
        // ---- compositing replay (as segment_backward)
        const float sig = S.sig[j];
        const float Tk = px.T;
        float alpha;
        composite_step(sig, g.dt, cr, cg, cb, px.T, px.Cr, px.Cg, px.Cb, alpha);
        const float Sr = __fsub_rn(px.fin.x, px.Cr), Sg = __fsub_rn(px.fin.y, px.Cg),
                    Sb = __fsub_rn(px.fin.z, px.Cb);
        float dtau = -px.GT_Tfin;
        dtau = fmaf(px.G.x, fmaf(px.T, cr, -Sr), dtau);
        dtau = fmaf(px.G.y, fmaf(px.T, cg, -Sg), dtau);
        dtau = fmaf(px.G.z, fmaf(px.T, cb, -Sb), dtau);
        const float wa = __fmul_rn(Tk, alpha);
        gs = dtau * g.dt;
        const float gdt = dtau * sig;
        float g_ts = 0.0f;
        if (gdt != 0.0f) {
            const float4 none = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
            end_grad<true, true>(R, g, g.hi_q, g.hi, gdt, S.r[j], ds.edges, ds.nbr_idx, acc, o,
                                 none, S.eb[j], g_ts);
            end_grad<true, true>(R, g, g.lo_q, g.lo, -gdt, S.r[j], ds.edges, ds.nbr_idx, acc, o,
                                 none, S.eb[j], g_ts);
        }
        detail_reverse<T, KT>(ds, cell, X, ys0, ys1, ys2, qs0, qs1, ws, dG, wa, g_ts, S.r[j],
                              px.G, om, &buf[lane][0], &gbuf[lane][0], o);
    }
    const unsigned segall = __ballot_sync(0xffffffffu, seg);   // rows of buf that were written
    __syncwarp();
    // one column reduction per record of the pass (a group of records with disjoint lane
    // masks holds several cells; lanes without a segment never match)
    for (unsigned rem = segall; rem;) {
        const int jr = __shfl_sync(0xffffffffu, j, __ffs(rem) - 1);
        const unsigned segm = __ballot_sync(0xffffffffu, seg && j == jr);
        rem &= ~segm;
        const uint32_t cr = S.cell[jr];
        // dL/dv: lane -> site k = lane / 4 and 6 consecutive (a, c) entries
        const int k = lane >> 2, ac0 = (lane & 3) * 6;
        float accv[6] = {0, 0, 0, 0, 0, 0};
        for (unsigned mm = segm; mm; mm &= mm - 1) {
            const int l = __ffs(mm) - 1;
            const float wk = buf[l][k];
#pragma unroll
            for (int q = 0; q < 6; ++q) accv[q] = fmaf(wk, buf[l][8 + ac0 + q], accv[q]);
        }
        if (k < K && ds.g_sv) {
            float2 *dst = reinterpret_cast<float2 *>(ds.g_sv + ((size_t)K * cr + k) * 24 + ac0);
            atomicAdd(dst, make_float2(accv[0], accv[1]));
            atomicAdd(dst + 1, make_float2(accv[2], accv[3]));
            atomicAdd(dst + 2, make_float2(accv[4], accv[5]));
        }
        if (lane < 24) {
            float t = 0.0f;
            for (unsigned mm = segm; mm; mm &= mm - 1) t += gbuf[__ffs(mm) - 1][lane];
            if (lane < 16) {
                if ((lane >> 1) < K && ds.g_uv) atomicAdd(ds.g_uv + (size_t)2 * K * cr + lane, t);
            } else if (lane - 16 < K && ds.g_disp) {
                atomicAdd(ds.g_disp + (size_t)K * cr + (lane - 16), t);
            }
        }
    }
    __syncwarp();
    // own-cell terms (rgb_i is unused by detail cells: no colour gradient)
    float *accc = acc + 12 * (size_t)cell;
    if (grouped || __popc(segall) <= PF_K7_DIRECT_MAX) {
        if (seg) {
            atomicAdd(reinterpret_cast<float4 *>(accc), make_float4(o.px, o.py, o.pz, o.w));
            atomicAdd(reinterpret_cast<float4 *>(accc) + 2, make_float4(0.0f, o.nx, o.ny, o.nz));
            atomicAdd(reinterpret_cast<float4 *>(accc) + 1, make_float4(o.r, gs, 0.0f, 0.0f));
        }
    } else {
        float v[16] = {o.px, o.py, o.pz, o.w, o.r, gs, 0, 0, 0, o.nx, o.ny, o.nz, 0, 0, 0, 0};
        warp_reduce16_atomic<12>(v, accc, lane);
    }
}

// ---------------------------------------------------------------------------
// Split detail backward (PF_K7D_SPLIT).  The monolithic detail_segment runs the
// whole per-segment chain in the record replay's lockstep, where a record holds
// ~3 of 32 lanes.  Split: K7 replays the records (a pass = up to PF_K7D_GROUP
// disjoint records) and does only what the compositing order needs -- the
// segment colour (Eq. svrad, as K6), the compositing replay, dL/dt of the
// interval ends (neighbour REDs, own-cell terms, g_ts of the displaced face) --
// and emits one item per segment with a detail gradient; K7D then runs the chart
// geometry, radiance pass and reverse chain of P:284-293 one item per lane, with
// the per-cell column sums over the warp's 32 consecutive items.
// ---------------------------------------------------------------------------
template <int KT>
__device__ __forceinline__ void detail_segment_a(const Ray &R, const Seg &g, bool seg,
                                                 const WarpStage &S, int j, BwdPixel &px,
                                                 const DeviceScene &ds, float *acc, int lane,
                                                 const DetailCtx &X, const float *om, bool grouped,
                                                 const DetailItems &DI, uint32_t pixtag,
                                                 bool have_col, float cr, float cg, float cb)
{
    const uint32_t cell = S.cell[j];
    OwnGrad o = {0, 0, 0, 0, 0, 0, 0, 0};
    float gs = 0.0f, wa = 0.0f, g_ts = 0.0f, tpar = 0.0f;
    if (seg) {
        // the chart parameter of a ray parallel to the face (K7D uses it only then)
        tpar = __fadd_rn(g.tc, g.lo);
        if (!have_col)   // K6's colour slot was not available: Eq. svrad as K6
            detail_color<KT>(ds, cell, X.d, X.c, X.G.parallel ? (double)tpar : X.G.ts, om, cr, cg, cb);
        const float sig = S.sig[j];
        const float Tk = px.T;
        float alpha;
        composite_step(sig, g.dt, cr, cg, cb, px.T, px.Cr, px.Cg, px.Cb, alpha);
        const float Sr = __fsub_rn(px.fin.x, px.Cr), Sg = __fsub_rn(px.fin.y, px.Cg),
                    Sb = __fsub_rn(px.fin.z, px.Cb);
        float dtau = -px.GT_Tfin;
        dtau = fmaf(px.G.x, fmaf(px.T, cr, -Sr), dtau);
        dtau = fmaf(px.G.y, fmaf(px.T, cg, -Sg), dtau);
        dtau = fmaf(px.G.z, fmaf(px.T, cb, -Sb), dtau);
        wa = __fmul_rn(Tk, alpha);
        gs = dtau * g.dt;
        const float gdt = dtau * sig;
        if (gdt != 0.0f) {
            const float4 none = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
            end_grad<true, true>(R, g, g.hi_q, g.hi, gdt, S.r[j], ds.edges, ds.nbr_idx, acc, o,
                                 none, S.eb[j], g_ts);
            end_grad<true, true>(R, g, g.lo_q, g.lo, -gdt, S.r[j], ds.edges, ds.nbr_idx, acc, o,
                                 none, S.eb[j], g_ts);
        }
    }
    // own-cell terms of the interval ends and sigma
    float *accc = acc + 12 * (size_t)cell;
    const unsigned segm = __ballot_sync(0xffffffffu, seg);
    if (grouped || __popc(segm) <= PF_K7_DIRECT_MAX) {
        if (seg) {
            atomicAdd(reinterpret_cast<float4 *>(accc), make_float4(o.px, o.py, o.pz, o.w));
            atomicAdd(reinterpret_cast<float2 *>(accc + 4), make_float2(o.r, gs));
        }
    } else {
        float v[10] = {o.px, o.py, o.pz, o.w, o.r, gs, 0.0f, 0.0f, 0.0f, 0.0f};
        warp_reduce9_atomic(v, accc, lane);
    }
    // one item per segment whose detail chain has a gradient to give
    const bool emit = seg && (wa != 0.0f || g_ts != 0.0f);
    const unsigned em = __ballot_sync(0xffffffffu, emit);
    if (em) {
        const int l0 = __ffs(em) - 1;
        uint32_t base = 0;
        if (lane == l0) base = atomicAdd(DI.used, (uint32_t)__popc(em));
        base = __shfl_sync(0xffffffffu, base, l0);
        if (emit) {
            const uint32_t idx = base + (uint32_t)__popc(em & ((1u << lane) - 1u));
            if (idx < DI.cap) {
                DI.it[idx] = make_uint4(cell, pixtag, __float_as_uint(wa), __float_as_uint(g_ts));
                DI.tpar[idx] = tpar;
            }
        }
    }
}

#ifndef PF_K7D_SPLIT   // detail backward split into the replay (K7) and the chain (K7D)
#define PF_K7D_SPLIT 1
#endif
#ifndef PF_K7D_MINB_REPLAY   // split detail K7 (replay + colour + items): CTAs per SM
#define PF_K7D_MINB_REPLAY 3
#endif
#ifndef PF_K7D_PREFETCH   // K7D: next item one iteration ahead (measured: within noise, off)
#define PF_K7D_PREFETCH 0
#endif
#ifndef PF_K7D_RUNFAST   // K7D column sums: counted loop over contiguous runs (measured slower: 21.9 -> 22.6 ms, off)
#define PF_K7D_RUNFAST 0
#endif
#ifndef PF_K7D_ROWORDER   // split detail K7: row-major tile order (measured: train8 +1.2 ms, nerfsynth -0.2 ms; off)
#define PF_K7D_ROWORDER 0
#endif
#ifndef PF_K7D_MINB_CHAIN   // K7D (the chain, thread per item): CTAs per SM
#define PF_K7D_MINB_CHAIN 2
#endif
constexpr int kChainRow = 34;   // even: 8-byte aligned float2 reads of the outer-product rows
constexpr int kChainStride = 2 * kChainRow;   // per lane: a row of each of the two tiles

// K7D: the detail chain of the split backward, 32 consecutive items per warp
// (grid-stride).  va: the call's device ViewArgs (camera, grad_out per view).
template <int KT>
__global__ void __launch_bounds__(256, PF_K7D_MINB_CHAIN)
k7d_detail_chain(DeviceScene ds, const ViewArgs *__restrict__ va, DetailItems DI,
                 float *__restrict__ acc)
{
    extern __shared__ float dyn_smem[];   // per warp: [32][33] outer-product tile, [32][33] gradient tile
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float (*buf)[kChainRow] = reinterpret_cast<float (*)[kChainRow]>(dyn_smem + warp * 32 * kChainStride);
    float (*gbuf)[kChainRow] = buf + 32;
    const int K = KT == 8 ? 8 : ds.K;
    const uint32_t n = min(*DI.used, DI.cap);
    const uint32_t stride = gridDim.x * kWarps * 32u;
    uint32_t base = (blockIdx.x * kWarps + warp) * 32u;
    // the next batch's item is loaded while this one is processed (the chain starts
    // with a dependent walk: item -> view, pixel, cell -> their records)
    uint4 itn = (PF_K7D_PREFETCH && base + lane < n) ? DI.it[base + lane] : make_uint4(0u, 0u, 0u, 0u);
    for (; base < n; base += stride) {
        const uint32_t i = base + (uint32_t)lane;
        const bool seg = i < n;
        uint4 it;
        if (PF_K7D_PREFETCH) {
            it = itn;
            if (base + stride + lane < n) itn = DI.it[base + stride + lane];
        } else {
            it = seg ? DI.it[i] : make_uint4(0u, 0u, 0u, 0u);
        }
        uint32_t cell = 0xffffffffu;
        OwnGrad o = {0, 0, 0, 0, 0, 0, 0, 0};
        if (seg) {
            cell = it.x;
            const float wa = __uint_as_float(it.z), g_ts = __uint_as_float(it.w);
            const ViewArgs &V = va[it.y >> 25];
            const CamParams &cam = V.cam;
            const uint32_t pix = it.y & 0x1ffffffu;
            const int py = (int)(pix / (uint32_t)cam.W), pxx = (int)(pix - (uint32_t)py * cam.W);
            DetailCtx X;
            ray_dir(cam, pxx + 0.5, py + 0.5, X.d, nullptr);
            Ray R;
            R.dx = __double2float_rn(X.d[0]);
            R.dy = __double2float_rn(X.d[1]);
            R.dz = __double2float_rn(X.d[2]);
            float om[8];
            sv_axis_weights(ds, R, om);
            cell_c(ds, cam, cell, X.c);
            const float rad = __ldg(ds.cellA + cell).w;
            detail_plane<KT>(ds, cell, X.d, X.c, rad, X.G);
            const float4 Gp = V.grad_out[pix];
            // Eq. svrad at x (the interval entry for a parallel ray), by detail_color's
            // explicit op sequence: the weights w_k and the per-site c_k . G
            const double *F = ds.cellF + (size_t)kCellF * cell;
            const double tcol = X.G.parallel ? (double)DI.tpar[i] : X.G.ts;
            const double ys0 = __fma_rn(tcol, X.d[0], -X.c[0]), ys1 = __fma_rn(tcol, X.d[1], -X.c[1]),
                         ys2 = __fma_rn(tcol, X.d[2], -X.c[2]);
            const double qs0 = __fma_rn(ys0, __ldg(F + 3), __fma_rn(ys1, __ldg(F + 4), __dmul_rn(ys2, __ldg(F + 5))));
            const double qs1 = __fma_rn(ys0, __ldg(F + 6), __fma_rn(ys1, __ldg(F + 7), __dmul_rn(ys2, __ldg(F + 8))));
            float ws[kMaxDetail], dG[kMaxDetail];
            float2 st[kMaxDetail];
            load_sites(reinterpret_cast<const float2 *>(ds.duv) + (size_t)K * cell, K, st);
            soft_voronoi(st, K, qs0, qs1, ds.sv_tau, ws);
            const float4 *sv = reinterpret_cast<const float4 *>(ds.dsv) + (size_t)6 * K * cell;
#pragma unroll
            for (int k = 0; k < kMaxDetail; ++k) {
                dG[k] = 0.0f;
                if (k < K) {
                    float v[24];
#pragma unroll
                    for (int q = 0; q < 6; ++q) {
                        const float4 x = __ldg(sv + 6 * k + q);
                        v[4 * q] = x.x; v[4 * q + 1] = x.y; v[4 * q + 2] = x.z; v[4 * q + 3] = x.w;
                    }
                    float kr = 0.0f, kg = 0.0f, kb = 0.0f;
#pragma unroll
                    for (int a = 0; a < 8; ++a) {
                        kr = fmaf(om[a], v[3 * a], kr);
                        kg = fmaf(om[a], v[3 * a + 1], kg);
                        kb = fmaf(om[a], v[3 * a + 2], kb);
                    }
                    dG[k] = fmaf(kr, Gp.x, fmaf(kg, Gp.y, kb * Gp.z));   // c_k . G
                }
            }
            detail_reverse<double, KT>(ds, cell, X, ys0, ys1, ys2, qs0, qs1, ws, dG, wa, g_ts, rad,
                                       Gp, om, &buf[lane][0], &gbuf[lane][0], o);
            // own-cell terms of the chain as tile columns 24..30
            gbuf[lane][24] = o.px;
            gbuf[lane][25] = o.py;
            gbuf[lane][26] = o.pz;
            gbuf[lane][27] = o.r;
            gbuf[lane][28] = o.nx;
            gbuf[lane][29] = o.ny;
            gbuf[lane][30] = o.nz;
        }
        __syncwarp();
        // per-cell column sums over the warp's items (consecutive items mostly share a cell)
        const unsigned valid = __ballot_sync(0xffffffffu, seg);
        for (unsigned rem = valid; rem;) {
            const uint32_t cr = __shfl_sync(0xffffffffu, cell, __ffs(rem) - 1);
            const unsigned segm = __ballot_sync(0xffffffffu, seg && cell == cr);
            rem &= ~segm;
            // one pass over the run's items: lane (k = lane / 4, 6 consecutive (a, c)) of
            // the outer product (float2 rows: stride kRow) and column `lane` of gbuf
            const int k = lane >> 2, ac0 = (lane & 3) * 6;
            float2 a0 = make_float2(0.0f, 0.0f), a1 = a0, a2 = a0;
            float t = 0.0f;
            auto add_item = [&](int l) {
                const float wk = buf[l][k];
                const float2 *row = reinterpret_cast<const float2 *>(&buf[l][8 + ac0]);
                const float2 b0 = row[0], b1 = row[1], b2 = row[2];
                a0.x = fmaf(wk, b0.x, a0.x); a0.y = fmaf(wk, b0.y, a0.y);
                a1.x = fmaf(wk, b1.x, a1.x); a1.y = fmaf(wk, b1.y, a1.y);
                a2.x = fmaf(wk, b2.x, a2.x); a2.y = fmaf(wk, b2.y, a2.y);
                t += gbuf[l][lane];
            };
            const int l0 = __ffs(segm) - 1, nrun = __popc(segm);
            if (PF_K7D_RUNFAST && (segm >> l0) == (nrun == 32 ? 0xffffffffu : (1u << nrun) - 1u)) {
                // a contiguous run of lanes (the common case): a plain counted loop
                for (int l = l0; l < l0 + nrun; ++l) add_item(l);
            } else {
                for (unsigned mm = segm; mm; mm &= mm - 1) add_item(__ffs(mm) - 1);
            }
            if (k < K && ds.g_sv) {
                float2 *dst = reinterpret_cast<float2 *>(ds.g_sv + ((size_t)K * cr + k) * 24 + ac0);
                atomicAdd(dst, a0);
                atomicAdd(dst + 1, a1);
                atomicAdd(dst + 2, a2);
            }
            if (lane < 31) {
                if (lane < 16) {
                    if ((lane >> 1) < K && ds.g_uv) atomicAdd(ds.g_uv + (size_t)2 * K * cr + lane, t);
                } else if (lane < 24) {
                    if (lane - 16 < K && ds.g_disp) atomicAdd(ds.g_disp + (size_t)K * cr + (lane - 16), t);
                } else {
                    // 24..26 -> p (slots 0..2), 27 -> r (slot 4), 28..30 -> n (slots 9..11)
                    const int slot = lane < 27 ? lane - 24 : (lane == 27 ? 4 : lane - 19);
                    if (t != 0.0f) atomicAdd(acc + 12 * (size_t)cr + slot, t);
                }
            }
        }
        __syncwarp();
    }
}

// Backward of one segment (lanes with seg) + scatter of the cell's gradients.
template <bool kDipole, int kDetail, bool kSplit = false>
__device__ __forceinline__ void segment_backward(const Ray &R, const Seg &g, bool seg,
                                                 const WarpStage &S, int j, BwdPixel &px,
                                                 const DeviceScene &ds, float *acc, int lane,
                                                 float cr, float cg, float cb, const float4 &dnrm,
                                                 const DetailCtx *X, const float *om,
                                                 float (*buf)[33], bool grouped,
                                                 const DetailItems &DI, uint32_t pixtag,
                                                 bool have_col = false)
{
    if (kDetail && kSplit) {
        detail_segment_a<kDetail>(R, g, seg, S, j, px, ds, acc, lane, *X, om, grouped, DI, pixtag,
                                  have_col, cr, cg, cb);
        return;
    }
    if (kDetail) {
        // (an fp32 instantiation for non-grazing warps measured slower on B200: the
        // fp64 -> fp32 conversions cost more than the fp64 arithmetic they save)
        detail_segment<double, kDetail>(R, g, seg, S, j, px, ds, acc, lane, *X, om, buf,
                                        reinterpret_cast<float (*)[25]>(&buf[32][0]), grouped);
        return;
    }
    constexpr bool dipole = kDipole;
    OwnGrad o = {0, 0, 0, 0, 0, 0, 0, 0};
    float gs = 0.0f, gR = 0.0f, gG = 0.0f, gB = 0.0f, g_ts = 0.0f;
    int nj_hi = -1, nj_lo = -1;   // neighbour terms for the aggregated scatter
    float4 nv_hi = make_float4(0.0f, 0.0f, 0.0f, 0.0f), nv_lo = nv_hi;
    if (seg) {
        const float sig = S.sig[j];
        const float Tk = px.T;
        float alpha;
        composite_step(sig, g.dt, cr, cg, cb, px.T, px.Cr, px.Cg, px.Cb, alpha);
        // px.T is now T_{k+1}; C is C_k; S_k = out_rgb - C_k
        const float Sr = __fsub_rn(px.fin.x, px.Cr), Sg = __fsub_rn(px.fin.y, px.Cg),
                    Sb = __fsub_rn(px.fin.z, px.Cb);
        float dtau = -px.GT_Tfin;
        dtau = fmaf(px.G.x, fmaf(px.T, cr, -Sr), dtau);
        dtau = fmaf(px.G.y, fmaf(px.T, cg, -Sg), dtau);
        dtau = fmaf(px.G.z, fmaf(px.T, cb, -Sb), dtau);
        const float wa = __fmul_rn(Tk, alpha);
        gR = wa * px.G.x;
        gG = wa * px.G.y;
        gB = wa * px.G.z;
        gs = dtau * g.dt;
        const float gdt = dtau * sig;
        if (gdt != 0.0f) {
            const float rad = S.r[j];
            const uint32_t eb = S.eb[j];
            end_grad<kDipole, false>(R, g, g.hi_q, g.hi, gdt, rad, ds.edges, ds.nbr_idx, acc, o,
                                     dnrm, eb, g_ts, PF_K7_AGG ? &nj_hi : nullptr, &nv_hi);
            end_grad<kDipole, false>(R, g, g.lo_q, g.lo, -gdt, rad, ds.edges, ds.nbr_idx, acc, o,
                                     dnrm, eb, g_ts, PF_K7_AGG ? &nj_lo : nullptr, &nv_lo);
        }
    }
    if (PF_K7_AGG) {
        red_nbr_agg(acc, nj_hi, nv_hi, lane);
        red_nbr_agg(acc, nj_lo, nv_lo, lane);
    }
    // own-cell terms: one lane alone issues its atomics, else a transposing warp
    // reduction then one 9-lane atomic instruction
    float *accc = acc + 12 * (size_t)S.cell[j];
    const unsigned sm = __ballot_sync(0xffffffffu, seg);
    if (grouped || __popc(sm) <= PF_K7_DIRECT_MAX) {   // (a group spans several cells)
        if (seg) {
            atomicAdd(reinterpret_cast<float4 *>(accc), make_float4(o.px, o.py, o.pz, o.w));
            if (dipole)
                atomicAdd(reinterpret_cast<float4 *>(accc) + 2, make_float4(gB, o.nx, o.ny, o.nz));
            else
                atomicAdd(accc + 8, gB);
            atomicAdd(reinterpret_cast<float4 *>(accc) + 1, make_float4(o.r, gs, gR, gG));
        }
    } else if (dipole) {
        float v[16] = {o.px, o.py, o.pz, o.w, o.r, gs, gR, gG, gB, o.nx, o.ny, o.nz, 0, 0, 0, 0};
        warp_reduce16_atomic<12>(v, accc, lane);
    } else {
        float v[10] = {o.px, o.py, o.pz, o.w, o.r, gs, gR, gG, gB, 0.0f};
        warp_reduce9_atomic(v, accc, lane);
    }
}

}  // namespace

template <bool kDipole, int kDetail, bool kFused = false, bool kSplit = false>
__global__ void __launch_bounds__(256, kDetail ? (kSplit ? PF_K7D_MINB_REPLAY : PF_K7D_MINB)
                                               : PF_K7_MINB)
k7_backward(DeviceScene ds, const ViewArgs one, const ViewArgs *__restrict__ va, int ntiles,
            float *__restrict__ acc, int view0, DetailItems DI)
{
    __shared__ ViewArgs VAs[1];
    if (kFused) load_view_args(va, ntiles, VAs[0]);
    const ViewArgs &VA = kFused ? VAs[0] : one;
    const CamParams &cam = VA.cam;
    const uint2 *__restrict__ ranges = VA.ranges;
    const uint32_t *__restrict__ vals = VA.vals;
    const float4 *__restrict__ saved = VA.saved;
    const float4 *__restrict__ grad_out = VA.grad_out;
    const uint32_t *__restrict__ chunk_off = VA.chunk_off;
    const uint2 *__restrict__ desc = VA.desc;
    const uint32_t *__restrict__ wdone = VA.wdone;
    const uint32_t *__restrict__ rec = VA.rec;
    __shared__ WarpStage WS[kWarps];
    __shared__ PixelRays PR;
    __shared__ WarpCtx WC[kWarps];
    __shared__ float4 WN[kDipole ? kWarps * 32 : 1];
    extern __shared__ float dyn_smem[];   // detail variant: [kWarps][32][33] reduction tiles
    // split detail K7: tiles in row-major order, so the K7D items of concurrent CTAs come
    // from neighbouring tiles (shared cells: L2 reuse in K7D); else the LPT order
    const int bt = kFused ? (int)(blockIdx.x % ntiles) : (int)blockIdx.x;
    const int tile = (kSplit && PF_K7D_ROWORDER) ? bt : (int)VA.order[bt], lane = threadIdx.x & 31,
              warp = threadIdx.x >> 5;
    WarpStage &S = WS[warp];
    if (lane == 0) S.nrm = kDipole ? WN + warp * 32 : nullptr;
    WarpCtx &W = WC[warp];
    // detail: per warp a [32][33] outer-product tile followed by a [32][25] tile of
    // the per-lane site / displacement gradients
    float (*buf)[33] = reinterpret_cast<float (*)[33]>(dyn_smem + (kDetail ? warp * 32 * 58 : 0));
    PixelSetup P;
    setup_pixel(cam, tile, P, PR, W);
    const uint2 rg = ranges[tile];
    BwdPixel px;
    px.T = 1.0f;
    px.Cr = px.Cg = px.Cb = 0.0f;
    bool done = !P.valid;
    px.fin = make_float4(0, 0, 0, 1);
    px.G = make_float4(0, 0, 0, 0);
    if (P.valid) {
        const size_t pix = (size_t)P.y * cam.W + P.x;
        px.fin = saved[pix];
        px.G = grad_out[pix];
    }
    px.GT_Tfin = __fmul_rn(px.G.w, px.fin.w);
    // split detail backward: the item's (view, pixel)
    const uint32_t pixtag = ((uint32_t)(kFused ? (int)blockIdx.x / ntiles : view0) << 25) |
                            (uint32_t)(P.y * cam.W + P.x);
    float om[8];
    if (kDetail) sv_axis_weights(ds, P.R, om);
    DetailCtx X;
    if (kDetail) {
        X.d[0] = PR.dx[threadIdx.x];
        X.d[1] = PR.dy[threadIdx.x];
        X.d[2] = PR.dz[threadIdx.x];
    }
    // per entry: the dipole face (plain: the staged normal; detail: the lane's
    // displaced face) and the segment colour
    auto prepare = [&](int j, bool active, float4 &dpl, float &cr, float &cg, float &cb) {
        cr = S.cr[j];
        cg = S.cg[j];
        cb = S.cb[j];
        dpl = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        if (kDetail) {
            if (active) {
                cell_c(ds, cam, S.cell[j], X.c);
                dpl = detail_plane<kDetail>(ds, S.cell[j], X.d, X.c, S.r[j], X.G);
            }
        } else if (kDipole) {
            dpl = S.nrm[j];
        }
    };
    constexpr bool kGroup = (kDetail ? PF_K7D_GROUP : PF_K7_GROUP) > 1;
    constexpr uint32_t kGroupMax = kDetail ? PF_K7D_GROUP : PF_K7_GROUP;
    const uint32_t nchunks = wdone[(size_t)tile * kWarps + warp];
    const uint32_t c0 = chunk_off[tile];
    uint2 dnext = nchunks ? desc[(size_t)c0 * kWarps + warp] : make_uint2(0u, 0u);
    for (uint32_t c = 0; c < nchunks; ++c) {
        const uint2 d = dnext;
        if (PF_K7_PREFETCH && c + 1 < nchunks) {
            // the next chunk's descriptor now, and its record block pulled into L2 while
            // this chunk is replayed (records were written by K6 long before: DRAM)
            dnext = desc[(size_t)(c0 + c + 1) * kWarps + warp];
            if (dnext.y != 0u && dnext.y != kOverflow) {
                const char *rb = reinterpret_cast<const char *>(rec + (size_t)dnext.x * kRecWords);
                const uint32_t bytes = dnext.y * (uint32_t)(4 * kRecWords);
                for (uint32_t o = (uint32_t)lane * 128u; o < bytes; o += 32u * 128u)
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(rb + o));
            }
        } else if (c + 1 < nchunks) {
            dnext = desc[(size_t)(c0 + c + 1) * kWarps + warp];
        }
        if (d.y == 0u) continue;
        const uint32_t base = rg.x + 32u * c;
        if (d.y == kOverflow) {
            // records did not fit: full replay of this chunk (same code as K6)
            unsigned m = stage_chunk<kDipole>(S, ds, cam, vals, base + lane, rg.y, W, lane);
            while (m) {
                const int j = __ffs(m) - 1;
                m &= m - 1;
                Seg g;
                bool hit = false;
                if (!done) hit = sphere_hit(P.R, S, j, g, ds, cam, PR);
                if (!__any_sync(0xffffffffu, hit)) continue;
                float4 dpl;
                float cr, cg, cb;
                if (kDetail) {   // as K6: the face only where the interval is non-empty
                    clip_interval<true, false>(P.R, ds.edges, S.eb[j], S.deg[j], g, hit, dpl);
                    const bool pre = g.dt > 0.0f;
                    prepare(j, pre, dpl, cr, cg, cb);
                    if (__any_sync(0xffffffffu, pre)) {
                        clip_plane<true>(P.R, dpl, kEndDipole, g);
                        const float dt = __fsub_rn(g.hi, g.lo);
                        g.dt = (pre && dt > 0.0f) ? dt : 0.0f;
                    }
                } else {
                    prepare(j, hit, dpl, cr, cg, cb);
                    clip_interval<true, kDipole>(P.R, ds.edges, S.eb[j], S.deg[j], g, hit, dpl);
                }
                const bool seg = g.dt > 0.0f;
                if (!__any_sync(0xffffffffu, seg)) continue;
                segment_backward<kDipole, kDetail, kSplit>(P.R, g, seg, S, j, px, ds, acc, lane, cr,
                                                           cg, cb, dpl, &X, om, buf, false, DI,
                                                           pixtag);
                if (seg && px.T < kTStop) done = true;
            }
            __syncwarp();
            continue;
        }
        // recorded entries only: stage them (lane k <-> record k)
        const uint32_t nrec = d.y;
        const uint32_t *R0 = rec + (size_t)d.x * kRecWords;
        uint32_t my_mask = 0, my_cslot = kNoCol;
        if (lane < (int)nrec) {
            const uint2 mp = __ldg(reinterpret_cast<const uint2 *>(R0 + (size_t)lane * kRecWords));
            my_mask = mp.x;
            if (kDetail) my_cslot = mp.y >> 5;
            const uint32_t cell = kDetail ? __ldg(vals + base + (mp.y & 31u)) : mp.y;
            const float4 A = __ldg(ds.cellA + cell);
            double x0, x1, x2;
            const double t = cell_offset(cam, A, W, x0, x1, x2);
            stage_slot<kDipole>(S, lane, ds, cell, A, x0, x1, x2, t, W);
        }
        __syncwarp();
        for (uint32_t k = 0; k < nrec;) {
            // one pass over a group of consecutive records whose lane masks are
            // pairwise disjoint: each lane takes the record holding it (at most one),
            // so every pixel still replays its own segments in list order
            uint32_t uni = __shfl_sync(0xffffffffu, my_mask, (int)k);
            int jl = ((uni >> lane) & 1u) ? (int)k : -1;
            uint32_t k1 = k + 1;
            if (kGroup) {
                while (k1 < nrec && k1 - k < kGroupMax) {
                    const uint32_t m2 = __shfl_sync(0xffffffffu, my_mask, (int)k1);
                    if (m2 & uni) break;
                    uni |= m2;
                    if ((m2 >> lane) & 1u) jl = (int)k1;
                    ++k1;
                }
            }
            const bool grouped = k1 - k > 1u;
            const bool seg = jl >= 0;
            // lanes without a segment take the group's first record (a single-record
            // group's warp reduction reads S.cell[j] on any lane)
            const int j = seg ? jl : (int)k;
            k = k1;
            const uint32_t code =
                seg ? __ldg(reinterpret_cast<const uint16_t *>(R0 + (size_t)j * kRecWords + 2) + lane) : 0u;
            Seg g;
            g.dt = 0.0f;
            float4 dpl;
            float cr, cg, cb;
            if (seg) sphere_hit(P.R, S, j, g, ds, cam, PR);   // identical to K6 (recorded hit)
            // split detail: the segment's colour and displacement as K6 stored them
            const float4 *colp = nullptr;
            if (kSplit) {
                const uint32_t cs = __shfl_sync(0xffffffffu, my_cslot, j),
                               mj = __shfl_sync(0xffffffffu, my_mask, j);
                if (seg && cs != kNoCol && VA.col)
                    colp = VA.col + cs + __popc(mj & ((1u << lane) - 1u));
            }
            if (kSplit && colp) {
                // the displaced face (m, delta) without the chart evaluation: m as
                // detail_plane rounds it, delta as K6 computed it (bit-identical ends)
                const double *F = ds.cellF + (size_t)kCellF * S.cell[j];
                const float4 cv = __ldg(colp);
                dpl = make_float4(__double2float_rn(__ldg(F)), __double2float_rn(__ldg(F + 1)),
                                  __double2float_rn(__ldg(F + 2)), cv.w);
                cr = cv.x;
                cg = cv.y;
                cb = cv.z;
            } else {
                prepare(j, seg, dpl, cr, cg, cb);
            }
            if (seg) {
                const uint32_t eb = S.eb[j];
                g.lo = coded_end<kDipole>(P.R, ds.edges, ds.nbr_idx, eb, code & 0xffu, true, g,
                                          g.lo_q, dpl);
                g.hi = coded_end<kDipole>(P.R, ds.edges, ds.nbr_idx, eb, code >> 8, false, g,
                                          g.hi_q, dpl);
            }
            const bool full = seg && (((code & 0xffu) == 255u) || ((code >> 8) == 255u));
            if (__any_sync(0xffffffffu, full)) {
                Seg h = g;
                if (full) {
                    clip_interval<true, kDipole>(P.R, ds.edges, S.eb[j], S.deg[j], h, true, dpl);
                    g = h;
                } else {
                    clip_interval<true, kDipole>(P.R, ds.edges, S.eb[j], S.deg[j], h, false, dpl);
                }
            }
            if (seg) g.dt = __fsub_rn(g.hi, g.lo);
            segment_backward<kDipole, kDetail, kSplit>(P.R, g, seg, S, j, px, ds, acc, lane, cr, cg,
                                                       cb, dpl, &X, om, buf, grouped, DI, pixtag,
                                                       colp != nullptr);
            if (seg && px.T < kTStop) done = true;   // for a later overflow chunk
        }
        __syncwarp();
    }
}

static bool backward_fused(const pf_scene *s, int T)
{
    return s->k6_per_view == 0 || (s->k6_per_view != 1 && T < kFuseTiles);
}

// items the split detail backward needs at once: all views of a fused launch, else
// the largest view (K7 / K7D alternate per view on the stream)
int64_t detail_items_needed(const pf_scene *s, const ViewState *views, int V)
{
    if (!s->ds.K || !PF_K7D_SPLIT) return 0;
    const int T = views[0].cam.tiles_x * views[0].cam.tiles_y;
    int64_t sum = 0, mx = 0;
    for (int v = 0; v < V; ++v) {
        sum += views[v].nseg;
        mx = views[v].nseg > mx ? views[v].nseg : mx;
    }
    return backward_fused(s, T) ? sum : mx;
}

template <bool kDipole, int kDetail>
static int launch_backward_t(pf_scene *s, const ViewState *views, int V, const ViewArgs *args,
                             cudaStream_t st)
{
    const int T = views[0].cam.tiles_x * views[0].cam.tiles_y;
    constexpr bool kSplit = kDetail && PF_K7D_SPLIT;
    constexpr int smem = (kDetail && !kSplit) ? kWarps * 32 * 58 * (int)sizeof(float) : 0;
    constexpr int smem_chain = kWarps * 32 * kChainStride * (int)sizeof(float);
    if (!s->attrs_k7) {
        if (smem) {
            cudaFuncSetAttribute(k7_backward<kDipole, kDetail>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            cudaFuncSetAttribute(k7_backward<kDipole, kDetail, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        }
        if (kSplit)
            cudaFuncSetAttribute(k7d_detail_chain<kDetail>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, smem_chain);
    }
    s->attrs_k7 = true;
    const ViewArgs *h = s->host_args.data();
    float *acc = s->acc.as<float>();
    // the split detail backward: items of view group g counted in item_cnt[g]
    // (zeroed by the caller), K7D right after the group's K7
    auto items = [&](int g, int64_t n) {
        DetailItems DI = {};
        if (kSplit) {
            DI.it = s->items.as<uint4>();
            DI.tpar = s->item_tpar.as<float>();
            DI.used = s->item_cnt.as<uint32_t>() + g;
            DI.cap = (uint32_t)n;
        }
        return DI;
    };
    auto chain = [&](const DetailItems &DI, int64_t n) {
        if (!kSplit || n <= 0) return 0;
        const int64_t blocks = (n + 255) / 256, cap_blocks = 148 * PF_K7D_MINB_CHAIN * 8;
        k7d_detail_chain<kDetail><<<(unsigned)(blocks < cap_blocks ? blocks : cap_blocks), 256,
                                    smem_chain, st>>>(s->ds, args, DI, acc);
        return 1;
    };
    if (backward_fused(s, T)) {
        int64_t nseg = 0;
        for (int v = 0; v < V; ++v) nseg += views[v].nseg;
        const DetailItems DI = items(0, nseg);
        k7_backward<kDipole, kDetail, true, kSplit><<<(unsigned)(T * V), 256, smem, st>>>(
            s->ds, h[0], args, T, acc, 0, DI);
        return 1 + chain(DI, nseg);
    }
    int n = 0;
    // plain scenes: views alternate between two streams (the split detail backward
    // shares one item arena between a view's K7 and K7D: one stream)
    const bool two = !kSplit && view_streams_begin(s, st, V);
    for (int v = 0; v < V; ++v) {
        if (views[v].P == 0) continue;
        const DetailItems DI = items(v, views[v].nseg);
        cudaStream_t sv = (two && (v & 1)) ? s->pair : st;
        k7_backward<kDipole, kDetail, false, kSplit><<<T, 256, smem, sv>>>(s->ds, h[v], nullptr, T,
                                                                           acc, v, DI);
        n += 1 + chain(DI, views[v].nseg);
    }
    view_streams_end(s, st, two);
    return n;
}

cudaError_t launch_backward(pf_scene *s, const ViewState *views, int V, const ViewArgs *args,
                            cudaStream_t st)
{
    cudaEvent_t ev;
    stage_begin(s, 7, st, &ev);
    int n;
    if (s->ds.K == 8)
        n = launch_backward_t<true, 8>(s, views, V, args, st);
    else if (s->ds.K)
        n = launch_backward_t<true, 1>(s, views, V, args, st);
    else if (s->ds.cellN)
        n = launch_backward_t<true, 0>(s, views, V, args, st);
    else
        n = launch_backward_t<false, 0>(s, views, V, args, st);
    s->launches += n;
    stage_end(s, 7, st, ev);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------
// K8: add the packed accumulators into the caller's arrays (+=)
// ------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
k8_unpack(int64_t N, const float4 *__restrict__ acc, float *gs, float *gw, float *gr, float *gd,
          float *gc, float *gn)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const float4 a = acc[3 * i], b = acc[3 * i + 1], c = acc[3 * i + 2];
    gs[3 * i + 0] += a.x;
    gs[3 * i + 1] += a.y;
    gs[3 * i + 2] += a.z;
    gw[i] += a.w;
    gr[i] += b.x;
    gd[i] += b.y;
    gc[3 * i + 0] += b.z;
    gc[3 * i + 1] += b.w;
    gc[3 * i + 2] += c.x;
    if (gn) {
        gn[3 * i + 0] += c.y;
        gn[3 * i + 1] += c.z;
        gn[3 * i + 2] += c.w;
    }
}

cudaError_t launch_unpack(pf_scene *s, float *gs, float *gw, float *gr, float *gd, float *gc,
                          float *gn, cudaStream_t st)
{
    int64_t N = s->ds.N;
    cudaEvent_t ev;
    stage_begin(s, 8, st, &ev);
    k8_unpack<<<ceil_div(N, 256), 256, 0, st>>>(N, s->acc.as<float4>(), gs, gw, gr, gd, gc, gn);
    ++s->launches;
    stage_end(s, 8, st, ev);
    return cudaGetLastError();
}

}  // namespace pf
