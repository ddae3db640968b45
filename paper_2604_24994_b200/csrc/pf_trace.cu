// pf_trace.cu -- NEXT-4: the adjacency-walk ray tracer of bounded power cells
// (§3.1 "walk from one cell to the next by checking all faces",
// P:210 §3.2 "the cell-to-cell traversal strategy ... still applies ... in
// addition to considering the sphere bounds", App. C; reading R7 of
// DESIGN.md).
//
// One thread per pixel ray (CTA = 16x16 tile, warp = 8x4 block as in K6, so a
// warp's rays walk through neighbouring cells).  The walk:
//   t <- t_near, c <- locate(t)
//   loop: c's interval inside its ball, clipped by its Čech-list radical planes
//         (the identical clip_interval of K6, in a per-pixel exact fp64 frame),
//         and the constraint that ends it; the occupied segment (dipole / detail
//         face applied) is composited front to back (a10, early stop T < 1e-4);
//         a plane exit moves to the neighbour that owns the face (one CSR read,
//         O(1) per transition); a sphere exit leaves the union of balls there
//         (w = r^2: no other ball contains the exit point), so the walk jumps
//         the gap: locate(t) on the ball BVH (pf_bvh.cuh, NEXT-3's LBVH).
//   locate(t): among the balls whose chord ends after t, the smallest
//         max(t_entry, t), ties by the smaller power at that point (fp64 at the
//         leaves, exactly the oracle's rule); boxes pruned by a widened fp32
//         slab test against the best entry found so far.
// A step without progress (a degenerate crossing, or fp32 slivers at a face)
// re-locates past the current and previous cells; after two such steps in a
// row the walk nudges t forward by 1e-6 (1 + |t|); a walk longer than
// kMaxSteps is counted as diverged and stops (stats[4]).
#include <cuda_runtime.h>
#include <math.h>

#include "pf_bvh.cuh"
#include "pf_internal.cuh"
#include "pf_pixel.cuh"

namespace pf {

namespace {

constexpr int kTraceStack = 64;
constexpr int kMaxSteps = 1 << 16;
constexpr uint32_t kNone = 0xffffffffu;

// Tracer node layout: internal node i stores both children's boxes (the walk
// tests them without fetching the children), 4 float4 = 64 B:
//   [0] = (L.lo, code L)  [1] = (L.hi, code R)  [2] = (R.lo, -)  [3] = (R.hi, -)
// code = internal node index, or kLeaf | ball id (the leaf's ball, no order[] read).
constexpr uint32_t kLeaf = 0x80000000u;

struct Bvh {
    const float4 *nodes;
    int64_t n;
};

__global__ void k9_pack_nodes(const uint32_t *__restrict__ left, const uint32_t *__restrict__ right,
                              const Box *__restrict__ bint, const Box *__restrict__ bleaf,
                              const uint32_t *__restrict__ order, int64_t n, float4 *__restrict__ nodes)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n - 1) return;
    const uint32_t L = left[i], R = right[i];
    const Box bl = (L & 1u) ? bleaf[L >> 1] : bint[L >> 1];
    const Box br = (R & 1u) ? bleaf[R >> 1] : bint[R >> 1];
    const uint32_t cl = (L & 1u) ? (kLeaf | order[L >> 1]) : (L >> 1);
    const uint32_t cr = (R & 1u) ? (kLeaf | order[R >> 1]) : (R >> 1);
    nodes[4 * i + 0] = make_float4(bl.lo[0], bl.lo[1], bl.lo[2], __uint_as_float(cl));
    nodes[4 * i + 1] = make_float4(bl.hi[0], bl.hi[1], bl.hi[2], __uint_as_float(cr));
    nodes[4 * i + 2] = make_float4(br.lo[0], br.lo[1], br.lo[2], 0.0f);
    nodes[4 * i + 3] = make_float4(br.hi[0], br.hi[1], br.hi[2], 0.0f);
}

// per-ray slab constants: t = b * id - Q * id -+ pad |id| for the widened box
struct SlabRay {
    float id[3], olo[3], ohi[3];
};

__device__ __forceinline__ bool slab2(const float4 lo, const float4 hi, const SlabRay &S, float t0,
                                      float t1, float &tent)
{
    float a0 = fmaf(lo.x, S.id[0], S.olo[0]), b0 = fmaf(hi.x, S.id[0], S.ohi[0]);
    float a1 = fmaf(lo.y, S.id[1], S.olo[1]), b1 = fmaf(hi.y, S.id[1], S.ohi[1]);
    float a2 = fmaf(lo.z, S.id[2], S.olo[2]), b2 = fmaf(hi.z, S.id[2], S.ohi[2]);
    const float lo_t = fmaxf(fmaxf(t0, fminf(a0, b0)), fmaxf(fminf(a1, b1), fminf(a2, b2)));
    const float hi_t = fminf(fminf(t1, fmaxf(a0, b0)), fminf(fmaxf(a1, b1), fmaxf(a2, b2)));
    tent = lo_t;
    return lo_t <= hi_t;
}

// exact (fp64) ball test of the oracle's locate rule; updates the best candidate
__device__ __forceinline__ void locate_ball(const DeviceScene &ds, uint32_t b, const double Q[3],
                                            const double d[3], double t, uint32_t &best, double &bt,
                                            double &bp)
{
    const float4 A = __ldg(ds.cellA + b);
    const double c0 = (double)A.x - Q[0], c1 = (double)A.y - Q[1], c2 = (double)A.z - Q[2];
    const double tc = d[0] * c0 + d[1] * c1 + d[2] * c2;
    const double e0 = c0 - tc * d[0], e1 = c1 - tc * d[1], e2 = c2 - tc * d[2];
    const double r = (double)A.w;
    const double h = r * r - (e0 * e0 + e1 * e1 + e2 * e2);
    if (!(h > 0.0)) return;
    const double sq = sqrt(h);
    if (!(tc + sq > t)) return;
    const double tt = tc - sq > t ? tc - sq : t;
    if (best != kNone && tt > bt) return;
    const double x0 = tt * d[0] - c0, x1 = tt * d[1] - c1, x2 = tt * d[2] - c2;
    const double pw = x0 * x0 + x1 * x1 + x2 * x2 - (double)__ldg(ds.weights + b);
    if (best == kNone || tt < bt || (pw < bp || (pw == bp && b < best))) {
        best = b;
        bt = tt;
        bp = pw;
    }
}

// the first point of the union of balls at or after t (see the file comment);
// returns the ball / cell, or kNone if the ray leaves every ball.  Front-to-back
// traversal: both child boxes are tested at the parent, leaf balls at once (the
// best entry tightens the slab's far bound), the nearer internal child is walked
// next and the farther one stacked with its entry (skipped if beyond the best).
__device__ uint32_t locate(const DeviceScene &ds, const Bvh &B, const double Q[3], const double d[3],
                           const SlabRay &SR, double t, uint32_t ex1, uint32_t ex2)
{
    uint32_t best = kNone;
    double bt = 1e300, bp = 0.0;
    if (B.n == 1) {
        if (ex1 != 0u && ex2 != 0u) locate_ball(ds, 0u, Q, d, t, best, bt, bp);
        return best;
    }
    const float t0 = (float)t - 1e-6f * (1.0f + fabsf((float)t));
    uint32_t stk[kTraceStack];
    float ste[kTraceStack];
    int sp = 0;
    uint32_t node = 0;
    while (true) {
        const float tmax = best == kNone ? 3.0e38f : (float)bt * 1.000001f + 1e-6f;
        const float4 *N = B.nodes + 4 * (size_t)node;
        const float4 l0 = __ldg(N), l1 = __ldg(N + 1), r0 = __ldg(N + 2), r1 = __ldg(N + 3);
        float tl, tr;
        bool hl = slab2(l0, l1, SR, t0, tmax, tl);
        bool hr = slab2(r0, r1, SR, t0, tmax, tr);
        const uint32_t cl = __float_as_uint(l0.w), cr = __float_as_uint(l1.w);
        if (hl && (cl & kLeaf)) {
            const uint32_t b = cl & ~kLeaf;
            if (b != ex1 && b != ex2) locate_ball(ds, b, Q, d, t, best, bt, bp);
            hl = false;
        }
        if (hr && (cr & kLeaf)) {
            const uint32_t b = cr & ~kLeaf;
            if (b != ex1 && b != ex2) locate_ball(ds, b, Q, d, t, best, bt, bp);
            hr = false;
        }
        if (hl && hr) {
            const bool lfirst = tl <= tr;
            if (sp < kTraceStack) {
                stk[sp] = lfirst ? cr : cl;
                ste[sp] = lfirst ? tr : tl;
                ++sp;
            }
            node = lfirst ? cl : cr;
            continue;
        }
        if (hl) {
            node = cl;
            continue;
        }
        if (hr) {
            node = cr;
            continue;
        }
        // pop the next stacked node still in front of the best entry
        const float tcut = best == kNone ? 3.0e38f : (float)bt * 1.000001f + 1e-6f;
        bool found = false;
        while (sp > 0) {
            --sp;
            if (ste[sp] <= tcut) {
                node = stk[sp];
                found = true;
                break;
            }
        }
        if (!found) break;
    }
    return best;
}

template <bool kDipole, int kDetail>
__global__ void __launch_bounds__(256)
k9_trace(DeviceScene ds, CamParams cam, Bvh B, float4 *__restrict__ out,
         unsigned long long *__restrict__ stats)
{
    const int tile = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int tx = tile % cam.tiles_x, ty = tile / cam.tiles_x;
    const int x = tx * kTile + (warp & 1) * 8 + (lane & 7), y = ty * kTile + (warp >> 1) * 4 + (lane >> 3);
    const bool in_image = x < cam.W && y < cam.H;
    double d[3], tn = 0.0;
    bool valid = false;
    ray_dir(cam, x + 0.5, y + 0.5, d, &tn, &valid);
    valid = valid && in_image;
    const double Q[3] = {(double)cam.M[3], (double)cam.M[7], (double)cam.M[11]};
    // slab constants; boxes are widened by pad = 1e-5 (1 + |Q|) so fp32 rounding of the
    // ray never prunes a ball the fp64 leaf test accepts
    SlabRay SR;
    {
        const float pad = 1e-5f * (1.0f + fabsf(cam.M[3]) + fabsf(cam.M[7]) + fabsf(cam.M[11]));
#pragma unroll
        for (int m = 0; m < 3; ++m) {
            const float idm = (float)(1.0 / (d[m] != 0.0 ? d[m] : 1e-30));
            const float q = cam.M[4 * m + 3];
            SR.id[m] = idm;
            const float pid = pad * fabsf(idm), qid = q * idm;
            // (lo - pad - q) id and (hi + pad - q) id for id > 0; swapped roles for id < 0
            // are harmless: slab2 takes min/max of the two
            SR.olo[m] = idm >= 0.0f ? -qid - pid : -qid + pid;
            SR.ohi[m] = idm >= 0.0f ? -qid + pid : -qid - pid;
        }
    }
    Ray R;
    R.dx = __double2float_rn(d[0]);
    R.dy = __double2float_rn(d[1]);
    R.dz = __double2float_rn(d[2]);
    R.ddx = R.ddy = R.ddz = 0.0f;
    R.tnear = __double2float_rn(tn);
    float om[8];
    if (kDetail) sv_axis_weights(ds, R, om);
    float T = 1.0f, Cr = 0.0f, Cg = 0.0f, Cb = 0.0f;
    unsigned long long visited = 0, located = 0, segs = 0, diverged = 0;
    if (valid) {
        double t = tn;
        uint32_t prev = kNone;
        uint32_t c = locate(ds, B, Q, d, SR, t, kNone, kNone);
        ++located;
        int nfail = 0, steps = 0;
        while (c != kNone) {
            if (++steps > kMaxSteps) {
                diverged = 1;
                break;
            }
            const float4 A = __ldg(ds.cellA + c);
            double cc[3];
            cc[0] = __dsub_rn((double)A.x, Q[0]);
            cc[1] = __dsub_rn((double)A.y, Q[1]);
            cc[2] = __dsub_rn((double)A.z, Q[2]);
            const double tc = __fma_rn(d[0], cc[0], __fma_rn(d[1], cc[1], __dmul_rn(d[2], cc[2])));
            const double e0 = __fma_rn(-tc, d[0], cc[0]), e1 = __fma_rn(-tc, d[1], cc[1]),
                         e2 = __fma_rn(-tc, d[2], cc[2]);
            const double rd = (double)A.w;
            const double h = __fma_rn(-e0, e0, __fma_rn(-e1, e1, __fma_rn(-e2, e2, __dmul_rn(rd, rd))));
            Seg g;
            bool ok = h > 0.0;
            const uint2 E = __ldg(ds.cellE + c);
            double tout = t;
            if (ok) {
                const double sq = sqrt(h);
                g.s = __double2float_rn(sq);
                g.tc = __double2float_rn(tc);
                g.ex = __double2float_rn(e0);
                g.ey = __double2float_rn(e1);
                g.ez = __double2float_rn(e2);
                ok = tc + sq > tn;
            }
            if (ok) {
                const float4 none = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
                clip_interval<true, false>(R, ds.edges, E.x, E.y, g, true, none);
                tout = tc + (double)g.hi;
                ok = g.hi > g.lo && tout > t;
            }
            if (!ok) {   // no progress in c: re-locate past it (and its predecessor)
                if (++nfail > 2) t += 1e-6 * (1.0 + fabs(t));
                const uint32_t ex = c;
                c = locate(ds, B, Q, d, SR, t, ex, prev);
                prev = ex;
                ++located;
                continue;
            }
            nfail = 0;
            ++visited;
            // the occupied segment: the walk interval, cut by the dipole / detail face
            Seg o = g;
            float cr, cg, cb;
            {
                const float4 Bc = __ldg(ds.cellB + c);
                cr = Bc.y;
                cg = Bc.z;
                cb = Bc.w;
                if (kDetail) {
                    DetailGeo G;
                    const float4 dpl = detail_plane<kDetail>(ds, c, d, cc, A.w, G);
                    clip_plane<false>(R, dpl, kEndDipole, o);
                    if (o.hi > o.lo)
                        detail_color<kDetail>(ds, c, d, cc,
                                              G.parallel ? (double)__fadd_rn(o.tc, o.lo) : G.ts, om,
                                              cr, cg, cb);
                } else if (kDipole) {
                    const float4 Nn = __ldg(ds.cellN + c);
                    clip_plane<false>(R, make_float4(Nn.x, Nn.y, Nn.z, 0.0f), kEndDipole, o);
                }
                const float dt = __fsub_rn(o.hi, o.lo);
                if (dt > 0.0f) {
                    float alpha;
                    composite_step(Bc.x, dt, cr, cg, cb, T, Cr, Cg, Cb, alpha);
                    ++segs;
                    if (T < kTStop) break;
                }
            }
            t = tout;
            prev = c;
            if (g.hi_q >= 2) {   // plane exit: the face's owner is the next cell
                c = (uint32_t)__ldg(ds.nbr_idx + E.x + (uint32_t)(g.hi_q - 2));
            } else {             // sphere exit: jump the gap in the union of balls
                c = locate(ds, B, Q, d, SR, t, prev, kNone);
                ++located;
            }
        }
    }
    if (in_image) {
        out[(size_t)y * cam.W + x] = make_float4(fmaf(T, ds.bg[0], Cr), fmaf(T, ds.bg[1], Cg),
                                                 fmaf(T, ds.bg[2], Cb), T);
    }
    if (stats) {
        unsigned long long v[5] = {valid ? 1ull : 0ull, visited, located, segs, diverged};
#pragma unroll
        for (int k = 0; k < 5; ++k) {
#pragma unroll
            for (int o2 = 16; o2 > 0; o2 >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o2);
        }
        if (lane == 0)
            for (int k = 0; k < 5; ++k)
                if (v[k]) atomicAdd(stats + k, v[k]);
    }
}

}  // namespace

cudaError_t pack_trace_nodes(pf_scene *s, BallBVH &bvh, DevBuf &nodes, cudaStream_t st)
{
    const int64_t n = bvh.n;
    cudaError_t e = nodes.reserve(sizeof(float4) * 4 * (size_t)(n > 1 ? n - 1 : 1));
    if (e != cudaSuccess) return e;
    if (n > 1) {
        k9_pack_nodes<<<ceil_div(n - 1, 256), 256, 0, st>>>(
            bvh.left.as<uint32_t>(), bvh.right.as<uint32_t>(), bvh.bint.as<Box>(),
            bvh.bleaf.as<Box>(), bvh.order, n, nodes.as<float4>());
        ++s->launches;
    }
    return cudaGetLastError();
}

cudaError_t launch_trace(pf_scene *s, const BallBVH &bvh, const CamParams &cam, float *out,
                         unsigned long long *stats, cudaStream_t st)
{
    const int T = cam.tiles_x * cam.tiles_y;
    Bvh B{s->trace_nodes.as<float4>(), bvh.n};
    if (s->ds.K == 8)
        k9_trace<true, 8><<<T, 256, 0, st>>>(s->ds, cam, B, (float4 *)out, stats);
    else if (s->ds.K)
        k9_trace<true, 1><<<T, 256, 0, st>>>(s->ds, cam, B, (float4 *)out, stats);
    else if (s->ds.cellN)
        k9_trace<true, 0><<<T, 256, 0, st>>>(s->ds, cam, B, (float4 *)out, stats);
    else
        k9_trace<false, 0><<<T, 256, 0, st>>>(s->ds, cam, B, (float4 *)out, stats);
    ++s->launches;
    return cudaGetLastError();
}

}  // namespace pf
