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

struct Bvh {
    const uint32_t *order, *left, *right;
    const Box *bint, *bleaf;
    int64_t n;
};

// slab entry/exit of a box for the fp32 ray (Q, 1/d); the box is widened by
// `pad` so fp32 rounding never prunes a ball the fp64 leaf test would accept
__device__ __forceinline__ bool slab(const Box &b, const float Q[3], const float id[3], float t0,
                                     float t1, float pad, float &tent)
{
    float lo = t0, hi = t1;
#pragma unroll
    for (int m = 0; m < 3; ++m) {
        const float a = (b.lo[m] - pad - Q[m]) * id[m], c = (b.hi[m] + pad - Q[m]) * id[m];
        lo = fmaxf(lo, fminf(a, c));
        hi = fminf(hi, fmaxf(a, c));
    }
    tent = lo;
    return lo <= hi;
}

// the first point of the union of balls at or after t (see the file comment);
// returns the ball / cell, or kNone if the ray leaves every ball
__device__ uint32_t locate(const DeviceScene &ds, const Bvh &B, const double Q[3], const double d[3],
                           const float Qf[3], const float id[3], double t, uint32_t ex1,
                           uint32_t ex2, double scale)
{
    uint32_t best = kNone;
    double bt = 1e300, bp = 0.0;
    const float pad = (float)(1e-5 * scale);
    const float t0 = (float)t - pad;
    uint32_t stack[kTraceStack];
    int sp = 0;
    stack[sp++] = (B.n == 1) ? 1u : 0u;   // (idx << 1) | leaf
    while (sp > 0) {
        const uint32_t nd = stack[--sp];
        const uint32_t idx = nd >> 1;
        const float tmax = best == kNone ? 3.0e38f : (float)bt + pad;
        float te;
        if (nd & 1u) {
            if (!slab(B.bleaf[idx], Qf, id, t0, tmax, pad, te)) continue;
            const uint32_t b = __ldg(B.order + idx);
            if (b == ex1 || b == ex2) continue;
            const float4 A = __ldg(ds.cellA + b);
            const double c0 = (double)A.x - Q[0], c1 = (double)A.y - Q[1], c2 = (double)A.z - Q[2];
            const double tc = d[0] * c0 + d[1] * c1 + d[2] * c2;
            const double e0 = c0 - tc * d[0], e1 = c1 - tc * d[1], e2 = c2 - tc * d[2];
            const double r = (double)A.w;
            const double h = r * r - (e0 * e0 + e1 * e1 + e2 * e2);
            if (!(h > 0.0)) continue;
            const double sq = sqrt(h);
            if (!(tc + sq > t)) continue;
            const double tt = tc - sq > t ? tc - sq : t;
            const double x0 = tt * d[0] - c0, x1 = tt * d[1] - c1, x2 = tt * d[2] - c2;
            const double pw = x0 * x0 + x1 * x1 + x2 * x2 - (double)__ldg(ds.weights + b);
            if (best == kNone || tt < bt || (tt == bt && (pw < bp || (pw == bp && b < best)))) {
                best = b;
                bt = tt;
                bp = pw;
            }
            continue;
        }
        if (!slab(B.bint[idx], Qf, id, t0, tmax, pad, te)) continue;
        if (sp + 2 > kTraceStack) continue;   // depth > 62: cannot happen for n < 2^30
        const uint32_t L = __ldg(B.left + idx), R = __ldg(B.right + idx);
        // visit the nearer child first (pushed last)
        float tl, tr;
        const bool hl = slab((L & 1u) ? B.bleaf[L >> 1] : B.bint[L >> 1], Qf, id, t0, tmax, pad, tl);
        const bool hr = slab((R & 1u) ? B.bleaf[R >> 1] : B.bint[R >> 1], Qf, id, t0, tmax, pad, tr);
        if (hl && hr) {
            if (tl <= tr) {
                stack[sp++] = R;
                stack[sp++] = L;
            } else {
                stack[sp++] = L;
                stack[sp++] = R;
            }
        } else if (hl) {
            stack[sp++] = L;
        } else if (hr) {
            stack[sp++] = R;
        }
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
    const float Qf[3] = {cam.M[3], cam.M[7], cam.M[11]};
    float id[3];
#pragma unroll
    for (int m = 0; m < 3; ++m) id[m] = (float)(1.0 / (d[m] != 0.0 ? d[m] : 1e-30));
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
        const double scale = 1.0 + fabs(Q[0]) + fabs(Q[1]) + fabs(Q[2]);
        uint32_t prev = kNone;
        uint32_t c = locate(ds, B, Q, d, Qf, id, t, kNone, kNone, scale + t);
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
                c = locate(ds, B, Q, d, Qf, id, t, ex, prev, scale + fabs(t));
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
                c = locate(ds, B, Q, d, Qf, id, t, prev, kNone, scale + fabs(t));
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

cudaError_t launch_trace(pf_scene *s, const BallBVH &bvh, const CamParams &cam, float *out,
                         unsigned long long *stats, cudaStream_t st)
{
    const int T = cam.tiles_x * cam.tiles_y;
    Bvh B{bvh.order, bvh.left.as<uint32_t>(), bvh.right.as<uint32_t>(), bvh.bint.as<Box>(),
          bvh.bleaf.as<Box>(), bvh.n};
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
