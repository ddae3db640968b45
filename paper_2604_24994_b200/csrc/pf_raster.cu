// pf_raster.cu -- K6 forward blend, K7 backward replay, K8 gradient unpack.
//
// One CTA per 16x16 tile (256 threads); warp w covers an 8x4 pixel block.
// The tile's sorted cell list is walked in batches of 256 entries: each thread
// stages one cell (record + the tile-centred ray frame computed in fp64,
// SURVEY C18) into shared memory; then every warp walks the batch in lockstep,
// all 32 lanes (pixels) on the same cell:
//   sphere test (a8) -> __any_sync cull -> half-space clipping against the
//   cell's neighbour planes (a9, division free) -> front-to-back compositing
//   (a10) -> warp vote / CTA count early termination.
// The backward (K7) replays the identical walk front to back (bit-identical
// intervals and transmittances, same inlined math with explicit IEEE
// intrinsics), recovers S_k = out_rgb - C_k from the saved final colour, and
// scatters gradients: own-cell terms warp-reduced by shuffles then one float4
// atomic per warp, neighbour terms as float4 atomics.
#include <cuda_runtime.h>
#include <math.h>

#include "pf_internal.cuh"

namespace pf {

namespace {

constexpr int kEndSphere = -1, kEndNear = -2;

struct Ray {
    float dx, dy, dz;      // unit direction
    float ddx, ddy, ddz;   // d - d0 (d0 = the tile-centre direction)
    float tnear;           // near * |d_cam|
};

// pixel ray through the continuous pixel coordinate (u, v) (pixel centre = x + 0.5)
__device__ __forceinline__ void ray_dir(const CamParams &cam, double u, double v, double d[3],
                                        double *tnear)
{
    // explicit IEEE double intrinsics: K6 and K7 must produce bit-identical rays
    double a = __ddiv_rn(__dsub_rn(u, (double)cam.cx), (double)cam.fx);
    double b = __ddiv_rn(__dsub_rn(v, (double)cam.cy), (double)cam.fy);
    double w0 = __dadd_rn(__fma_rn((double)cam.M[0], a, __dmul_rn((double)cam.M[1], b)), (double)cam.M[2]);
    double w1 = __dadd_rn(__fma_rn((double)cam.M[4], a, __dmul_rn((double)cam.M[5], b)), (double)cam.M[6]);
    double w2 = __dadd_rn(__fma_rn((double)cam.M[8], a, __dmul_rn((double)cam.M[9], b)), (double)cam.M[10]);
    double nrm = __dsqrt_rn(__fma_rn(w0, w0, __fma_rn(w1, w1, __dmul_rn(w2, w2))));
    d[0] = __ddiv_rn(w0, nrm);
    d[1] = __ddiv_rn(w1, nrm);
    d[2] = __ddiv_rn(w2, nrm);
    if (tnear)
        *tnear = __dmul_rn((double)cam.near_plane,
                           __dsqrt_rn(__fma_rn(a, a, __fma_rn(b, b, 1.0))));
}

// Staged cell: tile-centred frame t0 = d0.c, e0 = c - t0 d0 (fp64 -> fp32),
// c = p - Q, plus the record.  SoA in shared memory.
struct Stage {
    float t0[256], e0x[256], e0y[256], e0z[256], cx[256], cy[256], cz[256];
    float r[256], sig[256], cr[256], cg[256], cb[256];
    uint32_t eb[256], deg[256], cell[256];
};

__device__ __forceinline__ void stage_cell(Stage &S, int slot, const DeviceScene &ds, uint32_t cell,
                                           const double Q[3], const double d0[3])
{
    float4 A = ds.cellA[cell];
    float4 B = ds.cellB[cell];
    uint2 E = ds.cellE[cell];
    double c0 = __dsub_rn((double)A.x, Q[0]), c1 = __dsub_rn((double)A.y, Q[1]),
           c2 = __dsub_rn((double)A.z, Q[2]);
    double t0 = __fma_rn(d0[0], c0, __fma_rn(d0[1], c1, __dmul_rn(d0[2], c2)));
    S.t0[slot] = __double2float_rn(t0);
    S.e0x[slot] = __double2float_rn(__fma_rn(-t0, d0[0], c0));
    S.e0y[slot] = __double2float_rn(__fma_rn(-t0, d0[1], c1));
    S.e0z[slot] = __double2float_rn(__fma_rn(-t0, d0[2], c2));
    S.cx[slot] = __double2float_rn(c0);
    S.cy[slot] = __double2float_rn(c1);
    S.cz[slot] = __double2float_rn(c2);
    S.r[slot] = A.w;
    S.sig[slot] = B.x;
    S.cr[slot] = B.y;
    S.cg[slot] = B.z;
    S.cb[slot] = B.w;
    S.eb[slot] = E.x;
    S.deg[slot] = E.y;
    S.cell[slot] = cell;
}

// ---- the per-(pixel, cell) math shared verbatim by K6 and K7 -------------

struct Seg {
    float s, tc;           // sphere half-chord, t_c (local frame origin)
    float ex, ey, ez;      // e = c - t_c d  (offset of the centre from the ray)
    float lo_n, lo_d, hi_n, hi_d;   // t'_in = lo_n/lo_d, t'_out = hi_n/hi_d (d > 0)
    int lo_q, hi_q;        // edge index of the binding plane, or kEndSphere / kEndNear
    float dt;              // interval length (0 = empty)
};

// Per-pixel exact ray (fp64) kept in shared memory for the near-tangent path.
struct PixelRays {
    double dx[256], dy[256], dz[256];
};

// a8: ray-sphere test in the local frame: t_c = t0 + delta.c,
// e = e0 - t0 delta - (delta.c) d,  h = r^2 - |e|^2;  hit iff h > 0 and the
// exit t_c + sqrt(h) is beyond t_near.
// Near-tangent rays (|h| < kTangent r^2, ~0.1% of tests) are redone in fp64 from
// the exact ray and the fp32 site: there fp32 loses h (the endpoint derivative
// r/s is singular as s -> 0), and the hit decision and s, e
// come from the fp64 values.  K6 and K7 share this code, so they agree bitwise.
constexpr float kTangent = 1e-3f;

__device__ __forceinline__ bool sphere_hit(const Ray &R, const Stage &S, int j, Seg &g,
                                           const DeviceScene &ds, const CamParams &cam,
                                           const PixelRays &PR)
{
    const float cx = S.cx[j], cy = S.cy[j], cz = S.cz[j], t0 = S.t0[j], r = S.r[j];
    float dc = fmaf(R.ddx, cx, fmaf(R.ddy, cy, __fmul_rn(R.ddz, cz)));
    g.tc = __fadd_rn(t0, dc);
    g.ex = fmaf(-dc, R.dx, fmaf(-t0, R.ddx, S.e0x[j]));
    g.ey = fmaf(-dc, R.dy, fmaf(-t0, R.ddy, S.e0y[j]));
    g.ez = fmaf(-dc, R.dz, fmaf(-t0, R.ddz, S.e0z[j]));
    const float r2 = __fmul_rn(r, r);
    float h = fmaf(-g.ex, g.ex, fmaf(-g.ey, g.ey, fmaf(-g.ez, g.ez, r2)));
    if (fabsf(h) < __fmul_rn(kTangent, r2)) {
        const float4 A = ds.cellA[S.cell[j]];
        const int t = threadIdx.x;
        const double dx = PR.dx[t], dy = PR.dy[t], dz = PR.dz[t];
        const double c0 = __dsub_rn((double)A.x, (double)cam.M[3]);
        const double c1 = __dsub_rn((double)A.y, (double)cam.M[7]);
        const double c2 = __dsub_rn((double)A.z, (double)cam.M[11]);
        const double tcd = __fma_rn(dx, c0, __fma_rn(dy, c1, __dmul_rn(dz, c2)));
        const double e0 = __fma_rn(-tcd, dx, c0), e1 = __fma_rn(-tcd, dy, c1),
                     e2 = __fma_rn(-tcd, dz, c2);
        const double rd = (double)r;
        const double hd = __fma_rn(-e0, e0, __fma_rn(-e1, e1, __fma_rn(-e2, e2, __dmul_rn(rd, rd))));
        g.tc = __double2float_rn(tcd);
        g.ex = __double2float_rn(e0);
        g.ey = __double2float_rn(e1);
        g.ez = __double2float_rn(e2);
        h = (hd > 0.0) ? fmaxf(__double2float_rn(hd), 1e-37f) : -1.0f;
    }
    if (!(h > 0.0f)) return false;
    g.s = __fsqrt_rn(h);
    return __fadd_rn(g.tc, g.s) > R.tnear;
}

// a9: clip the chord [-s, s] by the near plane and by every neighbour's radical
// plane  a t' <= b,  a = d.n, b = k + n.e  (division free: bounds kept as
// fractions with positive denominators; strict comparisons, first binding
// constraint wins -- SURVEY C16).  Returns dt (0 if empty).
__device__ __forceinline__ void clip_interval(const Ray &R, const float4 *__restrict__ edges,
                                              uint32_t eb, uint32_t deg, Seg &g, bool active)
{
    g.lo_n = -g.s;
    g.lo_d = 1.0f;
    g.lo_q = kEndSphere;
    float tnl = __fsub_rn(R.tnear, g.tc);
    if (tnl > g.lo_n) {
        g.lo_n = tnl;
        g.lo_q = kEndNear;
    }
    g.hi_n = g.s;
    g.hi_d = 1.0f;
    g.hi_q = kEndSphere;
    bool empty = false;
#pragma unroll 4
    for (uint32_t q = eb; q < eb + deg; ++q) {
        float4 E = __ldg(edges + q);
        float a = fmaf(R.dx, E.x, fmaf(R.dy, E.y, __fmul_rn(R.dz, E.z)));
        float b = fmaf(E.x, g.ex, fmaf(E.y, g.ey, fmaf(E.z, g.ez, E.w)));
        if (a > 0.0f) {
            if (__fmul_rn(b, g.hi_d) < __fmul_rn(g.hi_n, a)) {
                g.hi_n = b;
                g.hi_d = a;
                g.hi_q = (int)q;
            }
        } else if (a < 0.0f) {
            if (__fmul_rn(-b, g.lo_d) > __fmul_rn(g.lo_n, -a)) {
                g.lo_n = -b;
                g.lo_d = -a;
                g.lo_q = (int)q;
            }
        } else if (b < 0.0f) {
            empty = true;
        }
    }
    float dt = __fsub_rn(__fdiv_rn(g.hi_n, g.hi_d), __fdiv_rn(g.lo_n, g.lo_d));
    g.dt = (active && !empty && dt > 0.0f) ? dt : 0.0f;
}

// a10: one front-to-back compositing step; returns exp(-tau)
__device__ __forceinline__ float composite_step(float sig, float dt, float cr, float cg, float cb,
                                                float &T, float &Cr, float &Cg, float &Cb,
                                                float &alpha)
{
    float tau = __fmul_rn(sig, dt);
    float ex = expf(-tau);
    alpha = __fsub_rn(1.0f, ex);
    float w = __fmul_rn(T, alpha);
    Cr = fmaf(w, cr, Cr);
    Cg = fmaf(w, cg, Cg);
    Cb = fmaf(w, cb, Cb);
    T = __fmul_rn(T, ex);
    return ex;
}

struct PixelSetup {
    int x, y;
    bool valid;
    Ray R;
    double Q[3], d0[3];
};

__device__ __forceinline__ void setup_pixel(const CamParams &cam, int tile, PixelSetup &P,
                                            PixelRays &PR)
{
    const int tx = tile % cam.tiles_x, ty = tile / cam.tiles_x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    P.x = tx * kTile + (warp & 1) * 8 + (lane & 7);
    P.y = ty * kTile + (warp >> 1) * 4 + (lane >> 3);
    P.valid = P.x < cam.W && P.y < cam.H;
    P.Q[0] = cam.M[3];
    P.Q[1] = cam.M[7];
    P.Q[2] = cam.M[11];
    ray_dir(cam, tx * kTile + 8.0, ty * kTile + 8.0, P.d0, nullptr);
    double d[3], tn;
    ray_dir(cam, P.x + 0.5, P.y + 0.5, d, &tn);
    P.R.dx = __double2float_rn(d[0]);
    P.R.dy = __double2float_rn(d[1]);
    P.R.dz = __double2float_rn(d[2]);
    P.R.ddx = __double2float_rn(__dsub_rn(d[0], P.d0[0]));
    P.R.ddy = __double2float_rn(__dsub_rn(d[1], P.d0[1]));
    P.R.ddz = __double2float_rn(__dsub_rn(d[2], P.d0[2]));
    P.R.tnear = __double2float_rn(tn);
    PR.dx[threadIdx.x] = d[0];
    PR.dy[threadIdx.x] = d[1];
    PR.dz[threadIdx.x] = d[2];
}

}  // namespace

// ------------------------------------------------------------------------
// K6 forward
// ------------------------------------------------------------------------
template <bool kCount>
__global__ void __launch_bounds__(256)
k6_forward(DeviceScene ds, CamParams cam, const uint2 *__restrict__ ranges,
           const uint32_t *__restrict__ vals, float4 *__restrict__ out, float4 *__restrict__ saved,
           long long *__restrict__ counters)
{
    __shared__ Stage S;
    __shared__ PixelRays PR;
    const int tile = blockIdx.x;
    PixelSetup P;
    setup_pixel(cam, tile, P, PR);
    const uint2 rg = ranges[tile];
    float T = 1.0f, Cr = 0.0f, Cg = 0.0f, Cb = 0.0f;
    bool done = !P.valid;
    long long xs = 0, xh = 0, xp = 0, xc = 0;
    for (uint32_t base = rg.x; base < rg.y; base += 256) {
        if (__syncthreads_count(!done) == 0) break;
        const int nb = (int)min(256u, rg.y - base);
        if ((int)threadIdx.x < nb) stage_cell(S, threadIdx.x, ds, vals[base + threadIdx.x], P.Q, P.d0);
        __syncthreads();
        for (int j = 0; j < nb; ++j) {
            if (__all_sync(0xffffffffu, done)) break;
            Seg g;
            bool hit = false;
            if (!done) {
                if (kCount) ++xs;
                hit = sphere_hit(P.R, S, j, g, ds, cam, PR);
            }
            if (!__any_sync(0xffffffffu, hit)) continue;
            clip_interval(P.R, ds.edges, S.eb[j], S.deg[j], g, hit);
            if (kCount && hit) {
                ++xh;
                xp += S.deg[j];
            }
            if (g.dt > 0.0f) {
                float alpha;
                composite_step(S.sig[j], g.dt, S.cr[j], S.cg[j], S.cb[j], T, Cr, Cg, Cb, alpha);
                if (kCount) ++xc;
                if (T < kTStop) done = true;
            }
        }
        __syncthreads();
    }
    if (P.valid) {
        float4 o = make_float4(fmaf(T, ds.bg[0], Cr), fmaf(T, ds.bg[1], Cg), fmaf(T, ds.bg[2], Cb), T);
        size_t pix = (size_t)P.y * cam.W + P.x;
        if (out) out[pix] = o;
        if (saved) saved[pix] = o;
        if (kCount) {
            counters[4 * pix + 0] = xs;
            counters[4 * pix + 1] = xh;
            counters[4 * pix + 2] = xp;
            counters[4 * pix + 3] = xc;
        }
    }
}

cudaError_t launch_forward(pf_scene *s, ViewState &v, float *out, int64_t *counters,
                           cudaStream_t st)
{
    int T = v.cam.tiles_x * v.cam.tiles_y;
    cudaEvent_t ev;
    stage_begin(s, 6, st, &ev);
    if (counters)
        k6_forward<true><<<T, 256, 0, st>>>(s->ds, v.cam, v.ranges.as<uint2>(), v.vals.as<uint32_t>(),
                                            (float4 *)out, v.saved.as<float4>(),
                                            (long long *)counters);
    else
        k6_forward<false><<<T, 256, 0, st>>>(s->ds, v.cam, v.ranges.as<uint2>(),
                                             v.vals.as<uint32_t>(), (float4 *)out,
                                             v.saved.as<float4>(), nullptr);
    ++s->launches;
    stage_end(s, 6, st, ev);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------
// K7 backward
// ------------------------------------------------------------------------
namespace {

__device__ __forceinline__ float warp_sum(float v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// d t_end / d theta times  w = +-dL/ddt  for one interval end:
//   sphere end at t' = +-s:  dt/dp_i = (t' d - e)/t',  dt/dr = r/t'
//   plane end (i,j), a = d.n: dt/dp_i = (t' d - e)/a, dt/dp_j = (n - t' d + e)/a,
//                             dt/dw_i = 1/(2a), dt/dw_j = -1/(2a)
//   near end: 0
struct OwnGrad {
    float px, py, pz, w, r;
};

__device__ __forceinline__ void end_grad(const Ray &R, const Seg &g, int q, float tprime, float a,
                                         float wgt, float rad, const float4 *__restrict__ edges,
                                         const int32_t *__restrict__ nbr, float4 *accA, OwnGrad &o)
{
    if (q == kEndNear) return;
    float xpx = fmaf(tprime, R.dx, -g.ex), xpy = fmaf(tprime, R.dy, -g.ey),
          xpz = fmaf(tprime, R.dz, -g.ez);   // x* - p_i
    if (q == kEndSphere) {
        float f = __fdiv_rn(wgt, tprime);
        o.px = fmaf(f, xpx, o.px);
        o.py = fmaf(f, xpy, o.py);
        o.pz = fmaf(f, xpz, o.pz);
        o.r = fmaf(f, rad, o.r);
        return;
    }
    float f = __fdiv_rn(wgt, a);
    o.px = fmaf(f, xpx, o.px);
    o.py = fmaf(f, xpy, o.py);
    o.pz = fmaf(f, xpz, o.pz);
    o.w = fmaf(0.5f, f, o.w);
    float4 E = __ldg(edges + q);
    int j = __ldg(nbr + q);
    float4 gj = make_float4(f * (E.x - xpx), f * (E.y - xpy), f * (E.z - xpz), -0.5f * f);
    atomicAdd(accA + j, gj);
}

}  // namespace

__global__ void __launch_bounds__(256)
k7_backward(DeviceScene ds, CamParams cam, const uint2 *__restrict__ ranges,
            const uint32_t *__restrict__ vals, const float4 *__restrict__ saved,
            const float4 *__restrict__ grad_out, float4 *__restrict__ accA,
            float4 *__restrict__ accB, float *__restrict__ accC)
{
    __shared__ Stage S;
    __shared__ PixelRays PR;
    const int tile = blockIdx.x;
    const int lane = threadIdx.x & 31;
    PixelSetup P;
    setup_pixel(cam, tile, P, PR);
    const uint2 rg = ranges[tile];
    float T = 1.0f, Cr = 0.0f, Cg = 0.0f, Cb = 0.0f;
    bool done = !P.valid;
    float4 fin = make_float4(0, 0, 0, 1), G = make_float4(0, 0, 0, 0);
    if (P.valid) {
        size_t pix = (size_t)P.y * cam.W + P.x;
        fin = saved[pix];
        G = grad_out[pix];
    }
    const float GT_Tfin = __fmul_rn(G.w, fin.w);
    for (uint32_t base = rg.x; base < rg.y; base += 256) {
        if (__syncthreads_count(!done) == 0) break;
        const int nb = (int)min(256u, rg.y - base);
        if ((int)threadIdx.x < nb) stage_cell(S, threadIdx.x, ds, vals[base + threadIdx.x], P.Q, P.d0);
        __syncthreads();
        for (int j = 0; j < nb; ++j) {
            if (__all_sync(0xffffffffu, done)) break;
            Seg g;
            bool hit = false;
            if (!done) hit = sphere_hit(P.R, S, j, g, ds, cam, PR);
            if (!__any_sync(0xffffffffu, hit)) continue;
            clip_interval(P.R, ds.edges, S.eb[j], S.deg[j], g, hit);
            bool seg = g.dt > 0.0f;
            if (!__any_sync(0xffffffffu, seg)) continue;
            OwnGrad o = {0, 0, 0, 0, 0};
            float gs = 0.0f, gR = 0.0f, gG = 0.0f, gB = 0.0f;
            if (seg) {
                const float sig = S.sig[j], cr = S.cr[j], cg = S.cg[j], cb = S.cb[j];
                float Tk = T, alpha;
                composite_step(sig, g.dt, cr, cg, cb, T, Cr, Cg, Cb, alpha);
                // T is now T_{k+1}; C is C_k; S_k = out_rgb - C_k
                float Sr = __fsub_rn(fin.x, Cr), Sg = __fsub_rn(fin.y, Cg), Sb = __fsub_rn(fin.z, Cb);
                float dtau = -GT_Tfin;
                dtau = fmaf(G.x, fmaf(T, cr, -Sr), dtau);
                dtau = fmaf(G.y, fmaf(T, cg, -Sg), dtau);
                dtau = fmaf(G.z, fmaf(T, cb, -Sb), dtau);
                float wa = __fmul_rn(Tk, alpha);
                gR = wa * G.x;
                gG = wa * G.y;
                gB = wa * G.z;
                gs = dtau * g.dt;
                float gdt = dtau * sig;
                if (gdt != 0.0f) {
                    const float rad = S.r[j];
                    float tout = __fdiv_rn(g.hi_n, g.hi_d), tin = __fdiv_rn(g.lo_n, g.lo_d);
                    end_grad(P.R, g, g.hi_q, tout, g.hi_d, gdt, rad, ds.edges, ds.nbr_idx, accA, o);
                    end_grad(P.R, g, g.lo_q, tin, -g.lo_d, -gdt, rad, ds.edges, ds.nbr_idx, accA, o);
                }
                if (T < kTStop) done = true;
            }
            // own-cell terms: warp reduction, one lane issues the atomics
            float v0 = warp_sum(o.px), v1 = warp_sum(o.py), v2 = warp_sum(o.pz), v3 = warp_sum(o.w);
            float v4 = warp_sum(o.r), v5 = warp_sum(gs), v6 = warp_sum(gR), v7 = warp_sum(gG);
            float v8 = warp_sum(gB);
            if (lane == 0) {
                uint32_t cell = S.cell[j];
                atomicAdd(accA + cell, make_float4(v0, v1, v2, v3));
                atomicAdd(accB + cell, make_float4(v4, v5, v6, v7));
                atomicAdd(accC + cell, v8);
            }
        }
        __syncthreads();
    }
}

cudaError_t launch_backward(pf_scene *s, ViewState &v, const float *grad_out, cudaStream_t st)
{
    int T = v.cam.tiles_x * v.cam.tiles_y;
    int64_t N = s->ds.N;
    float4 *accA = s->acc.as<float4>();
    float4 *accB = accA + N;
    float *accC = reinterpret_cast<float *>(accB + N);
    cudaEvent_t ev;
    stage_begin(s, 7, st, &ev);
    k7_backward<<<T, 256, 0, st>>>(s->ds, v.cam, v.ranges.as<uint2>(), v.vals.as<uint32_t>(),
                                   v.saved.as<float4>(), (const float4 *)grad_out, accA, accB, accC);
    ++s->launches;
    stage_end(s, 7, st, ev);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------
// K8: add the packed accumulators into the caller's arrays (+=)
// ------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
k8_unpack(int64_t N, const float4 *__restrict__ accA, const float4 *__restrict__ accB,
          const float *__restrict__ accC, float *gs, float *gw, float *gr, float *gd, float *gc)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    float4 a = accA[i], b = accB[i];
    float c = accC[i];
    gs[3 * i + 0] += a.x;
    gs[3 * i + 1] += a.y;
    gs[3 * i + 2] += a.z;
    gw[i] += a.w;
    gr[i] += b.x;
    gd[i] += b.y;
    gc[3 * i + 0] += b.z;
    gc[3 * i + 1] += b.w;
    gc[3 * i + 2] += c;
}

cudaError_t launch_unpack(pf_scene *s, float *gs, float *gw, float *gr, float *gd, float *gc,
                          cudaStream_t st)
{
    int64_t N = s->ds.N;
    float4 *accA = s->acc.as<float4>();
    float4 *accB = accA + N;
    float *accC = reinterpret_cast<float *>(accB + N);
    cudaEvent_t ev;
    stage_begin(s, 8, st, &ev);
    k8_unpack<<<ceil_div(N, 256), 256, 0, st>>>(N, accA, accB, accC, gs, gw, gr, gd, gc);
    ++s->launches;
    stage_end(s, 8, st, ev);
    return cudaGetLastError();
}

}  // namespace pf
