// pf_pixel.cuh -- per-pixel device math of the hot path, shared by K6/K7
// (pf_raster.cu) and the NEXT-4 tracer (pf_trace.cu): pixel rays, the warp
// stage / cone cull, the ray-sphere test (a8), radical-plane clipping (a9),
// the warp plane cull, compositing (a10), the detail-site geometry (NEXT-2) and
// the K6 -> K7 record codes.  Internal linkage: every including TU gets its own
// copy, so K6, K7 and the tracer evaluate the identical instruction sequences.
#pragma once

#include <cuda_runtime.h>
#include <math.h>
#include <stdlib.h>

#include "pf_internal.cuh"

#ifndef PF_RAY_FAST   // pixel rays without fp64 divides (ray_dir)
#define PF_RAY_FAST 1
#endif
#ifndef PF_K6_POSTRACK   // K6 kept-plane loop: track kept positions, map to list indices once
                         // (measured: recording K6 11.71 -> 11.22 ms per 8 train8_1m views)
#define PF_K6_POSTRACK 1
#endif
#ifndef PF_PREDTRACK   // tracked plane clip (K6 recording, K7): predicated moves, not min/max
                       // (measured: recording K6 11.23 -> 10.90 ms per 8 train8_1m views)
#define PF_PREDTRACK 1
#endif
#ifndef PF_K6_KEPT_UNROLL4   // (with PF_K6_POSTRACK) kept-plane loop unrolled by 4
#define PF_K6_KEPT_UNROLL4 0
#endif

namespace pf {

namespace {

// binding-constraint codes (tracked by K6/K7, stored in the K6 -> K7 records):
// 0 sphere, 1 near plane, 2 + k the cell's k-th neighbour plane, kEndDipole the
// dipole face (NEXT-1)
constexpr int kEndSphere = 0, kEndNear = 1, kEndDipole = 0x1000;

struct Ray {
    float dx, dy, dz;      // unit direction
    float ddx, ddy, ddz;   // d - d0 (d0 = the tile-centre direction)
    float tnear;           // near * |d_cam|
};

// pixel ray through the continuous pixel coordinate (u, v) (pixel centre = x + 0.5).
// Pinhole: d = normalize(R (a, b, 1)), t_near = near |(a, b, 1)|.  Equidistant
// fisheye (NEXT-4): d = R (sin(th) a/th, sin(th) b/th, cos(th)), th = |(a, b)|,
// t_near = near; *valid = false outside the image circle (th > pi).
__device__ __forceinline__ void ray_dir(const CamParams &cam, double u, double v, double d[3],
                                        double *tnear, bool *valid = nullptr)
{
    // explicit IEEE double intrinsics: K6 and K7 must produce bit-identical rays
    // (multiplications by the host's 1/f and one rsqrt instead of fp64 divides:
    // the ray differs from the exact one by a few fp64 ulps, far below fp32)
#if PF_RAY_FAST
    double a = __dmul_rn(__dsub_rn(u, (double)cam.cx), cam.ifx);
    double b = __dmul_rn(__dsub_rn(v, (double)cam.cy), cam.ify);
#else
    double a = __ddiv_rn(__dsub_rn(u, (double)cam.cx), (double)cam.fx);
    double b = __ddiv_rn(__dsub_rn(v, (double)cam.cy), (double)cam.fy);
#endif
    double c = 1.0;
    if (cam.model == PF_FISHEYE) {
        const double th = __dsqrt_rn(__fma_rn(a, a, __dmul_rn(b, b)));
        if (valid) *valid = th <= 3.14159265358979323846;
        if (th > 0.0) {
            double sn, cs;
            sincos(th, &sn, &cs);
            const double f = __ddiv_rn(sn, th);
            a = __dmul_rn(f, a);
            b = __dmul_rn(f, b);
            c = cs;
        } else {
            a = b = 0.0;
        }
    } else if (valid) {
        *valid = true;
    }
    double w0 = __fma_rn((double)cam.M[2], c, __fma_rn((double)cam.M[0], a, __dmul_rn((double)cam.M[1], b)));
    double w1 = __fma_rn((double)cam.M[6], c, __fma_rn((double)cam.M[4], a, __dmul_rn((double)cam.M[5], b)));
    double w2 = __fma_rn((double)cam.M[10], c, __fma_rn((double)cam.M[8], a, __dmul_rn((double)cam.M[9], b)));
#if PF_RAY_FAST
    const double inrm = rsqrt(__fma_rn(w0, w0, __fma_rn(w1, w1, __dmul_rn(w2, w2))));
    d[0] = __dmul_rn(w0, inrm);
    d[1] = __dmul_rn(w1, inrm);
    d[2] = __dmul_rn(w2, inrm);
#else
    double nrm = __dsqrt_rn(__fma_rn(w0, w0, __fma_rn(w1, w1, __dmul_rn(w2, w2))));
    d[0] = __ddiv_rn(w0, nrm);
    d[1] = __ddiv_rn(w1, nrm);
    d[2] = __ddiv_rn(w2, nrm);
#endif
    if (tnear)
        *tnear = cam.model == PF_FISHEYE
                     ? (double)cam.near_plane
                     : __dmul_rn((double)cam.near_plane, __dsqrt_rn(__fma_rn(a, a, __fma_rn(b, b, 1.0))));
}

// ---------------------------------------------------------------------------
// Per-warp state.  Warp w of the tile's CTA owns an 8x4 pixel block and walks
// the tile's sorted list on its own (no CTA barriers): 32 list entries at a
// time, one per lane, are culled against the warp's ray cone (fp64, exact
// conservative test), and the survivors are staged in the warp's shared-memory
// slots with the warp-centred ray frame t0 = d_w.c, e0 = c - t0 d_w (fp64 ->
// fp32, SURVEY C18 applied per warp block instead of per tile).
// ---------------------------------------------------------------------------
constexpr int kWarps = 8;

struct WarpStage {
    float t0[32], e0x[32], e0y[32], e0z[32], cx[32], cy[32], cz[32], r[32];
    float sig[32], cr[32], cg[32], cb[32];
    float4 *nrm;                    // dipole normals (NEXT-1) of the slots: separate smem, or null
    uint32_t eb[32], deg[32], cell[32];
    float smax[32], rhom[32];       // K6 plane cull: chord bound and rho + M/|n| (cull_planes)
};

// Per-pixel exact ray (fp64), read only by the near-tangent path.
struct PixelRays {
    double dx[256], dy[256], dz[256];
};

struct WarpCtx {           // one per warp, in shared memory
    double wx, wy, wz;     // warp-centre direction d_w
    double cos_t, sin_t;   // half-angle of the cone containing the warp's pixel rays
    float fwx, fwy, fwz;   // d_w rounded to fp32 (plane cull)
    float tan_t;           // tan of the half-angle, rounded up (plane cull)
};

// ---- the per-(pixel, cell) math shared verbatim by K6 and K7 -------------

struct Seg {
    float s, tc;           // sphere half-chord, t_c (local frame origin)
    float ex, ey, ez;      // e = c - t_c d  (offset of the centre from the ray)
    float lo, hi;          // t'_in, t'_out (local frame)
    int lo_q, hi_q;        // binding constraint code (kEnd*, or 2 + local plane index)
    float dt;              // interval length (0 = empty)
};

__device__ __forceinline__ float rcp_approx(float x)
{
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// a8: ray-sphere test in the local frame: t_c = t0 + delta.c,
// e = e0 - t0 delta - (delta.c) d,  h = r^2 - |e|^2;  hit iff h > 0 and the
// exit t_c + sqrt(h) is beyond t_near.
// Near-tangent rays (|h| < kTangent r^2, ~0.1% of tests) are redone in fp64 from
// the exact ray and the fp32 site: there fp32 loses h (the endpoint derivative
// r/s is singular as s -> 0), and the hit decision and s, e
// come from the fp64 values.  K6 and K7 share this code, so they agree bitwise.
constexpr float kTangent = 1e-3f;

__device__ __forceinline__ bool sphere_hit(const Ray &R, const WarpStage &S, int j, Seg &g,
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
        h = (hd > 0.0) ? fmaxf(__double2float_rn(hd), 1e-30f) : -1.0f;
    }
    if (!(h > 0.0f)) return false;
    g.s = __fmul_rn(h, rsqrtf(h));
    return __fadd_rn(g.tc, g.s) > R.tnear;
}

// one radical plane  a t' <= b,  a = d.n, b = k + n.e:  t = b/a bounds t' from
// above if a > 0, from below if a < 0; a == +0 with b < 0 empties the interval
// (rcp(+0) = +inf, so t = -inf lands on the upper bound).  K6 and K7
// evaluate the identical instruction sequence (min/max of the same values), K7
// additionally records which constraint binds (strict: the first one wins,
// SURVEY C16).
template <bool kTrack>
__device__ __forceinline__ void clip_plane(const Ray &R, const float4 E, int q, Seg &g)
{
    const float a = fmaf(R.dx, E.x, fmaf(R.dy, E.y, __fmul_rn(R.dz, E.z)));
    const float b = fmaf(E.x, g.ex, fmaf(E.y, g.ey, fmaf(E.z, g.ez, E.w)));
    const float t = __fmul_rn(b, rcp_approx(a));
    const bool up = a >= 0.0f;
    if (kTrack && PF_PREDTRACK) {
        // the bound moves iff t is strictly inside it (a NaN t never moves it, as
        // fminf/fmaxf ignore it); only the sign of a zero bound can differ from the
        // min/max form below, which leaves dt = hi - lo and the codes unchanged
        const bool ch = up && t < g.hi, cl = !up && t > g.lo;
        g.hi = ch ? t : g.hi;
        g.hi_q = ch ? q : g.hi_q;
        g.lo = cl ? t : g.lo;
        g.lo_q = cl ? q : g.lo_q;
        return;
    }
    const float th = up ? t : __int_as_float(0x7f800000);
    const float tl = up ? __int_as_float(0xff800000) : t;
    const float nh = fminf(g.hi, th), nl = fmaxf(g.lo, tl);
    if (kTrack) {
        g.hi_q = (nh != g.hi) ? q : g.hi_q;
        g.lo_q = (nl != g.lo) ? q : g.lo_q;
    }
    g.hi = nh;
    g.lo = nl;
}

// a9: clip the chord [-s, s] by the near plane and every neighbour's radical
// plane (P:228, P:577-585 with the weight sign of SURVEY C1).
template <bool kTrack, bool kDipole>
__device__ __forceinline__ void clip_interval(const Ray &R, const float4 *__restrict__ edges,
                                              uint32_t eb, uint32_t deg, Seg &g, bool active,
                                              const float4 &dplane)
{
    g.lo = -g.s;
    g.lo_q = kEndSphere;
    const float tnl = __fsub_rn(R.tnear, g.tc);
    if (tnl > g.lo) {
        g.lo = tnl;
        g.lo_q = kEndNear;
    }
    g.hi = g.s;
    g.hi_q = kEndSphere;
    const float4 *ep = edges + eb;
    uint32_t k = 0;
    for (; k + 4 <= deg; k += 4) {
        const float4 E0 = __ldg(ep + k), E1 = __ldg(ep + k + 1), E2 = __ldg(ep + k + 2),
                     E3 = __ldg(ep + k + 3);
        clip_plane<kTrack>(R, E0, (int)k + 2, g);
        clip_plane<kTrack>(R, E1, (int)k + 3, g);
        clip_plane<kTrack>(R, E2, (int)k + 4, g);
        clip_plane<kTrack>(R, E3, (int)k + 5, g);
    }
    if (k < deg) {   // 1..3 left (deg is warp-uniform: these branches do not diverge)
        const float4 E0 = __ldg(ep + k);
        const float4 E1 = k + 1 < deg ? __ldg(ep + k + 1) : E0;
        const float4 E2 = k + 2 < deg ? __ldg(ep + k + 2) : E0;
        clip_plane<kTrack>(R, E0, (int)k + 2, g);
        if (k + 1 < deg) clip_plane<kTrack>(R, E1, (int)k + 3, g);
        if (k + 2 < deg) clip_plane<kTrack>(R, E2, (int)k + 4, g);
    }
    if (kDipole)  // the occupied half (x - p_i).n_i <= k: the dipole face (k = 0) or the
        clip_plane<kTrack>(R, dplane, kEndDipole, g);   // displaced detail face (k = delta)
    const float dt = __fsub_rn(g.hi, g.lo);
    g.dt = (active && dt > 0.0f) ? dt : 0.0f;
}

// ---------------------------------------------------------------------------
// Warp-level plane cull (K6).  All rays of the warp lie in the cone (d_w, th),
// so every chord point x of cell i seen by the warp lies in the cylinder
//   x - p_i = t' d_w - e0 + v,   |t'| <= s_max,  v _|_ d_w,  |v| <= rho,
//   rho = (t0 + r) tan(th),  s_max = sqrt(r^2 - max(0, |e0| - rho)^2)
// (axial coordinate of a ball point <= t0 + r; radial <= axial tan(th)).  On it
// the plane function f = a t' - b of neighbour j (a = d.n, b = k + n.e; the
// cell keeps f <= 0) ranges within  -b_w +- (|d_w.n| s_max + rho |n|)  with
// b_w = k + n.e0.  After a hit, lane k tests plane k of the cell at once:
//   sup f < -M  : plane k cannot bind for any pixel of the warp -> dropped
//                 (fminf/fmaxf with a strictly non-binding value is the identity,
//                 so the interval is bit-identical to clipping by every plane);
//   inf f >  M  : the warp's beam through B_i lies in j's cell: every pixel's
//                 interval is empty -> the whole cell is skipped.
// The ball radius is inflated by 1e-5 (|t0| + |e0| + r) and M = 1e-5 (|k| +
// |n| (|e0| + r + |t0|)) so fp32 rounding of the staged frame, the lanes' own
// rounding and the fp64 near-tangent path (exact centre) are all covered.
// ---------------------------------------------------------------------------
__device__ __forceinline__ float sqrt_apx(float x)   // sqrt.approx (rel. error ~1e-7)
{
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

struct PlaneBuf {
    float4 E[32];          // kept edge records (n, k) of the current cell
    uint8_t q[32];         // their index in the cell's neighbour list
};

// Per-slot constants of the plane cull, computed by the staging lane.
__device__ __forceinline__ void cull_consts(WarpStage &S, int slot, const WarpCtx &W)
{
    const float t0 = S.t0[slot], ex = S.e0x[slot], ey = S.e0y[slot], ez = S.e0z[slot];
    const float en = sqrt_apx(fmaf(ex, ex, fmaf(ey, ey, ez * ez)));
    const float r = S.r[slot] + 1e-5f * (fabsf(t0) + en + S.r[slot]);
    const float rho = fmaxf(t0 + r, 0.0f) * W.tan_t * 1.00001f;
    const float off = fmaxf(en - rho - 1e-5f * (en + rho), 0.0f);
    S.smax[slot] = sqrt_apx(fmaxf(r - off, 0.0f) * (r + off)) * 1.00001f;
    S.rhom[slot] = fmaf(1e-5f, en + r + fabsf(t0), rho);   // rho + M / |n| (see above)
}

// Lane k tests plane k of slot j (deg <= 32) and the kept planes are compacted
// into B in list order.  Returns -1 if every pixel's interval is empty, else the
// number of kept planes.
__device__ __forceinline__ int cull_planes(const WarpStage &S, int j, const WarpCtx &W,
                                           const float4 *__restrict__ edges, PlaneBuf &B, int lane)
{
    const uint32_t deg = S.deg[j];
    const float ex = S.e0x[j], ey = S.e0y[j], ez = S.e0z[j], smax = S.smax[j], rhom = S.rhom[j];
    bool keep = false, kill = false;
    float4 E = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    if ((uint32_t)lane < deg) {
        E = __ldg(edges + S.eb[j] + lane);
        const float aw = fmaf(W.fwx, E.x, fmaf(W.fwy, E.y, W.fwz * E.z));
        const float bw = fmaf(E.x, ex, fmaf(E.y, ey, fmaf(E.z, ez, E.w)));
        const float nn = sqrt_apx(fmaf(E.x, E.x, fmaf(E.y, E.y, E.z * E.z)));
        const float thr = fmaf(fabsf(aw), smax, fmaf(nn, rhom, 1e-5f * fabsf(E.w)));
        keep = bw <= thr;
        kill = bw < -thr;
    }
    if (__any_sync(0xffffffffu, kill)) return -1;
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    const int n = __popc(m);
    __syncwarp();   // every lane's reads of the previous cell's kept planes happen before
    if (keep) {     // this cell's planes overwrite them (racecheck: WAR across lanes)
        const int p = __popc(m & ((1u << lane) - 1u));
        B.E[p] = E;
        B.q[p] = (uint8_t)lane;
    }
    __syncwarp();
    return n;
}

// a9 over the planes kept by cull_planes (same per-plane math and order as
// clip_interval; the tracked code is 2 + the plane's list index)
template <bool kTrack, bool kDipole>
__device__ __forceinline__ void clip_interval_kept(const Ray &R, const PlaneBuf &B, int n, Seg &g,
                                                   bool active, const float4 &dplane)
{
    g.lo = -g.s;
    g.lo_q = kEndSphere;
    const float tnl = __fsub_rn(R.tnear, g.tc);
    if (tnl > g.lo) {
        g.lo = tnl;
        g.lo_q = kEndNear;
    }
    g.hi = g.s;
    g.hi_q = kEndSphere;
    int k = 0;
#if PF_K6_POSTRACK
    // track 2 + the kept position, mapped to 2 + the list index once at the end
    // (the same binding plane: positions are increasing in list order)
#if PF_K6_KEPT_UNROLL4
    for (; k + 4 <= n; k += 4) {
        const float4 E0 = B.E[k], E1 = B.E[k + 1], E2 = B.E[k + 2], E3 = B.E[k + 3];
        clip_plane<kTrack>(R, E0, k + 2, g);
        clip_plane<kTrack>(R, E1, k + 3, g);
        clip_plane<kTrack>(R, E2, k + 4, g);
        clip_plane<kTrack>(R, E3, k + 5, g);
    }
    if (k + 2 <= n) {
        const float4 E0 = B.E[k], E1 = B.E[k + 1];
        clip_plane<kTrack>(R, E0, k + 2, g);
        clip_plane<kTrack>(R, E1, k + 3, g);
        k += 2;
    }
#else
    for (; k + 2 <= n; k += 2) {
        const float4 E0 = B.E[k], E1 = B.E[k + 1];
        clip_plane<kTrack>(R, E0, k + 2, g);
        clip_plane<kTrack>(R, E1, k + 3, g);
    }
#endif
    if (k < n) clip_plane<kTrack>(R, B.E[k], k + 2, g);
    if (kTrack) {
        if (g.hi_q >= 2) g.hi_q = (int)B.q[g.hi_q - 2] + 2;
        if (g.lo_q >= 2) g.lo_q = (int)B.q[g.lo_q - 2] + 2;
    }
#else
    for (; k + 2 <= n; k += 2) {
        const float4 E0 = B.E[k], E1 = B.E[k + 1];
        const uint32_t qq = kTrack ? *reinterpret_cast<const uint16_t *>(B.q + k) : 0u;
        clip_plane<kTrack>(R, E0, (int)(qq & 0xffu) + 2, g);
        clip_plane<kTrack>(R, E1, (int)(qq >> 8) + 2, g);
    }
    if (k < n) clip_plane<kTrack>(R, B.E[k], kTrack ? (int)B.q[k] + 2 : 0, g);
#endif
    if (kDipole) clip_plane<kTrack>(R, dplane, kEndDipole, g);
    const float dt = __fsub_rn(g.hi, g.lo);
    g.dt = (active && dt > 0.0f) ? dt : 0.0f;
}

// a10: one front-to-back compositing step (alpha = 1 - exp(-sigma dt))
__device__ __forceinline__ void composite_step(float sig, float dt, float cr, float cg, float cb,
                                               float &T, float &Cr, float &Cg, float &Cb,
                                               float &alpha)
{
    const float tau = __fmul_rn(sig, dt);
    const float ex = __expf(-tau);
    alpha = __fsub_rn(1.0f, ex);
    const float w = __fmul_rn(T, alpha);
    Cr = fmaf(w, cr, Cr);
    Cg = fmaf(w, cg, Cg);
    Cb = fmaf(w, cb, Cb);
    T = __fmul_rn(T, ex);
}

// the ViewArgs of this CTA's view into shared memory (fused multi-view launches)
__device__ __forceinline__ void load_view_args(const ViewArgs *__restrict__ va, int T, ViewArgs &VA)
{
    static_assert(sizeof(ViewArgs) % 4 == 0 && sizeof(ViewArgs) <= 4 * 256, "ViewArgs");
    const uint32_t *src = reinterpret_cast<const uint32_t *>(va + blockIdx.x / (unsigned)T);
    if (threadIdx.x < sizeof(ViewArgs) / 4)
        reinterpret_cast<uint32_t *>(&VA)[threadIdx.x] = __ldg(src + threadIdx.x);
    __syncthreads();
}

struct PixelSetup {
    int x, y;
    bool in_image;   // inside the W x H image (gets an output)
    bool valid;      // and has a ray (fisheye: inside the image circle)
    Ray R;
};

// pixel ray, warp cone and warp frame.  Every lane of a warp runs this.
__device__ __forceinline__ void setup_pixel(const CamParams &cam, int tile, PixelSetup &P,
                                            PixelRays &PR, WarpCtx &W)
{
    const int tx = tile % cam.tiles_x, ty = tile / cam.tiles_x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int x0 = tx * kTile + (warp & 1) * 8, y0 = ty * kTile + (warp >> 1) * 4;
    P.x = x0 + (lane & 7);
    P.y = y0 + (lane >> 3);
    P.in_image = P.x < cam.W && P.y < cam.H;
    P.valid = P.in_image;
    double dw[3];
    ray_dir(cam, x0 + 4.0, y0 + 2.0, dw, nullptr);
    // cone half-angle.  Pinhole: the largest angle to the four corner pixel rays
    // (the angle to d_w is quasi-convex over the image plane, so corners bound it).
    // Fisheye: the (a, b) -> ray map is 1-Lipschitz in angle, so the largest
    // (a, b) distance to a corner pixel centre bounds it.
    const int cxo = (lane & 1) ? 7 : 0, cyo = (lane & 2) ? 3 : 0;
    double cs;
    if (cam.model == PF_FISHEYE) {
        const double da = (cxo + 0.5 - 4.0) / (double)cam.fx, db = (cyo + 0.5 - 2.0) / (double)cam.fy;
        cs = cos(fmin(sqrt(da * da + db * db) * 1.000001 + 1e-9, 3.14159265358979323846));
    } else {
        double dcn[3];
        ray_dir(cam, x0 + cxo + 0.5, y0 + cyo + 0.5, dcn, nullptr);
        cs = __fma_rn(dw[0], dcn[0], __fma_rn(dw[1], dcn[1], __dmul_rn(dw[2], dcn[2])));
    }
    cs = fmin(cs, __shfl_xor_sync(0xffffffffu, cs, 1));
    cs = fmin(cs, __shfl_xor_sync(0xffffffffu, cs, 2));
    cs = fmin(cs, 1.0);
    if (lane == 0) {
        W.wx = dw[0];
        W.wy = dw[1];
        W.wz = dw[2];
        W.cos_t = cs;
        W.sin_t = sqrt(fmax(0.0, 1.0 - cs * cs));
        W.fwx = (float)dw[0];
        W.fwy = (float)dw[1];
        W.fwz = (float)dw[2];
        W.tan_t = (float)(W.sin_t / fmax(cs, 1e-3) * (1.0 + 1e-6));
    }
    double d[3], tn;
    bool in_circle;
    ray_dir(cam, P.x + 0.5, P.y + 0.5, d, &tn, &in_circle);
    P.valid = P.valid && in_circle;
    P.R.dx = __double2float_rn(d[0]);
    P.R.dy = __double2float_rn(d[1]);
    P.R.dz = __double2float_rn(d[2]);
    P.R.ddx = __double2float_rn(__dsub_rn(d[0], dw[0]));
    P.R.ddy = __double2float_rn(__dsub_rn(d[1], dw[1]));
    P.R.ddz = __double2float_rn(__dsub_rn(d[2], dw[2]));
    P.R.tnear = __double2float_rn(tn);
    PR.dx[threadIdx.x] = d[0];
    PR.dy[threadIdx.x] = d[1];
    PR.dz[threadIdx.x] = d[2];
    __syncwarp();
}

// Stage cell `cell` into slot `slot` with the warp-centred frame (fp64 -> fp32).
template <bool kDipole>
__device__ __forceinline__ void stage_slot(WarpStage &S, int slot, const DeviceScene &ds,
                                           uint32_t cell, const float4 A, double c0, double c1,
                                           double c2, double t, const WarpCtx &W)
{
    const float4 B = __ldg(ds.cellB + cell);
    const uint2 E = __ldg(ds.cellE + cell);
    S.t0[slot] = __double2float_rn(t);
    S.e0x[slot] = __double2float_rn(__fma_rn(-t, W.wx, c0));
    S.e0y[slot] = __double2float_rn(__fma_rn(-t, W.wy, c1));
    S.e0z[slot] = __double2float_rn(__fma_rn(-t, W.wz, c2));
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
    if (kDipole) {
        const float4 Nn = __ldg(ds.cellN + cell);
        S.nrm[slot] = make_float4(Nn.x, Nn.y, Nn.z, 0.0f);
    }
    // pull the cell's edge records towards L1 while the warp walks earlier cells
    if (E.y) {
        const float4 *ep = ds.edges + E.x;
        asm volatile("prefetch.global.L1 [%0];" ::"l"(ep));
        asm volatile("prefetch.global.L1 [%0];" ::"l"(ep + (E.y - 1)));
        if (E.y > 8) asm volatile("prefetch.global.L1 [%0];" ::"l"(ep + (E.y >> 1)));
    }
}

__device__ __forceinline__ double cell_offset(const CamParams &cam, const float4 A, const WarpCtx &W,
                                              double &c0, double &c1, double &c2)
{
    c0 = __dsub_rn((double)A.x, (double)cam.M[3]);
    c1 = __dsub_rn((double)A.y, (double)cam.M[7]);
    c2 = __dsub_rn((double)A.z, (double)cam.M[11]);
    return __fma_rn(W.wx, c0, __fma_rn(W.wy, c1, __dmul_rn(W.wz, c2)));
}

// Lane `lane` takes list entry e (if < end): conservative sphere-vs-warp-cone
// test in fp64; survivors are staged in slot `lane`.  Returns the ballot.
// Cone test: the sphere (c, r) meets the cone (axis d_w, half-angle th) iff
// the angle between c and d_w is <= th + asin(r/|c|), i.e. (|c| > r)
// d_w.c >= cos(th) sqrt(|c|^2 - r^2) - sin(th) r;  always if |c| <= r.
template <bool kDipole, bool kCull = false>
__device__ __forceinline__ unsigned stage_chunk(WarpStage &S, const DeviceScene &ds,
                                                const CamParams &cam,
                                                const uint32_t *__restrict__ vals, uint32_t e,
                                                uint32_t end, const WarpCtx &W, int lane)
{
    bool pass = false;
    uint32_t cell = 0;
    float4 A;
    double t = 0.0, c0 = 0.0, c1 = 0.0, c2 = 0.0;
    if (e < end) {
        cell = __ldg(vals + e);
        A = __ldg(ds.cellA + cell);
        t = cell_offset(cam, A, W, c0, c1, c2);
        const double cc = __fma_rn(c0, c0, __fma_rn(c1, c1, __dmul_rn(c2, c2)));
        const double rr = (double)A.w;
        const double r2 = __dmul_rn(rr, rr);
        if (cc <= r2) {
            pass = true;
        } else {
#if PF_RAY_FAST   // x rsqrt(x): a few fp64 ulps, far inside the 1e-7 |c| margin
            const double q = cc - r2;
            const double lim = W.cos_t * (q * rsqrt(q)) - W.sin_t * rr;
            pass = t >= lim - 1e-7 * (cc * rsqrt(cc));
#else
            const double lim = W.cos_t * sqrt(cc - r2) - W.sin_t * rr;
            pass = t >= lim - 1e-7 * sqrt(cc);
#endif
        }
    }
    const unsigned m = __ballot_sync(0xffffffffu, pass);
    if (pass) {
        stage_slot<kDipole>(S, lane, ds, cell, A, c0, c1, c2, t, W);
        if (kCull) cull_consts(S, lane, W);
    }
    __syncwarp();
    return m;
}

// ---------------------------------------------------------------------------
// Detail sites (NEXT-2, P:278-297 Eqs. svdisp/svrad).  Per (pixel,
// cell): the base-face hit x_bar, its chart point, the soft-Voronoi
// displacement delta (clamped to [-r, r]), the displaced face (m, delta) that
// clips the interval like the plain dipole face, and the radiance at the
// displaced-face hit x.  The chart geometry runs in fp64 from the exact ray
// (PixelRays) and c = p - Q: at grazing incidence the chart point moves by
// |c| eps / |d.m| per rounding, which fp32 would turn into visible colour
// error (condition number tau r / |d.m|).  Weights, blending and the reverse
// pass are fp32 on fp64-derived values.
// ---------------------------------------------------------------------------
struct DetailGeo {
    double A, ts;     // d.m and the absolute t of the displaced-face hit
    float delta;      // clamped displacement
    float dr;         // unclamped soft-Voronoi displacement
    bool parallel;    // d.m == 0: no base-face hit (reading R6e)
    float w[kMaxDetail];   // the soft-Voronoi weights at x_bar (reused by K7)
};

// softmax_a(gamma d.a_a) of the pixel's ray
__device__ __forceinline__ void sv_axis_weights(const DeviceScene &ds, const Ray &R, float om[8])
{
    float zmax = -3.0e38f;
#pragma unroll
    for (int a = 0; a < 8; ++a) {
        om[a] = ds.sv_gamma * fmaf(R.dx, ds.sv_axes[3 * a],
                                   fmaf(R.dy, ds.sv_axes[3 * a + 1], R.dz * ds.sv_axes[3 * a + 2]));
        zmax = fmaxf(zmax, om[a]);
    }
    float sum = 0.0f;
#pragma unroll
    for (int a = 0; a < 8; ++a) {
        om[a] = __expf(om[a] - zmax);
        sum += om[a];
    }
    const float inv = __frcp_rn(sum);
#pragma unroll
    for (int a = 0; a < 8; ++a) om[a] *= inv;
}

__device__ __forceinline__ float sqrt_approx(float x)
{
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// soft-Voronoi weights w_k = softmax_k(-tau |q - s_k|) at the chart point q
// (fp64 in, fp32 arithmetic).  Exponents relative to the nearest site j:
// rho_k - rho_j = (s_j - s_k).(2q - s_k - s_j) / (rho_k + rho_j), which keeps
// full relative precision when q is far from every site (grazing rays), where
// rho_k - rho_j from two rounded distances would not.
__device__ __forceinline__ void load_sites(const float2 *__restrict__ uv, int K,
                                           float2 s[kMaxDetail])
{
#pragma unroll
    for (int k = 0; k < kMaxDetail; ++k) s[k] = k < K ? __ldg(uv + k) : make_float2(0.0f, 0.0f);
}

__device__ __forceinline__ void soft_voronoi(const float2 s[kMaxDetail], int K, double q0d,
                                             double q1d, float tau, float w[kMaxDetail])
{
    const float q0 = __double2float_rn(q0d), q1 = __double2float_rn(q1d);
    float sx[kMaxDetail], sy[kMaxDetail], r2[kMaxDetail];
    float r2m = 3.0e38f, jx = 0.0f, jy = 0.0f;
#pragma unroll
    for (int k = 0; k < kMaxDetail; ++k) {
        if (k < K) {
            const float2 sk = s[k];
            sx[k] = sk.x;
            sy[k] = sk.y;
            const float dx = q0 - sk.x, dy = q1 - sk.y;
            r2[k] = fmaf(dx, dx, dy * dy);
            if (r2[k] < r2m) {
                r2m = r2[k];
                jx = sk.x;
                jy = sk.y;
            }
        }
    }
    const float rj = sqrt_approx(r2m), tx = fmaf(2.0f, q0, -jx), ty = fmaf(2.0f, q1, -jy);
    float sum = 0.0f;
#pragma unroll
    for (int k = 0; k < kMaxDetail; ++k) {
        w[k] = 0.0f;
        if (k < K) {
            const float num = fmaf(jx - sx[k], tx - sx[k], (jy - sy[k]) * (ty - sy[k]));
            const float den = sqrt_approx(r2[k]) + rj;
            const float diff = den > 0.0f ? num * rcp_approx(den) : 0.0f;
            w[k] = __expf(-tau * diff);
            sum += w[k];
        }
    }
    const float inv = rcp_approx(sum);
#pragma unroll
    for (int k = 0; k < kMaxDetail; ++k) w[k] *= inv;
}

// c = p - Q in fp64 (the exact site minus the exact camera centre)
__device__ __forceinline__ void cell_c(const DeviceScene &ds, const CamParams &cam, uint32_t cell,
                                       double c[3])
{
    const float4 A = __ldg(ds.cellA + cell);
    c[0] = __dsub_rn((double)A.x, (double)cam.M[3]);
    c[1] = __dsub_rn((double)A.y, (double)cam.M[7]);
    c[2] = __dsub_rn((double)A.z, (double)cam.M[11]);
}

__device__ __forceinline__ double dot3d(const double a[3], double b0, double b1, double b2)
{
    return __fma_rn(a[0], b0, __fma_rn(a[1], b1, __dmul_rn(a[2], b2)));
}

// Eq. svdisp: base-face hit, displacement, displaced face.  Returns the face as
// a clip plane (m, delta):  (x - p).m <= delta  <=>  a t' <= m.e + delta.
template <int KT>
__device__ __forceinline__ float4 detail_plane(const DeviceScene &ds, uint32_t cell,
                                               const double d[3], const double c[3], float r,
                                               DetailGeo &G)
{
    const double *F = ds.cellF + (size_t)kCellF * cell;
    const double m0 = __ldg(F), m1 = __ldg(F + 1), m2 = __ldg(F + 2);
    G.A = dot3d(d, m0, m1, m2);
    const double B = dot3d(c, m0, m1, m2);
    G.parallel = (G.A == 0.0);
    G.delta = 0.0f;
    G.dr = 0.0f;
    G.ts = 0.0;
    if (!G.parallel) {
        const double iA = __drcp_rn(G.A);   // one reciprocal for both face hits
        const double tb = __dmul_rn(B, iA);
        const double y0 = __fma_rn(tb, d[0], -c[0]), y1 = __fma_rn(tb, d[1], -c[1]),
                     y2 = __fma_rn(tb, d[2], -c[2]);
        const double q0 = __fma_rn(y0, __ldg(F + 3), __fma_rn(y1, __ldg(F + 4), __dmul_rn(y2, __ldg(F + 5))));
        const double q1 = __fma_rn(y0, __ldg(F + 6), __fma_rn(y1, __ldg(F + 7), __dmul_rn(y2, __ldg(F + 8))));
        float *w = G.w;
        const int K = KT == 8 ? 8 : ds.K;   // K == 8 (the paper's setting) known at compile time
        float2 st[kMaxDetail];
        load_sites(reinterpret_cast<const float2 *>(ds.duv) + (size_t)K * cell, K, st);
        soft_voronoi(st, K, q0, q1, ds.sv_tau, w);
        const float *dk = ds.ddisp + (size_t)K * cell;
        float dr = 0.0f;
#pragma unroll
        for (int k = 0; k < kMaxDetail; ++k)
            if (k < K) dr = fmaf(w[k], __ldg(dk + k), dr);
        G.dr = dr;
        G.delta = fminf(fmaxf(dr, -r), r);
        G.ts = __dmul_rn(__dadd_rn(B, (double)G.delta), iA);
    }
    return make_float4(__double2float_rn(m0), __double2float_rn(m1), __double2float_rn(m2), G.delta);
}

// detail_plane for the lanes of one cell at once (K6, every lane calls it; `pre`
// lanes want the face).  The fp64 chart runs per lane as in detail_plane; the
// soft-Voronoi weights at the base-face hit are spread over the warp, lane 8g + k
// taking site k of the g-th wanting lane (up to 4 lanes per round): the same per-site
// operations, the argmin with detail_plane's first-minimum tie rule, then each lane
// gathers its 8 weights and normalises / blends them in site order -- bit-identical to
// detail_plane (delta, ts; G.w is not produced: K6 does not use it).
template <int KT>
__device__ __forceinline__ float4 detail_plane_warp(const DeviceScene &ds, uint32_t cell, bool pre,
                                                    const double d[3], const double c[3], float r,
                                                    DetailGeo &G, int lane)
{
    const double *F = ds.cellF + (size_t)kCellF * cell;
    const double m0 = __ldg(F), m1 = __ldg(F + 1), m2 = __ldg(F + 2);
    float q0f = 0.0f, q1f = 0.0f;
    double B = 0.0, iA = 0.0;
    G.delta = 0.0f;
    G.dr = 0.0f;
    G.ts = 0.0;
    G.parallel = true;
    if (pre) {
        G.A = dot3d(d, m0, m1, m2);
        B = dot3d(c, m0, m1, m2);
        G.parallel = (G.A == 0.0);
        if (!G.parallel) {
            iA = __drcp_rn(G.A);
            const double tb = __dmul_rn(B, iA);
            const double y0 = __fma_rn(tb, d[0], -c[0]), y1 = __fma_rn(tb, d[1], -c[1]),
                         y2 = __fma_rn(tb, d[2], -c[2]);
            const double q0 = __fma_rn(y0, __ldg(F + 3), __fma_rn(y1, __ldg(F + 4), __dmul_rn(y2, __ldg(F + 5))));
            const double q1 = __fma_rn(y0, __ldg(F + 6), __fma_rn(y1, __ldg(F + 7), __dmul_rn(y2, __ldg(F + 8))));
            q0f = __double2float_rn(q0);
            q1f = __double2float_rn(q1);
        }
    }
    const int K = KT == 8 ? 8 : ds.K;
    const int k = lane & 7, gbase = lane & ~7;
    const float2 sk = k < K ? __ldg(reinterpret_cast<const float2 *>(ds.duv) + (size_t)K * cell + k)
                            : make_float2(0.0f, 0.0f);
    const float *dk = ds.ddisp + (size_t)K * cell;
    const float tau = ds.sv_tau;
    unsigned want = __ballot_sync(0xffffffffu, pre && !G.parallel);
    while (want) {
        // this round: the first (up to) 4 wanting lanes, group g = lane / 8 serves the g-th
        const int g = lane >> 3;
        unsigned rest = want, mg = 0u;   // rest: want without its 4 lowest set bits
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if (i == g) mg = rest;       // want without its g lowest set bits
            rest &= rest - 1u;
        }
        const int src = mg ? __ffs(mg) - 1 : lane;
        const unsigned round = want & ~rest;
        want = rest;
        const float qa = __shfl_sync(0xffffffffu, q0f, src), qb = __shfl_sync(0xffffffffu, q1f, src);
        const float dx = qa - sk.x, dy = qb - sk.y;
        const float r2 = k < K ? fmaf(dx, dx, dy * dy) : 3.0e38f;
        // argmin over the group's 8 sites, ties to the lower site index
        float mr = r2;
        int mk = k;
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
            const float orr = __shfl_xor_sync(0xffffffffu, mr, o);
            const int ok = __shfl_xor_sync(0xffffffffu, mk, o);
            if (orr < mr || (orr == mr && ok < mk)) {
                mr = orr;
                mk = ok;
            }
        }
        const float jx = __shfl_sync(0xffffffffu, sk.x, gbase | mk),
                    jy = __shfl_sync(0xffffffffu, sk.y, gbase | mk);
        const float rj = sqrt_approx(mr), tx = fmaf(2.0f, qa, -jx), ty = fmaf(2.0f, qb, -jy);
        float w = 0.0f;
        if (k < K) {
            const float num = fmaf(jx - sk.x, tx - sk.x, (jy - sk.y) * (ty - sk.y));
            const float den = sqrt_approx(r2) + rj;
            const float diff = den > 0.0f ? num * rcp_approx(den) : 0.0f;
            w = __expf(-tau * diff);
        }
        // each wanting lane of the round gathers its group's weights in site order
        const bool mine = (round >> lane) & 1u;
        const int gme = __popc(round & ((1u << lane) - 1u));
        float wk[kMaxDetail];
        float sum = 0.0f;
#pragma unroll
        for (int kk = 0; kk < kMaxDetail; ++kk) {
            wk[kk] = __shfl_sync(0xffffffffu, w, ((mine ? gme : 0) << 3) | kk);
            if (kk < K) sum += wk[kk];
        }
        if (mine) {
            const float inv = rcp_approx(sum);
            float dr = 0.0f;
#pragma unroll
            for (int kk = 0; kk < kMaxDetail; ++kk)
                if (kk < K) dr = fmaf(wk[kk] * inv, __ldg(dk + kk), dr);
            G.dr = dr;
            G.delta = fminf(fmaxf(dr, -r), r);
            G.ts = __dmul_rn(__dadd_rn(B, (double)G.delta), iA);
        }
    }
    return make_float4(__double2float_rn(m0), __double2float_rn(m1), __double2float_rn(m2), G.delta);
}

// Eq. svrad at the point Q + t d (t = the displaced-face hit, or the interval
// entry for a parallel ray): sum_k w_k sum_a om_a v_{k,a}
template <int KT>
__device__ __forceinline__ void detail_color(const DeviceScene &ds, uint32_t cell, const double d[3],
                                             const double c[3], double t, const float om[8],
                                             float &cr, float &cg, float &cb)
{
    const double *F = ds.cellF + (size_t)kCellF * cell;
    const double y0 = __fma_rn(t, d[0], -c[0]), y1 = __fma_rn(t, d[1], -c[1]),
                 y2 = __fma_rn(t, d[2], -c[2]);
    const double q0 = __fma_rn(y0, __ldg(F + 3), __fma_rn(y1, __ldg(F + 4), __dmul_rn(y2, __ldg(F + 5))));
    const double q1 = __fma_rn(y0, __ldg(F + 6), __fma_rn(y1, __ldg(F + 7), __dmul_rn(y2, __ldg(F + 8))));
    float w[kMaxDetail];
    const int K = KT == 8 ? 8 : ds.K;   // K == 8 (the paper's setting) known at compile time
    float2 st[kMaxDetail];
    load_sites(reinterpret_cast<const float2 *>(ds.duv) + (size_t)K * cell, K, st);
    soft_voronoi(st, K, q0, q1, ds.sv_tau, w);
    const float4 *sv = reinterpret_cast<const float4 *>(ds.dsv) + (size_t)6 * K * cell;
    cr = cg = cb = 0.0f;
#pragma unroll
    for (int k = 0; k < kMaxDetail; ++k) {
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
            cr = fmaf(w[k], kr, cr);
            cg = fmaf(w[k], kg, cg);
            cb = fmaf(w[k], kb, cb);
        }
    }
}

// ---------------------------------------------------------------------------
// K6 -> K7 segment records.  For every 32-entry chunk of its tile list a warp
// walked, K6 writes a descriptor (first record, count); for every chunk entry
// that produced a non-empty segment in at least one lane it writes a 72-byte
// record: the lane mask, the entry (cell id, or its chunk slot), and per lane the
// binding constraints of the interval (lo, hi) coded in one byte each
// (0 sphere, 1 near, 2+k plane k of the cell's list, 254 dipole face,
// 255 = not codable).  K7
// then replays only those entries and evaluates only the binding planes: the
// interval values are bit-identical (fminf/fmaxf return one of their inputs,
// and the winning input is recomputed with the same instructions).
// The arena is sized from the pair count; a chunk whose records do not fit is
// marked kOverflow and K7 recomputes it in full.
// ---------------------------------------------------------------------------
constexpr uint32_t kOverflow = 0xffffffffu;
// A record's second word is the cell id (plain scenes; K7 stages it without the
// tile-list gather) or, for detail scenes,  slot | first colour slot << 5  (K6 stores
// each segment's colour and displacement, float4 (rgb, delta), in the view's colour
// arena, in lane order); kNoCol = no slots (arena full): K7 recomputes them
constexpr uint32_t kNoCol = 0x7ffffffu;
constexpr uint32_t kColBlock = 64;   // colour slots a K6 warp claims at a time
constexpr int kRecWords = 18;   // mask, pos, 32 x u16 codes

struct WarpRec {                 // a chunk's records in their global layout (flushed as is)
    uint32_t w[32 * kRecWords];  // per record: mask, pos (slot), 32 lanes x u16 codes
};

template <bool kDipole>
__device__ __forceinline__ uint32_t end_code(int q)
{
    // tracked codes are already record codes (0 sphere, 1 near, 2 + plane index);
    // 255 = not representable (K7 replays the entry in full).  With dipoles 254 is
    // the dipole face, so plane 252 must not produce it.
    if (!kDipole) return min((uint32_t)q, 255u);
    return q == kEndDipole ? 254u : ((uint32_t)q >= 254u ? 255u : (uint32_t)q);
}

}  // namespace

}  // namespace pf
