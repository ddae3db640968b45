// pf_prep.cu -- K0 edge records, scene validation, K1 projection + tile binning +
// sort key, K2 scan of the per-cell pair counts, K3 pair emission, K5 tile ranges.
//
// K1 is an fp32 SPECIFICATION: it produces
// integers (tile rectangles, key bits) that must be bit-identical to the CPU
// oracle, so every operation is an explicit IEEE round-to-nearest intrinsic
// evaluated left to right with no FMA contraction.
#include <cuda_runtime.h>
#include <math.h>

#include "pf_internal.cuh"

namespace pf {

// ------------------------------------------------------------------------
// K0: cell and edge records
// ------------------------------------------------------------------------
// Face chart of a detail cell (NEXT-2; the frame of SPEC S:186-189), fp64:
// m = n/|n|, k = the axis of the smallest |n_k| (ties to the higher index),
// u = (e_k x m)/|e_k x m|, v = m x u.  cellF[i] = (m, u, v, 1/|n|, 1/|e_k x m|, k).
__device__ __forceinline__ void face_frame(const DeviceScene &ds, int64_t i)
{
    const float fx = ds.normals[3 * i], fy = ds.normals[3 * i + 1], fz = ds.normals[3 * i + 2];
    const double nn = sqrt((double)fx * fx + (double)fy * fy + (double)fz * fz);
    const double m0 = fx / nn, m1 = fy / nn, m2 = fz / nn;
    const float ax = fabsf(fx), ay = fabsf(fy), az = fabsf(fz);
    const int k = (ax < ay && ax < az) ? 0 : (ay <= az ? 1 : 2);
    // w = e_k x m
    const double w0 = k == 0 ? 0.0 : (k == 1 ? m2 : -m1);
    const double w1 = k == 0 ? -m2 : (k == 1 ? 0.0 : m0);
    const double w2 = k == 0 ? m1 : (k == 1 ? -m0 : 0.0);
    const double wl = sqrt(w0 * w0 + w1 * w1 + w2 * w2);
    const double u0 = w0 / wl, u1 = w1 / wl, u2 = w2 / wl;
    double *F = ds.cellF + (size_t)kCellF * i;
    F[0] = m0; F[1] = m1; F[2] = m2;
    F[3] = u0; F[4] = u1; F[5] = u2;
    F[6] = m1 * u2 - m2 * u1;
    F[7] = m2 * u0 - m0 * u2;
    F[8] = m0 * u1 - m1 * u0;
    F[9] = 1.0 / nn; F[10] = 1.0 / wl; F[11] = (double)k;   // reciprocals: read by K7 only
}

__global__ void __launch_bounds__(256) k0_edge_records(DeviceScene ds)
{
    // cell records: one thread per cell.  Edge records: the warp's 32 cells own
    // the contiguous CSR range [off[i0], off[i0+32]); the warp walks it 32 edges
    // at a time (coalesced index reads and record writes), each lane finding its
    // edge's source cell by a binary search over the lanes' offsets (shuffles).
    const int lane = threadIdx.x & 31;
    const int64_t i0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) & ~31ll;
    const int64_t i = i0 + lane;
    if (i0 >= ds.N) return;
    float px = 0.f, py = 0.f, pz = 0.f, wi = 0.f;
    int64_t ob = 0, oe = 0;
    if (i < ds.N) {
        px = ds.sites[3 * i];
        py = ds.sites[3 * i + 1];
        pz = ds.sites[3 * i + 2];
        wi = ds.weights[i];
        ob = ds.nbr_off[i];
        oe = ds.nbr_off[i + 1];
        ds.cellA[i] = make_float4(px, py, pz, ds.radii[i]);
        ds.cellB[i] = make_float4(ds.density[i], ds.rgb[3 * i], ds.rgb[3 * i + 1], ds.rgb[3 * i + 2]);
        ds.cellE[i] = make_uint2((uint32_t)ob, (uint32_t)(oe - ob));
        if (ds.normals)
            ds.cellN[i] = make_float4(ds.normals[3 * i], ds.normals[3 * i + 1],
                                      ds.normals[3 * i + 2], 0.0f);
        if (ds.K) face_frame(ds, i);
    }
    const int64_t base = __shfl_sync(0xffffffffu, ob, 0);
    const int last = (int)min((int64_t)31, ds.N - 1 - i0);
    const int64_t end = __shfl_sync(0xffffffffu, oe, last);
    const uint32_t rel = (i < ds.N) ? (uint32_t)(ob - base) : 0xffffffffu;
    const uint32_t total = (uint32_t)(end - base);
    for (uint32_t e0 = 0; e0 < total; e0 += 32) {
        const uint32_t e = e0 + lane;
        int src = 0;
#pragma unroll
        for (int step = 16; step > 0; step >>= 1) {
            const int cand = src + step;
            const uint32_t r = __shfl_sync(0xffffffffu, rel, cand & 31);
            if (cand < 32 && r <= e) src = cand;
        }
        const float sx = __shfl_sync(0xffffffffu, px, src), sy = __shfl_sync(0xffffffffu, py, src),
                    sz = __shfl_sync(0xffffffffu, pz, src), sw = __shfl_sync(0xffffffffu, wi, src);
        if (e < total) {
            const int64_t q = base + e;
            const int j = ds.nbr_idx[q];
            const float nx = ds.sites[3 * j] - sx, ny = ds.sites[3 * j + 1] - sy,
                        nz = ds.sites[3 * j + 2] - sz;
            const float nn = nx * nx + ny * ny + nz * nz;
            // pow(x,i) <= pow(x,j)  <=>  (x - p_i).n <= 0.5 (|n|^2 - (w_j - w_i))
            const float k = 0.5f * (nn - (ds.weights[j] - sw));
            ds.edges[q] = make_float4(nx, ny, nz, k);
        }
    }
}

cudaError_t launch_edge_records(pf_scene *s, cudaStream_t st)
{
    cudaEvent_t ev;
    stage_begin(s, 0, st, &ev);
    k0_edge_records<<<ceil_div(s->ds.N, 256), 256, 0, st>>>(s->ds);
    ++s->launches;
    stage_end(s, 0, st, ev);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------
// validation (PF_VALIDATE)
// ------------------------------------------------------------------------
__global__ void k_validate(DeviceScene ds, int *flag)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= ds.N) return;
    int bad = 0;
    for (int m = 0; m < 3; ++m) {
        bad |= !isfinite(ds.sites[3 * i + m]) ? 1 : 0;
        bad |= !isfinite(ds.rgb[3 * i + m]) ? 2 : 0;
    }
    bad |= !isfinite(ds.weights[i]) ? 4 : 0;
    bad |= !(ds.radii[i] > 0.0f) || !isfinite(ds.radii[i]) ? 8 : 0;
    bad |= !(ds.density[i] >= 0.0f) || !isfinite(ds.density[i]) ? 16 : 0;
    if (ds.normals) {
        const float nx = ds.normals[3 * i], ny = ds.normals[3 * i + 1], nz = ds.normals[3 * i + 2];
        if (!isfinite(nx) || !isfinite(ny) || !isfinite(nz) || (nx == 0.f && ny == 0.f && nz == 0.f))
            bad |= 128;
    }
    for (int k = 0; k < ds.K; ++k) {
        const size_t q = (size_t)ds.K * i + k;
        bad |= (!isfinite(ds.duv[2 * q]) || !isfinite(ds.duv[2 * q + 1]) ||
                !isfinite(ds.ddisp[q])) ? 256 : 0;
        for (int a = 0; a < 24; ++a) bad |= !isfinite(ds.dsv[24 * q + a]) ? 256 : 0;
    }
    int64_t b = ds.nbr_off[i], e = ds.nbr_off[i + 1];
    if (b < 0 || e < b || e > ds.E) bad |= 32;
    else
        for (int64_t q = b; q < e; ++q) {
            int j = ds.nbr_idx[q];
            if (j < 0 || j >= ds.N || j == i) bad |= 64;
        }
    if (bad) atomicOr(flag, bad);
}

cudaError_t launch_validate(pf_scene *s, int *d_flag, cudaStream_t st)
{
    k_validate<<<ceil_div(s->ds.N, 256), 256, 0, st>>>(s->ds, d_flag);
    ++s->launches;
    return cudaGetLastError();
}

// ------------------------------------------------------------------------
// K1: project the bounding sphere, tile rectangle, count, key bits
// ------------------------------------------------------------------------
__device__ __forceinline__ uint32_t order_bits(float K)
{
    uint32_t u = __float_as_uint(K);
    return (u >> 31) ? ~u : (u | 0x80000000u);
}

// Extent of the sphere's image along one axis (a = camera coordinate along the
// axis, z = depth), in pixels.  Sphere in front of the near plane: the two
// tangent planes through the camera centre; straddling: the box
// [a-r, a+r] x [near, z+r].
__device__ __forceinline__ void sphere_extent(float a, float z, float r, float f, float c,
                                              float nearp, bool in_front, float &lo, float &hi)
{
    float ulo, uhi;
    if (in_front) {
        float q = __fsqrt_rn(__fsub_rn(__fadd_rn(__fmul_rn(a, a), __fmul_rn(z, z)),
                                       __fmul_rn(r, r)));
        float den = __fmul_rn(__fsub_rn(z, r), __fadd_rn(z, r));
        float az = __fmul_rn(a, z), rq = __fmul_rn(r, q);
        ulo = __fdiv_rn(__fsub_rn(az, rq), den);
        uhi = __fdiv_rn(__fadd_rn(az, rq), den);
    } else {
        float amin = __fsub_rn(a, r), amax = __fadd_rn(a, r);
        float zfar = __fadd_rn(z, r);
        ulo = __fdiv_rn(amin, amin >= 0.0f ? zfar : nearp);
        uhi = __fdiv_rn(amax, amax >= 0.0f ? nearp : zfar);
    }
    lo = __fadd_rn(__fmul_rn(f, ulo), c);
    hi = __fadd_rn(__fmul_rn(f, uhi), c);
}

__device__ __forceinline__ int tile_lo(float px, int ntiles)
{
    float t = floorf(__fmul_rn(__fsub_rn(px, 1.0f), 0.0625f));
    return (int)fminf(fmaxf(t, 0.0f), (float)ntiles);
}
__device__ __forceinline__ int tile_hi(float px, int ntiles)
{
    float t = __fadd_rn(floorf(__fmul_rn(__fadd_rn(px, 1.0f), 0.0625f)), 1.0f);
    return (int)fminf(fmaxf(t, 0.0f), (float)ntiles);
}

// ---- equidistant fisheye binning (NEXT-4) --------------------------------
// The map (a, b) -> camera ray is 1-Lipschitz in angle, so every pixel ray of a
// tile is within th = |(9/fx, 9/fy)| of the ray through the tile centre (8 px to
// the border + 1 px guard); the sphere (c, r) can meet a ray of the tile only if
// c.a_t >= cos(th) sqrt(|c|^2 - r^2) - sin(th) r, or |c| <= r.  Evaluated in fp64;
// the candidate rectangle (bounding box of the angular cap's annular sector) is
// any superset, the count is the number of passing tiles.
__device__ __forceinline__ void fisheye_dir(const CamParams &cam, double u, double v, double dc[3])
{
    const double a = (u - (double)cam.cx) / (double)cam.fx, b = (v - (double)cam.cy) / (double)cam.fy;
    const double th = sqrt(a * a + b * b);
    if (th > 0.0) {
        double sn, cs;
        sincos(th, &sn, &cs);
        dc[0] = sn / th * a;
        dc[1] = sn / th * b;
        dc[2] = cs;
    } else {
        dc[0] = dc[1] = 0.0;
        dc[2] = 1.0;
    }
}

__device__ __forceinline__ double fisheye_half_angle(const CamParams &cam)
{
    const double ax = 9.0 / (double)cam.fx, ay = 9.0 / (double)cam.fy;
    return sqrt(ax * ax + ay * ay);
}

// per-view table: the ray through every tile centre (3 doubles per tile), then
// cos(th), sin(th) -- computed once per view instead of per (cell, tile)
__global__ void __launch_bounds__(256) k1_fisheye_dirs(CamParams cam, double *__restrict__ tdir)
{
    const int T = cam.tiles_x * cam.tiles_y;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < T) {
        const int tx = t % cam.tiles_x, ty = t / cam.tiles_x;
        double at[3];
        fisheye_dir(cam, 16.0 * tx + 8.0, 16.0 * ty + 8.0, at);
        tdir[3 * t] = at[0];
        tdir[3 * t + 1] = at[1];
        tdir[3 * t + 2] = at[2];
    }
    if (t == 0) {
        const double th = fisheye_half_angle(cam);
        tdir[3 * T] = cos(th);
        tdir[3 * T + 1] = sin(th);
    }
}

__device__ __forceinline__ bool fisheye_tile_pass(const CamParams &cam, const double c[3], double r,
                                                  double cth, double sth, int tx, int ty,
                                                  const double *__restrict__ tdir)
{
    const double cc = c[0] * c[0] + c[1] * c[1] + c[2] * c[2];
    if (cc <= r * r) return true;
    const double *at = tdir + 3 * (ty * cam.tiles_x + tx);
    const double lhs = c[0] * __ldg(at) + c[1] * __ldg(at + 1) + c[2] * __ldg(at + 2);
    return lhs >= cth * sqrt(cc - r * r) - sth * r;
}

__device__ void fisheye_rect(const CamParams &cam, const double c[3], double r, double th, int4 &rc)
{
    const double PI = 3.14159265358979323846;
    const double cc = sqrt(c[0] * c[0] + c[1] * c[1] + c[2] * c[2]);
    double amin, amax, bmin, bmax;
    if (cc <= r) {
        amin = bmin = -PI;
        amax = bmax = PI;
    } else {
        const double beta = asin(r / cc) + th + 1e-6;
        const double thc = acos(fmax(-1.0, fmin(1.0, c[2] / cc)));
        const double phc = atan2(c[1], c[0]);
        const double rmax = fmin(thc + beta, PI);
        if (thc - beta <= 0.0 || thc + beta >= PI) {
            amin = bmin = -rmax;
            amax = bmax = rmax;
        } else {
            const double rmin = thc - beta;
            const double dph = asin(fmin(1.0, sin(beta) / sin(thc)));
            const double p0 = phc - dph, p1 = phc + dph;
            amin = bmin = 1e30;
            amax = bmax = -1e30;
            for (int k = 0; k < 2; ++k)
                for (int q = 0; q < 2; ++q) {
                    const double rr = q ? rmax : rmin, ph = k ? p1 : p0;
                    double sn, cs;
                    sincos(ph, &sn, &cs);
                    amin = fmin(amin, rr * cs); amax = fmax(amax, rr * cs);
                    bmin = fmin(bmin, rr * sn); bmax = fmax(bmax, rr * sn);
                }
            for (int k = -4; k <= 4; ++k) {   // axis directions inside the sector
                const double ph = k * (PI / 2);
                if (ph >= p0 && ph <= p1) {
                    double sn, cs;
                    sincos(ph, &sn, &cs);
                    amin = fmin(amin, rmax * cs); amax = fmax(amax, rmax * cs);
                    bmin = fmin(bmin, rmax * sn); bmax = fmax(bmax, rmax * sn);
                }
            }
        }
    }
    const double u0 = cam.cx + cam.fx * amin, u1 = cam.cx + cam.fx * amax;
    const double v0 = cam.cy + cam.fy * bmin, v1 = cam.cy + cam.fy * bmax;
    rc.x = (int)fmax(0.0, fmin((double)cam.tiles_x, floor((u0 - 1.0) / 16.0)));
    rc.z = (int)fmax(0.0, fmin((double)cam.tiles_x, floor((u1 + 1.0) / 16.0) + 1.0));
    rc.y = (int)fmax(0.0, fmin((double)cam.tiles_y, floor((v0 - 1.0) / 16.0)));
    rc.w = (int)fmax(0.0, fmin((double)cam.tiles_y, floor((v1 + 1.0) / 16.0) + 1.0));
}

__device__ __forceinline__ void camera_coords(const CamParams &cam, const float *p, double c[3])
{
    const float *M = cam.M;
    const double v0 = (double)p[0] - (double)M[3], v1 = (double)p[1] - (double)M[7],
                 v2 = (double)p[2] - (double)M[11];
    for (int k = 0; k < 3; ++k)
        c[k] = (double)M[k] * v0 + (double)M[4 + k] * v1 + (double)M[8 + k] * v2;
}

// one cell, one pinhole view: tile rect, pair count, key bits (every op a
// separate IEEE-rn fp32 op, the binning is an fp32 specification)
__device__ __forceinline__ uint32_t k1_pinhole(const CamParams &cam, float sx, float sy, float sz,
                                               float w, float r, int4 &rc, int &cnt)
{
    const float *M = cam.M;
    float v0 = __fsub_rn(sx, M[3]);
    float v1 = __fsub_rn(sy, M[7]);
    float v2 = __fsub_rn(sz, M[11]);
    // camera coordinates: c_k = (R_0k v0 + R_1k v1) + R_2k v2
    float ca = __fadd_rn(__fadd_rn(__fmul_rn(M[0], v0), __fmul_rn(M[4], v1)), __fmul_rn(M[8], v2));
    float cb = __fadd_rn(__fadd_rn(__fmul_rn(M[1], v0), __fmul_rn(M[5], v1)), __fmul_rn(M[9], v2));
    float cz = __fadd_rn(__fadd_rn(__fmul_rn(M[2], v0), __fmul_rn(M[6], v1)), __fmul_rn(M[10], v2));
    // sort key K_i = pow(Q, p_i) = |p_i - Q|^2 - w_i   (Theorem 2)
    float K = __fsub_rn(__fadd_rn(__fadd_rn(__fmul_rn(v0, v0), __fmul_rn(v1, v1)),
                                  __fmul_rn(v2, v2)),
                        w);
    rc = make_int4(0, 0, 0, 0);
    cnt = 0;
    if ((__fadd_rn(cz, r) > cam.near_plane) && (r > 0.0f)) {
        bool in_front = __fsub_rn(cz, r) > cam.near_plane;
        float xlo, xhi, ylo, yhi;
        sphere_extent(ca, cz, r, cam.fx, cam.cx, cam.near_plane, in_front, xlo, xhi);
        sphere_extent(cb, cz, r, cam.fy, cam.cy, cam.near_plane, in_front, ylo, yhi);
        int tx0 = tile_lo(xlo, cam.tiles_x), tx1 = tile_hi(xhi, cam.tiles_x);
        int ty0 = tile_lo(ylo, cam.tiles_y), ty1 = tile_hi(yhi, cam.tiles_y);
        if (tx1 > tx0 && ty1 > ty0) {
            rc = make_int4(tx0, ty0, tx1, ty1);
            cnt = (tx1 - tx0) * (ty1 - ty0);
        }
    }
    return order_bits(K);
}

__global__ void __launch_bounds__(256)
k1_preprocess(const float *__restrict__ sites, const float *__restrict__ weights,
              const float *__restrict__ radii, int64_t N, CamParams cam, int4 *__restrict__ rect,
              int *__restrict__ count, uint32_t *__restrict__ keybits,
              const double *__restrict__ tdir)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (cam.model == PF_FISHEYE) {   // warp-uniform: every lane of the warp stays
        const bool live = i < N;
        const int lane = threadIdx.x & 31;
        int4 cand = make_int4(0, 0, 0, 0);
        double c[3] = {0.0, 0.0, 0.0};
        double r = 0.0;
        if (live) {
            const float *M = cam.M;
            const float v0 = __fsub_rn(sites[3 * i + 0], M[3]), v1 = __fsub_rn(sites[3 * i + 1], M[7]),
                        v2 = __fsub_rn(sites[3 * i + 2], M[11]);
            const float K = __fsub_rn(__fadd_rn(__fadd_rn(__fmul_rn(v0, v0), __fmul_rn(v1, v1)),
                                                __fmul_rn(v2, v2)),
                                      weights[i]);
            keybits[i] = order_bits(K);
            const float rf = radii[i];
            r = rf;
            camera_coords(cam, sites + 3 * i, c);
            const double dist = sqrt(c[0] * c[0] + c[1] * c[1] + c[2] * c[2]);
            if ((rf > 0.0f) && !(dist + r <= (double)cam.near_plane))
                fisheye_rect(cam, c, r, fisheye_half_angle(cam), cand);
        }
        // count the passing tiles: the warp's cells one after another, lanes over tiles
        const int T = cam.tiles_x * cam.tiles_y;
        const double cth = __ldg(tdir + 3 * T), sth = __ldg(tdir + 3 * T + 1);
        const int w = cand.z - cand.x, n = w > 0 && cand.w > cand.y ? w * (cand.w - cand.y) : 0;
        unsigned todo = __ballot_sync(0xffffffffu, n > 0);
        int my_cnt = 0;
        while (todo) {
            const int src = __ffs(todo) - 1;
            todo &= todo - 1;
            const int sx = __shfl_sync(0xffffffffu, cand.x, src), sy = __shfl_sync(0xffffffffu, cand.y, src);
            const int sw = __shfl_sync(0xffffffffu, w, src), sn = __shfl_sync(0xffffffffu, n, src);
            const double s0 = __shfl_sync(0xffffffffu, c[0], src), s1 = __shfl_sync(0xffffffffu, c[1], src),
                         s2 = __shfl_sync(0xffffffffu, c[2], src), sr = __shfl_sync(0xffffffffu, r, src);
            const double sc[3] = {s0, s1, s2};
            int tot = 0;
            for (int b = 0; b < sn; b += 32) {
                const int t = b + lane;
                const bool pass = t < sn && fisheye_tile_pass(cam, sc, sr, cth, sth, sx + t % sw,
                                                              sy + t / sw, tdir);
                tot += __popc(__ballot_sync(0xffffffffu, pass));
            }
            if (lane == src) my_cnt = tot;
        }
        if (live) {
            rect[i] = my_cnt ? cand : make_int4(0, 0, 0, 0);
            count[i] = my_cnt;
        }
        return;
    }
    if (i >= N) return;
    int4 rc;
    int cnt;
    keybits[i] = k1_pinhole(cam, sites[3 * i + 0], sites[3 * i + 1], sites[3 * i + 2], weights[i],
                            radii[i], rc, cnt);
    rect[i] = rc;
    count[i] = cnt;
}

// K1 of a batch of pinhole views in one launch: each cell's site, weight and radius
// read once for all views of the batch (the per-view code is k1_pinhole, the same
// instructions as the one-view kernel: bit-identical binning)
__global__ void __launch_bounds__(256)
k1_preprocess_batch(const float *__restrict__ sites, const float *__restrict__ weights,
                    const float *__restrict__ radii, int64_t N, BatchViews bv)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const float x = sites[3 * i + 0], y = sites[3 * i + 1], z = sites[3 * i + 2];
    const float w = weights[i], r = radii[i];
    for (int v = 0; v < bv.n; ++v) {
        int4 rc;
        int cnt;
        const uint32_t kb = k1_pinhole(bv.cam[v], x, y, z, w, r, rc, cnt);
        const_cast<uint32_t *>(bv.keybits[v])[i] = kb;
        const_cast<int4 *>(bv.rect[v])[i] = rc;
        const_cast<int *>(bv.count[v])[i] = cnt;
    }
}

cudaError_t launch_preprocess_batch(pf_scene *s, const BatchViews &bv, cudaStream_t st)
{
    cudaEvent_t ev;
    stage_begin(s, 1, st, &ev);
    k1_preprocess_batch<<<ceil_div(s->ds.N, 256), 256, 0, st>>>(s->ds.sites, s->ds.weights,
                                                               s->ds.radii, s->ds.N, bv);
    ++s->launches;
    stage_end(s, 1, st, ev);
    return cudaGetLastError();
}

cudaError_t launch_preprocess(pf_scene *s, ViewState &v, cudaStream_t st)
{
    cudaEvent_t ev;
    stage_begin(s, 1, st, &ev);
    if (v.cam.model == PF_FISHEYE) {
        k1_fisheye_dirs<<<ceil_div((int64_t)v.cam.tiles_x * v.cam.tiles_y, 256), 256, 0, st>>>(
            v.cam, v.tdir.as<double>());
        ++s->launches;
    }
    k1_preprocess<<<ceil_div(s->ds.N, 256), 256, 0, st>>>(
        s->ds.sites, s->ds.weights, s->ds.radii, s->ds.N, v.cam, v.rect.as<int4>(),
        v.count.as<int>(), v.keybits.as<uint32_t>(), v.tdir.as<double>());
    ++s->launches;
    stage_end(s, 1, st, ev);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------
// K2: exclusive scan of the counts (3 phases: block sums, scan of sums, rescan)
// ------------------------------------------------------------------------
constexpr int kScanThreads = 256, kScanItems = 16, kScanChunk = kScanThreads * kScanItems;

template <class T> __device__ __forceinline__ T warp_incl_scan(T v)
{
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
    }
    return v;
}

// exclusive block scan of one value per thread; returns the block total in *total
template <class T> __device__ __forceinline__ T block_excl_scan(T v, T *smem_warp, T *total)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    T inc = warp_incl_scan(v);
    if (lane == 31) smem_warp[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        T w = lane < nw ? smem_warp[lane] : T(0);
        T wi = warp_incl_scan(w);
        if (lane < nw) smem_warp[lane] = wi - w;
        if (lane == nw - 1) smem_warp[32] = wi;
    }
    __syncthreads();
    T res = inc - v + smem_warp[warp];
    *total = smem_warp[32];
    __syncthreads();
    return res;
}

__global__ void __launch_bounds__(kScanThreads) k2_block_sums(const int *__restrict__ cnt, int64_t n,
                                                             long long *__restrict__ sums)
{
    __shared__ long long sw[33];
    int64_t base = (int64_t)blockIdx.x * kScanChunk;
    long long acc = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        int64_t idx = base + (int64_t)k * kScanThreads + threadIdx.x;
        if (idx < n) acc += cnt[idx];
    }
    long long tot;
    block_excl_scan<long long>(acc, sw, &tot);
    if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

// single block: exclusive scan of nb block sums in place, total -> *total
__global__ void __launch_bounds__(1024) k2_scan_sums(long long *sums, int nb, long long *total)
{
    __shared__ long long sw[33];
    long long carry = 0;
    for (int base = 0; base < nb; base += 1024) {
        int i = base + threadIdx.x;
        long long v = i < nb ? sums[i] : 0;
        long long tot;
        long long ex = block_excl_scan<long long>(v, sw, &tot);
        if (i < nb) sums[i] = ex + carry;
        carry += tot;
    }
    if (threadIdx.x == 0) *total = carry;
}

__global__ void __launch_bounds__(kScanThreads)
k2_rescan(const int *__restrict__ cnt, int64_t n, const long long *__restrict__ sums,
          uint32_t *__restrict__ offs)
{
    __shared__ long long sw[33];
    __shared__ int tile[kScanChunk];
    int64_t base = (int64_t)blockIdx.x * kScanChunk;
    // coalesced load into smem, then each thread scans a contiguous run of items
    for (int k = 0; k < kScanItems; ++k) {
        int64_t idx = base + (int64_t)k * kScanThreads + threadIdx.x;
        tile[k * kScanThreads + threadIdx.x] = idx < n ? cnt[idx] : 0;
    }
    __syncthreads();
    long long run = 0;
    int v[kScanItems];
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        v[k] = tile[threadIdx.x * kScanItems + k];
        run += v[k];
    }
    long long tot;
    long long ex = block_excl_scan<long long>(run, sw, &tot) + sums[blockIdx.x];
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        tile[threadIdx.x * kScanItems + k] = (int)(uint32_t)ex;  // low 32 bits (P < 2^32)
        ex += v[k];
    }
    __syncthreads();
    for (int k = 0; k < kScanItems; ++k) {
        int64_t idx = base + (int64_t)k * kScanThreads + threadIdx.x;
        if (idx < n) offs[idx] = (uint32_t)tile[k * kScanThreads + threadIdx.x];
    }
}

// small inputs (the per-block visible counts of a batch, a few thousand entries):
// one block walks the array in 1024-item steps with a running carry (one launch
// instead of three)
constexpr int64_t kScanSmall = 1 << 15;
__global__ void __launch_bounds__(1024) k2_scan_small(const int *__restrict__ cnt, int n,
                                                      uint32_t *__restrict__ offs, long long *total)
{
    __shared__ long long sw[33];
    long long carry = 0;
    for (int base = 0; base < n; base += 1024) {
        const int i = base + threadIdx.x;
        const long long v = i < n ? cnt[i] : 0;
        long long tot;
        const long long ex = block_excl_scan<long long>(v, sw, &tot);
        if (i < n) offs[i] = (uint32_t)(ex + carry);
        carry += tot;
    }
    if (threadIdx.x == 0 && total) *total = carry;
}

cudaError_t exclusive_scan_counts(pf_scene *s, const int *cnt, int64_t n, uint32_t *offs,
                                  long long *d_total, cudaStream_t st)
{
    if (n <= kScanSmall) {
        k2_scan_small<<<1, 1024, 0, st>>>(cnt, (int)n, offs, d_total);
        ++s->launches;
        return cudaGetLastError();
    }
    int nb = ceil_div(n, kScanChunk);
    cudaError_t err = s->scan_tmp.reserve(sizeof(long long) * (size_t)(nb + 1));
    if (err != cudaSuccess) return err;
    long long *sums = s->scan_tmp.as<long long>();
    k2_block_sums<<<nb, kScanThreads, 0, st>>>(cnt, n, sums);
    k2_scan_sums<<<1, 1024, 0, st>>>(sums, nb, d_total);
    k2_rescan<<<nb, kScanThreads, 0, st>>>(cnt, n, sums, offs);
    s->launches += 3;
    return cudaGetLastError();
}


// ------------------------------------------------------------------------
// Depth-first binning of a batch of up to kBatchViews views (replaces the
// 48-bit pair sort): every view's VISIBLE cells (count > 0) are compacted in
// cell order, sorted ONCE by (view, depth key) -- ~N_vis items instead of P
// pairs --, their tile pairs are emitted in that order with a 16-bit
// (view, tile) key, and a stable 2-pass radix sort by (view, tile) finishes:
// inside a tile the pairs keep the (depth key, cell) order of the emission,
// which is exactly the order of the stable (tile << 32 | key) sort of
// cell-major pairs (ties by cell index).
// ------------------------------------------------------------------------
constexpr int kVisThreads = 256, kVisItems = 8, kVisChunk = kVisThreads * kVisItems;

// KV1: per (view, block of kVisChunk cells): number of visible cells -> bvis,
// and the view's pair total (sum of counts) -> ptot[view] (atomics; integers)
__global__ void __launch_bounds__(kVisThreads)
kv1_count(BatchViews bv, int64_t N, int nbx, int *__restrict__ bvis, long long *__restrict__ ptot)
{
    __shared__ long long sw[33];
    __shared__ int swi[33];
    const int v = blockIdx.y;
    const int *cnt = bv.count[v];
    const int64_t base = (int64_t)blockIdx.x * kVisChunk;
    int nv = 0;
    long long sum = 0;
#pragma unroll
    for (int k = 0; k < kVisItems; ++k) {
        const int64_t i = base + (int64_t)k * kVisThreads + threadIdx.x;
        if (i < N) {
            const int c = cnt[i];
            nv += c > 0;
            sum += c;
        }
    }
    long long tot;
    block_excl_scan<long long>(sum, sw, &tot);
    int ntot;
    block_excl_scan<int>(nv, swi, &ntot);
    if (threadIdx.x == 0) {
        bvis[(size_t)(bv.first + v) * nbx + blockIdx.x] = ntot;
        if (tot) atomicAdd(reinterpret_cast<unsigned long long *>(ptot + bv.first + v),
                           (unsigned long long)tot);
    }
}

// KV2: compaction of the visible cells (view-major, ascending cell index) into
// (view << 32 | keybits, cell) at the scanned block offsets
__global__ void __launch_bounds__(kVisThreads)
kv2_compact(BatchViews bv, int64_t N, int nbx, const uint32_t *__restrict__ boff,
            unsigned long long *__restrict__ keys, uint32_t *__restrict__ vals)
{
    __shared__ int swi[33];
    const int v = blockIdx.y;
    const int *cnt = bv.count[v];
    const uint32_t *kb = bv.keybits[v];
    const int64_t base = (int64_t)blockIdx.x * kVisChunk + (int64_t)threadIdx.x * kVisItems;
    int f[kVisItems];
    int nv = 0;
#pragma unroll
    for (int k = 0; k < kVisItems; ++k) {
        const int64_t i = base + k;
        f[k] = (i < N) && cnt[i] > 0;
        nv += f[k];
    }
    int tot;
    int o = block_excl_scan<int>(nv, swi, &tot) + (int)boff[(size_t)v * nbx + blockIdx.x];
#pragma unroll
    for (int k = 0; k < kVisItems; ++k) {
        if (f[k]) {
            const int64_t i = base + k;
            keys[o] = ((unsigned long long)v << 32) | kb[i];
            vals[o] = (uint32_t)i;
            ++o;
        }
    }
}

// KV3: counts of the sorted visible cells (the emission sizes, in depth order)
__global__ void __launch_bounds__(256)
kv3_gather(BatchViews bv, const unsigned long long *__restrict__ keys,
           const uint32_t *__restrict__ vals, int64_t n, int *__restrict__ cnt_sorted)
{
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n) return;
    cnt_sorted[q] = bv.count[(int)(keys[q] >> 32)][vals[q]];
}

// KV4: emission in depth order, pinhole views (a warp writes its 32
// items' contiguous output range 32 pairs at a time), key = view << tb | tile
__global__ void __launch_bounds__(256)
kv4_emit(BatchViews bv, int tile_bits, const unsigned long long *__restrict__ skeys,
         const uint32_t *__restrict__ svals, const int *__restrict__ cnt_sorted,
         const uint32_t *__restrict__ offs, int64_t n, uint32_t *__restrict__ keys,
         uint32_t *__restrict__ vals)
{
    const int lane = threadIdx.x & 31;
    const int64_t i0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) & ~31ll;
    const int64_t i = i0 + lane;
    int cnt = 0, view = 0, tx = 1;
    uint32_t cell = 0, off = 0;
    int4 rc = make_int4(0, 0, 1, 0);
    if (i < n) {
        cnt = cnt_sorted[i];
        off = offs[i];
        view = (int)(skeys[i] >> 32);
        cell = svals[i];
        rc = bv.rect[view][cell];
        tx = bv.cam[view].tiles_x;
    }
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
    }
    const int excl = incl - cnt;
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    const uint32_t base = __shfl_sync(0xffffffffu, off, 0);
    const int w = rc.z - rc.x;
    const uint32_t vkey = (uint32_t)view << tile_bits;
    for (int p0 = 0; p0 < total; p0 += 32) {
        const int p = p0 + lane;
        int src = 0;
#pragma unroll
        for (int step = 16; step > 0; step >>= 1) {
            const int cand = src + step;
            const int ex = __shfl_sync(0xffffffffu, excl, cand & 31);
            if (cand < 32 && ex <= p) src = cand;
        }
        const int ex = __shfl_sync(0xffffffffu, excl, src);
        const int x0 = __shfl_sync(0xffffffffu, rc.x, src);
        const int y0 = __shfl_sync(0xffffffffu, rc.y, src);
        const int ww = __shfl_sync(0xffffffffu, w, src);
        const int tw = __shfl_sync(0xffffffffu, tx, src);
        const uint32_t vk = __shfl_sync(0xffffffffu, vkey, src);
        const uint32_t c = __shfl_sync(0xffffffffu, cell, src);
        if (p < total) {
            const int q = p - ex;
            const int dy = q / ww, dx = q - dy * ww;
            keys[base + p] = vk | (uint32_t)((y0 + dy) * tw + (x0 + dx));
            vals[base + p] = c;
        }
    }
}

// KV4 for batches with fisheye views: the warp's items one after another, the
// lanes over the item's candidate tiles (fisheye tiles re-tested as in
// K1 counted them; pinhole rects taken whole), ballot-compacted stores
__global__ void __launch_bounds__(256)
kv4_emit_items(BatchViews bv, int tile_bits, const float *__restrict__ sites,
               const float *__restrict__ radii, const unsigned long long *__restrict__ skeys,
               const uint32_t *__restrict__ svals, const uint32_t *__restrict__ offs, int64_t n,
               uint32_t *__restrict__ keys, uint32_t *__restrict__ vals)
{
    const int lane = threadIdx.x & 31;
    const int64_t i0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) & ~31ll;
    if (i0 >= n) return;
    const int m = (int)min((int64_t)32, n - i0);
    for (int src = 0; src < m; ++src) {
        const int64_t it = i0 + src;
        const int view = (int)(skeys[it] >> 32);
        const uint32_t cell = svals[it];
        const CamParams &cam = bv.cam[view];
        const int4 rc = bv.rect[view][cell];
        uint32_t o = offs[it];
        const uint32_t vkey = (uint32_t)view << tile_bits;
        const int w = rc.z - rc.x, cntt = w * (rc.w - rc.y);
        double c[3] = {0.0, 0.0, 0.0};
        double r = 0.0, cth = 0.0, sth = 0.0;
        const double *tdir = bv.tdir[view];
        const bool fish = cam.model == PF_FISHEYE;
        if (fish) {
            camera_coords(cam, sites + 3 * (size_t)cell, c);
            r = radii[cell];
            const int T = cam.tiles_x * cam.tiles_y;
            cth = __ldg(tdir + 3 * T);
            sth = __ldg(tdir + 3 * T + 1);
        }
        for (int b = 0; b < cntt; b += 32) {
            const int t = b + lane;
            const int tx = rc.x + (w ? t % w : 0), ty = rc.y + (w ? t / w : 0);
            const bool pass = t < cntt && (!fish || fisheye_tile_pass(cam, c, r, cth, sth, tx, ty, tdir));
            const unsigned msk = __ballot_sync(0xffffffffu, pass);
            if (pass) {
                const uint32_t q = o + __popc(msk & ((1u << lane) - 1u));
                keys[q] = vkey | (uint32_t)(ty * cam.tiles_x + tx);
                vals[q] = cell;
            }
            o += __popc(msk);
        }
    }
}

// debug export: full (tile << 32 | keybits) keys of a single-view call
__global__ void __launch_bounds__(256)
kv5_full_keys(const uint32_t *__restrict__ tkeys, const uint32_t *__restrict__ vals,
              const uint32_t *__restrict__ keybits, int64_t P, int tile_bits,
              unsigned long long *__restrict__ out)
{
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= P) return;
    const unsigned long long tile = tkeys[q] & ((1u << tile_bits) - 1u);
    out[q] = (tile << 32) | keybits[vals[q]];
}

cudaError_t launch_count_visible(pf_scene *s, const BatchViews &bv, int nbx, int *bvis,
                                 long long *ptot, cudaStream_t st)
{
    cudaEvent_t ev;
    stage_begin(s, 2, st, &ev);
    kv1_count<<<dim3(nbx, bv.n), kVisThreads, 0, st>>>(bv, s->ds.N, nbx, bvis, ptot);
    ++s->launches;
    stage_end(s, 2, st, ev);
    return cudaGetLastError();
}

int vis_blocks(int64_t N) { return ceil_div(N, kVisChunk); }

cudaError_t launch_compact_visible(pf_scene *s, const BatchViews &bv, int nbx, const int *bvis,
                                   uint32_t *boff, long long *d_nvis, unsigned long long *keys,
                                   uint32_t *vals, cudaStream_t st)
{
    cudaEvent_t ev;
    stage_begin(s, 2, st, &ev);
    cudaError_t err = exclusive_scan_counts(s, bvis + (size_t)bv.first * nbx, (int64_t)bv.n * nbx,
                                            boff, d_nvis, st);
    if (err != cudaSuccess) return err;
    kv2_compact<<<dim3(nbx, bv.n), kVisThreads, 0, st>>>(bv, s->ds.N, nbx, boff, keys, vals);
    ++s->launches;
    stage_end(s, 2, st, ev);
    return cudaGetLastError();
}

cudaError_t launch_emit_sorted(pf_scene *s, const BatchViews &bv, int tile_bits,
                               const unsigned long long *skeys, const uint32_t *svals, int64_t n,
                               int *cnt_sorted, uint32_t *offs, long long *d_tot,
                               uint32_t *keys, uint32_t *vals, cudaStream_t st)
{
    if (n == 0) return cudaSuccess;
    cudaEvent_t ev;
    stage_begin(s, 3, st, &ev);
    kv3_gather<<<ceil_div(n, 256), 256, 0, st>>>(bv, skeys, svals, n, cnt_sorted);
    ++s->launches;
    cudaError_t err = exclusive_scan_counts(s, cnt_sorted, n, offs, d_tot, st);
    if (err != cudaSuccess) return err;
    bool fish = false;
    for (int v = 0; v < bv.n; ++v) fish = fish || bv.cam[v].model == PF_FISHEYE;
    if (fish)
        kv4_emit_items<<<ceil_div(n, 256), 256, 0, st>>>(bv, tile_bits, s->ds.sites, s->ds.radii,
                                                          skeys, svals, offs, n, keys, vals);
    else
        kv4_emit<<<ceil_div(n, 256), 256, 0, st>>>(bv, tile_bits, skeys, svals, cnt_sorted, offs,
                                                    n, keys, vals);
    ++s->launches;
    stage_end(s, 3, st, ev);
    return cudaGetLastError();
}

cudaError_t launch_full_keys(pf_scene *s, const uint32_t *tkeys, const uint32_t *vals,
                             const uint32_t *keybits, int64_t P, int tile_bits, uint64_t *out,
                             cudaStream_t st)
{
    if (P == 0) return cudaSuccess;
    kv5_full_keys<<<ceil_div(P, 256), 256, 0, st>>>(tkeys, vals,
                                                    keybits, P, tile_bits,
                                                    (unsigned long long *)out);
    ++s->launches;
    return cudaGetLastError();
}

// ------------------------------------------------------------------------
// K5: per-tile ranges [start, end) of the sorted pairs ((0,0) for empty tiles)
// ------------------------------------------------------------------------
// keys of all views of a sort batch: (view << tile_bits) | tile (kv4_emit);
// ranges[view * T + tile] = [start, end) in the batch's sorted arrays.
__global__ void __launch_bounds__(256) k5_ranges(const uint32_t *__restrict__ keys,
                                                 int64_t P, int T, int tile_bits,
                                                 uint2 *__restrict__ ranges)
{
    int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= P) return;
    const uint32_t vt = keys[q];   // (view << tile_bits) | tile
    const uint32_t idx = (vt >> tile_bits) * (uint32_t)T + (vt & ((1u << tile_bits) - 1u));
    if (q == 0 || keys[q - 1] != vt) ranges[idx].x = (uint32_t)q;
    if (q == P - 1 || keys[q + 1] != vt) ranges[idx].y = (uint32_t)(q + 1);
}

// Grid order for K6/K7: tiles by decreasing list length (longest-processing-time
// first, so the long tiles do not form the tail of the launch).  Order within a
// length bucket is arbitrary: tiles are independent, results do not depend on it.
// Also writes chunk_off[t] = sum_{t' < t} ceil(len_t' / 32): the first 32-entry
// chunk of tile t in the per-view chunk-descriptor table of the K6 -> K7 records.
__global__ void __launch_bounds__(1024) k5_tile_order(const uint2 *__restrict__ ranges_all, int T,
                                                      uint32_t *__restrict__ order_all,
                                                      uint32_t *__restrict__ chunk_off_all)
{
    // one block per view
    const uint2 *ranges = ranges_all + (size_t)blockIdx.x * T;
    uint32_t *order = order_all + (size_t)blockIdx.x * T;
    uint32_t *chunk_off = chunk_off_all + (size_t)blockIdx.x * T;
    __shared__ int hist[64], off[64];
    __shared__ long long sw[33];
    if (threadIdx.x < 64) hist[threadIdx.x] = 0;
    long long carry = 0;
    for (int base = 0; base < T; base += 1024) {
        const int t = base + threadIdx.x;
        long long c = 0;
        if (t < T) {
            const uint2 r = ranges[t];
            c = (r.y - r.x + 31) / 32;
        }
        long long tot;
        const long long ex = block_excl_scan<long long>(c, sw, &tot);
        if (t < T) chunk_off[t] = (uint32_t)(carry + ex);
        carry += tot;
    }
    __syncthreads();
    auto bucket = [](uint32_t len) { return min(63, (int)(5.0f * __log2f((float)len + 1.0f))); };
    for (int t = threadIdx.x; t < T; t += blockDim.x) {
        const uint2 r = ranges[t];
        atomicAdd(&hist[bucket(r.y - r.x)], 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int run = 0;
        for (int b = 63; b >= 0; --b) {
            off[b] = run;
            run += hist[b];
        }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < T; t += blockDim.x) {
        const uint2 r = ranges[t];
        order[atomicAdd(&off[bucket(r.y - r.x)], 1)] = (uint32_t)t;
    }
}

cudaError_t launch_ranges(pf_scene *s, const uint32_t *keys, int64_t P, int T, int tile_bits,
                          uint2 *ranges_all, int V, cudaStream_t st)
{
    cudaError_t err = cudaMemsetAsync(ranges_all, 0, sizeof(uint2) * (size_t)T * V, st);
    if (err != cudaSuccess) return err;
    if (P == 0) return cudaSuccess;
    cudaEvent_t ev;
    stage_begin(s, 5, st, &ev);
    k5_ranges<<<ceil_div(P, 256), 256, 0, st>>>(keys, P, T, tile_bits,
                                                 ranges_all);
    ++s->launches;
    stage_end(s, 5, st, ev);
    return cudaGetLastError();
}

cudaError_t launch_tile_order(pf_scene *s, const uint2 *ranges_all, int T, int V,
                              uint32_t *order_all, uint32_t *chunk_off_all, cudaStream_t st)
{
    cudaEvent_t ev;
    stage_begin(s, 5, st, &ev);
    k5_tile_order<<<V, 1024, 0, st>>>(ranges_all, T, order_all, chunk_off_all);
    ++s->launches;
    stage_end(s, 5, st, ev);
    return cudaGetLastError();
}

}  // namespace pf
