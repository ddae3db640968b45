/*
 * pf_oracle.c -- plain, slow, obviously-correct CPU oracle for the Power Foam
 * rasterizer hot path (arXiv 2604.24994).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, constant or helper with the CUDA path
 * (paper_2604_24994_b200/csrc); the two meet only through the arrays of
 * pf_synth (the seeded generators).
 *
 * What it computes (citations: P:<line> = /root/reference/PAPER.md,
 * S:<line> = SPEC.md, SURVEY §x = /root/repo/SURVEY.md):
 *
 *  (1) The rendered image, by the plain definition.  For the
 *      pixel ray x(t) = Q + t d, t >= t_near, and every cell i:
 *        I_i = { t : |x(t)-p_i|^2 <= r_i^2                  (bounding sphere B_i,
 *                                                            P:189 "radius of a
 *                                                            bounding sphere")
 *                    pow(x(t),i) <= pow(x(t),j)  for all j  (power cell, P:570-573
 *                                                            Eq. power_cell)
 *                    t >= t_near }                          (near plane, C10)
 *      with pow(x,i) = |x-p_i|^2 - w_i  (P:565 Eq. pow_dist).  Every constraint
 *      is written straight from that definition: the sphere is a quadratic in
 *      t, and pow(x(t),i) - pow(x(t),j) = [pow(Q,i)-pow(Q,j)]
 *      + 2 t d.(p_j - p_i) is linear in t (the radical plane, P:577-585 with the
 *      sign of the weight term corrected).
 *      Non-empty intervals are sorted by entry t (ties by cell index) -- the
 *      order comes from the geometry, NOT from the sort key -- and composited
 *      front to back in double ("evaluated exactly as a sum over the
 *      segments"; alpha = 1-exp(-sigma dt); stop after the segment
 *      that makes T < 1e-4; out = (C + T bg, T), C5).
 *
 *      Candidate sets (which j enter the "for all j", which i are tried):
 *        O1: every cell is a candidate and every other cell is a plane
 *            (the literal definition);
 *        O2: every cell is a candidate; planes only from i's neighbour list
 *            (exact for Čech lists with w = r^2: P:230-235, SURVEY Lemma L1);
 *        O3: candidates are the cells of the pixel's tile list produced by the
 *            fp32 binning below (the paper's rasterisation algorithm, P:213,
 *            "global sort by depths ... similar to 3DGS"); planes from lists.
 *      O1 == O2 == O3 on shared pixels is itself a test.
 *
 *      Dipoles (NEXT-1): with per-cell normals n_i the cell is an
 *      oriented point whose occupied half is (x - p_i).n_i <= 0 (SPEC S:242:
 *      the side the normal points away from); the other half has zero density,
 *      so I_i is further intersected with that half-space.
 *
 *      Detail sites (NEXT-2, P:278-297 Eqs. svdisp/svrad): each
 *      dipole face carries K detail sites s_k in the face's 2D chart (the
 *      tangent frame of SPEC S:186-189), displacements d_k and per-site
 *      Spherical-Voronoi radiance (8 shared axes a_a, sharpness gamma).
 *      Step by step as P:284-293 describes it (with the readings R6 of
 *      DESIGN.md): x_bar = the ray's hit on the base face (x-p).n = 0;
 *      delta = sum_k softmax_k(-tau |q(x_bar) - s_k|) d_k (Eq. svdisp),
 *      clamped to [-r, r]; the occupied half becomes
 *      (x - p).n <= delta; x = the ray's hit on that displaced face; the
 *      segment colour is c(x) = sum_k softmax_k(-tau |q(x) - s_k|) c_k(d)
 *      (Eq. svrad) with c_k(d) = sum_a softmax_a(gamma d.a_a) v_{k,a}.
 *      q(y) = ((y-p).u, (y-p).v) are the chart coordinates.
 *
 *  (2) The backward pass: the exact derivative of (1) for a fixed active set
 *      and termination index, L = sum_pixels <grad_out, out> (
 *      endpoint derivatives of the sphere and the radical plane).
 *
 *  (3) The binning specification: per-cell
 *      screen rectangle of the bounding sphere, tile rectangle, count and the
 *      order-preserving bits of the sort key K_i = pow(Q, p_i) (P:596-603,
 *      Theorem 2), then the (tile<<32 | keybits, cell) pairs sorted stably and
 *      per-tile ranges.  This part is an fp32 *specification* (it defines
 *      integers, so it is evaluated in single precision, one IEEE op at a time,
 *      left to right, no FMA: compile with -ffp-contract=off).
 *
 * Pins: tests/test_oracle_*.py check every function here against values the
 * paper / SPEC print, closed forms, invariants, brute force and finite
 * differences.
 */
#include <float.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#if !defined(FLT_EVAL_METHOD) || FLT_EVAL_METHOD != 0
#error "the fp32 binning specification needs FLT_EVAL_METHOD == 0 (SSE float)"
#endif

typedef struct {
    int32_t width, height;
    float fx, fy, cx, cy;
    float c2w[12]; /* row-major [R | Q]: R[m][k] = c2w[4m+k], Q[m] = c2w[4m+3] */
    float near_plane;
    int32_t model; /* 0 pinhole, 1 equidistant fisheye (NEXT-4) */
} oc_camera;

typedef struct {
    int64_t N;
    const float *sites, *weights, *radii, *density, *rgb;
    const int64_t *nbr_off;
    const int32_t *nbr_idx;
    double bg[3];
    const float *normals; /* dipole normals n_i [N,3] or NULL (NEXT-1) */
    const struct oc_detail_s *det; /* detail sites (NEXT-2) or NULL */
} oc_scene;

/* Detail sites of the dipole faces (NEXT-2). */
#define OC_MAX_DETAIL 8
#define OC_SV_AXES 8
typedef struct oc_detail_s {
    int32_t K;           /* detail sites per cell, 1..8 (0 = none) */
    const float *uv;     /* s_{i,k} [N,K,2] chart coordinates (world units) */
    const float *disp;   /* d_{i,k} [N,K] displacement along the unit normal */
    const float *sv;     /* v_{i,k,a} [N,K,8,3] SV radiance per axis */
    float axes[OC_SV_AXES][3]; /* the shared SV axes a_a (unit) */
    float gamma;         /* SV sharpness */
    float tau;           /* soft-Voronoi temperature (1 / world units) */
} oc_detail;

#define O1_ALL_PAIRS 1
#define O2_LIST_PLANES 2
#define O3_TILE_LISTS 3

#define T_STOP 1e-4

/* ======================================================================== */
/* (3) fp32 binning specification                                           */
/* ======================================================================== */

static uint32_t key_bits(float K)
{
    /* order-preserving map float -> u32 */
    uint32_t u;
    memcpy(&u, &K, 4);
    return (u >> 31) ? ~u : (u ^ 0x80000000u);
}

/* screen-space extent of the sphere along one image axis.
 * a = camera-space coordinate along the axis (x or y), z = depth. */
static void axis_extent(float a, float z, float r, float f, float c, float near_plane,
                        int in_front, float *lo, float *hi)
{
    float ulo, uhi;
    if (in_front) {
        /* tangent planes through the camera centre containing the other axis */
        float q = sqrtf((a * a + z * z) - r * r);
        float den = (z - r) * (z + r);
        ulo = (a * z - r * q) / den;
        uhi = (a * z + r * q) / den;
    } else {
        /* sphere straddles the near plane: box [a-r,a+r] x [near, z+r] */
        float amin = a - r, amax = a + r;
        ulo = amin / (amin >= 0.0f ? z + r : near_plane);
        uhi = amax / (amax >= 0.0f ? near_plane : z + r);
    }
    *lo = f * ulo + c;
    *hi = f * uhi + c;
}

static float clampf_(float v, float lo, float hi)
{
    return fminf(fmaxf(v, lo), hi);
}

/* ---- equidistant fisheye (NEXT-4): pixel (u, v) -> a = (u-cx)/fx, b = (v-cy)/fy,
 * theta = |(a, b)|, camera ray (sin(theta) a/theta, sin(theta) b/theta, cos(theta))
 * (S:285); pixels with theta > pi are outside the image circle.  The map (a,b) ->
 * ray is 1-Lipschitz in angle, so every pixel ray of tile t lies within the angle
 * th = |(9/fx, 9/fy)| (8 px to the tile border + 1 px guard) of the ray through
 * the tile centre (16 tx + 8, 16 ty + 8); a sphere (c, r) in camera coordinates
 * can meet a ray of the tile only if  c.a_t >= cos(th) sqrt(|c|^2 - r^2) - sin(th) r
 * (angle(c, a_t) <= th + asin(r/|c|)), or if |c| <= r.  Binning = the tiles that
 * pass this test (evaluated in double; the candidate rectangle is any superset). */
static void fisheye_dir(const oc_camera *cam, double u, double v, double dc[3], int *valid)
{
    double a = (u - (double)cam->cx) / (double)cam->fx, b = (v - (double)cam->cy) / (double)cam->fy;
    double th = sqrt(a * a + b * b);
    *valid = th <= 3.14159265358979323846;
    if (th > 0.0) {
        double st = sin(th) / th;
        dc[0] = st * a;
        dc[1] = st * b;
        dc[2] = cos(th);
    } else {
        dc[0] = dc[1] = 0.0;
        dc[2] = 1.0;
    }
}

static int fisheye_tile_pass(const oc_camera *cam, const double c[3], double r, int tx, int ty)
{
    double cc = c[0] * c[0] + c[1] * c[1] + c[2] * c[2];
    if (cc <= r * r) return 1;
    double at[3];
    int valid;
    fisheye_dir(cam, 16.0 * tx + 8.0, 16.0 * ty + 8.0, at, &valid);
    double th = sqrt((9.0 / cam->fx) * (9.0 / cam->fx) + (9.0 / cam->fy) * (9.0 / cam->fy));
    double lhs = c[0] * at[0] + c[1] * at[1] + c[2] * at[2];
    double rhs = cos(th) * sqrt(cc - r * r) - sin(th) * r;
    return lhs >= rhs;
}

/* candidate tile rectangle of a sphere for the fisheye: the bounding box, in (a,b),
 * of the annular sector of directions within th + asin(r/|c|) of c (plus margin) */
static void fisheye_rect(const oc_camera *cam, const double c[3], double r, int tiles_x,
                         int tiles_y, int rc[4])
{
    double cc = sqrt(c[0] * c[0] + c[1] * c[1] + c[2] * c[2]);
    double th = sqrt((9.0 / cam->fx) * (9.0 / cam->fx) + (9.0 / cam->fy) * (9.0 / cam->fy));
    double amin, amax, bmin, bmax;
    const double PI = 3.14159265358979323846;
    if (cc <= r) {
        amin = bmin = -PI;
        amax = bmax = PI;
    } else {
        double beta = asin(r / cc) + th + 1e-6;
        double thc = acos(fmax(-1.0, fmin(1.0, c[2] / cc)));
        double phc = atan2(c[1], c[0]);
        double rmax = fmin(thc + beta, PI);
        if (thc - beta <= 0.0 || thc + beta >= PI) {
            amin = bmin = -rmax;
            amax = bmax = rmax;
        } else {
            double rmin = thc - beta;
            double dph = asin(fmin(1.0, sin(beta) / sin(thc)));
            double p0 = phc - dph, p1 = phc + dph;
            amin = bmin = 1e30;
            amax = bmax = -1e30;
            double cand[4] = {p0, p1, 0, 0};
            for (int k = 0; k < 2; ++k)
                for (int q = 0; q < 2; ++q) {
                    double rr = q ? rmax : rmin, ph = cand[k];
                    amin = fmin(amin, rr * cos(ph)); amax = fmax(amax, rr * cos(ph));
                    bmin = fmin(bmin, rr * sin(ph)); bmax = fmax(bmax, rr * sin(ph));
                }
            for (int k = -4; k <= 4; ++k) {   /* axis directions inside the sector */
                double ph = k * (PI / 2);
                if (ph >= p0 && ph <= p1) {
                    amin = fmin(amin, rmax * cos(ph)); amax = fmax(amax, rmax * cos(ph));
                    bmin = fmin(bmin, rmax * sin(ph)); bmax = fmax(bmax, rmax * sin(ph));
                }
            }
        }
    }
    double u0 = cam->cx + cam->fx * amin, u1 = cam->cx + cam->fx * amax;
    double v0 = cam->cy + cam->fy * bmin, v1 = cam->cy + cam->fy * bmax;
    rc[0] = (int)fmax(0.0, fmin((double)tiles_x, floor((u0 - 1.0) / 16.0)));
    rc[2] = (int)fmax(0.0, fmin((double)tiles_x, floor((u1 + 1.0) / 16.0) + 1.0));
    rc[1] = (int)fmax(0.0, fmin((double)tiles_y, floor((v0 - 1.0) / 16.0)));
    rc[3] = (int)fmax(0.0, fmin((double)tiles_y, floor((v1 + 1.0) / 16.0) + 1.0));
}

static void camera_coords(const oc_camera *cam, const float *p, double c[3])
{
    const float *M = cam->c2w;
    double v[3] = {(double)p[0] - M[3], (double)p[1] - M[7], (double)p[2] - M[11]};
    for (int k = 0; k < 3; ++k) c[k] = M[k] * v[0] + M[4 + k] * v[1] + M[8 + k] * v[2];
}

/* rect[4*i] = (tx0, ty0, tx1, ty1) half-open tile rectangle; count = area (pinhole)
 * or the number of tiles of the rectangle passing the fisheye test. */
int oracle_bin_cells(int64_t N, const float *sites, const float *weights, const float *radii,
                     const oc_camera *cam, int32_t *rect, int32_t *count, uint32_t *keybits)
{
    const int tiles_x = (cam->width + 15) / 16, tiles_y = (cam->height + 15) / 16;
    const float *M = cam->c2w;
    const float Q0 = M[3], Q1 = M[7], Q2 = M[11];
    for (int64_t i = 0; i < N; ++i) {
        float v0 = sites[3 * i + 0] - Q0;
        float v1 = sites[3 * i + 1] - Q1;
        float v2 = sites[3 * i + 2] - Q2;
        /* camera coordinates c = R^T v, c_k = (R0k v0 + R1k v1) + R2k v2 */
        float cxx = (M[0] * v0 + M[4] * v1) + M[8] * v2;
        float cyy = (M[1] * v0 + M[5] * v1) + M[9] * v2;
        float czz = (M[2] * v0 + M[6] * v1) + M[10] * v2;
        /* sort key: power distance of the camera centre */
        float K = ((v0 * v0 + v1 * v1) + v2 * v2) - weights[i];
        float r = radii[i];
        keybits[i] = key_bits(K);
        rect[4 * i + 0] = rect[4 * i + 1] = rect[4 * i + 2] = rect[4 * i + 3] = 0;
        count[i] = 0;
        if (cam->model == 1) {   /* fisheye: cull only inside the near ball */
            double c[3];
            camera_coords(cam, sites + 3 * i, c);
            double dist = sqrt(c[0] * c[0] + c[1] * c[1] + c[2] * c[2]);
            if (!(r > 0.0f) || dist + r <= (double)cam->near_plane) continue;
            int rc[4];
            fisheye_rect(cam, c, r, tiles_x, tiles_y, rc);
            int n = 0;
            for (int ty = rc[1]; ty < rc[3]; ++ty)
                for (int tx = rc[0]; tx < rc[2]; ++tx) n += fisheye_tile_pass(cam, c, r, tx, ty);
            if (n > 0) {
                for (int k = 0; k < 4; ++k) rect[4 * i + k] = rc[k];
                count[i] = n;
            }
            continue;
        }
        if (!(czz + r > cam->near_plane) || !(r > 0.0f))
            continue; /* entirely behind the near plane (or degenerate) */
        int in_front = (czz - r > cam->near_plane);
        float xlo, xhi, ylo, yhi;
        axis_extent(cxx, czz, r, cam->fx, cam->cx, cam->near_plane, in_front, &xlo, &xhi);
        axis_extent(cyy, czz, r, cam->fy, cam->cy, cam->near_plane, in_front, &ylo, &yhi);
        /* 1-pixel guard, 16-pixel tiles, clamp in float before the int conversion */
        float fx0 = clampf_(floorf((xlo - 1.0f) * 0.0625f), 0.0f, (float)tiles_x);
        float fx1 = clampf_(floorf((xhi + 1.0f) * 0.0625f) + 1.0f, 0.0f, (float)tiles_x);
        float fy0 = clampf_(floorf((ylo - 1.0f) * 0.0625f), 0.0f, (float)tiles_y);
        float fy1 = clampf_(floorf((yhi + 1.0f) * 0.0625f) + 1.0f, 0.0f, (float)tiles_y);
        int tx0 = (int)fx0, tx1 = (int)fx1, ty0 = (int)fy0, ty1 = (int)fy1;
        if (tx1 > tx0 && ty1 > ty0) {
            rect[4 * i + 0] = tx0;
            rect[4 * i + 1] = ty0;
            rect[4 * i + 2] = tx1;
            rect[4 * i + 3] = ty1;
            count[i] = (tx1 - tx0) * (ty1 - ty0);
        }
    }
    return 0;
}

typedef struct {
    uint64_t key;
    uint32_t val;
} oc_pair;

static int cmp_pair(const void *a, const void *b)
{
    const oc_pair *x = (const oc_pair *)a, *y = (const oc_pair *)b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    /* stable w.r.t. cell-major emission: equal keys keep cell order (C12) */
    if (x->val != y->val) return x->val < y->val ? -1 : 1;
    return 0;
}

/* Emits (tile<<32 | keybits, cell) in cell-major order and sorts stably.
 * Returns P (number of pairs); keys/vals may be NULL to query P. */
int64_t oracle_emit_sort(int64_t N, const int32_t *rect, const int32_t *count,
                         const uint32_t *keybits, int32_t tiles_x, uint64_t *keys, uint32_t *vals,
                         const oc_camera *cam, const float *sites, const float *radii)
{
    int64_t P = 0;
    for (int64_t i = 0; i < N; ++i) P += count[i];
    if (!keys || !vals) return P;
    oc_pair *pairs = (oc_pair *)malloc(sizeof(oc_pair) * (size_t)(P > 0 ? P : 1));
    int64_t k = 0;
    for (int64_t i = 0; i < N; ++i) {
        if (count[i] == 0) continue;
        double c[3] = {0, 0, 0};
        const int fish = cam && cam->model == 1;
        if (fish) camera_coords(cam, sites + 3 * i, c);
        for (int ty = rect[4 * i + 1]; ty < rect[4 * i + 3]; ++ty)
            for (int tx = rect[4 * i + 0]; tx < rect[4 * i + 2]; ++tx) {
                if (fish && !fisheye_tile_pass(cam, c, radii[i], tx, ty)) continue;
                uint64_t tile = (uint64_t)ty * (uint64_t)tiles_x + (uint64_t)tx;
                pairs[k].key = (tile << 32) | (uint64_t)keybits[i];
                pairs[k].val = (uint32_t)i;
                ++k;
            }
    }
    qsort(pairs, (size_t)P, sizeof(oc_pair), cmp_pair);
    for (int64_t q = 0; q < P; ++q) {
        keys[q] = pairs[q].key;
        vals[q] = pairs[q].val;
    }
    free(pairs);
    return P;
}

/* ranges[2t], ranges[2t+1] = [start, end) of tile t in the sorted keys; (0,0) if empty */
int oracle_tile_ranges(int64_t P, const uint64_t *keys, int32_t num_tiles, uint32_t *ranges)
{
    memset(ranges, 0, sizeof(uint32_t) * 2 * (size_t)num_tiles);
    for (int64_t q = 0; q < P; ++q) {
        uint32_t t = (uint32_t)(keys[q] >> 32);
        if (q == 0 || (uint32_t)(keys[q - 1] >> 32) != t) ranges[2 * t] = (uint32_t)q;
        if (q == P - 1 || (uint32_t)(keys[q + 1] >> 32) != t) ranges[2 * t + 1] = (uint32_t)(q + 1);
    }
    return 0;
}

/* ======================================================================== */
/* (1) rays, intervals, compositing in double                               */
/* ======================================================================== */

/* ray through the centre of pixel (px, py) = (x+0.5, y+0.5) (C11):
 * d_cam = ((px-cx)/fx, (py-cy)/fy, 1), d = normalize(R d_cam),
 * t_near = near * |d_cam| (C10: camera-space z >= near). */
static int pixel_ray(const oc_camera *cam, double px, double py, double Q[3], double d[3],
                     double *t_near)
{
    const float *M = cam->c2w;
    double dc[3] = {(px - (double)cam->cx) / (double)cam->fx,
                    (py - (double)cam->cy) / (double)cam->fy, 1.0};
    int valid = 1;
    if (cam->model == 1) fisheye_dir(cam, px, py, dc, &valid);
    double ndc = sqrt(dc[0] * dc[0] + dc[1] * dc[1] + dc[2] * dc[2]);
    double n2 = 0.0;
    for (int m = 0; m < 3; ++m) {
        d[m] = (double)M[4 * m + 0] * dc[0] + (double)M[4 * m + 1] * dc[1] +
               (double)M[4 * m + 2] * dc[2];
        n2 += d[m] * d[m];
        Q[m] = (double)M[4 * m + 3];
    }
    double nd = sqrt(n2);
    for (int m = 0; m < 3; ++m) d[m] /= nd;
    /* pinhole: camera-space z >= near (C10); fisheye: distance >= near (reading R5) */
    *t_near = (double)cam->near_plane * (cam->model == 1 ? 1.0 : ndc);
    return valid;
}

/* which constraint bounds an interval end */
#define END_SPHERE 0
#define END_NEAR 1
#define END_PLANE 2
#define END_DIPOLE 3 /* the cell's internal oriented face (NEXT-1) */

typedef struct {
    double t_in, t_out;
    int32_t cell;
    int32_t kin, kout;   /* END_* */
    int32_t jin, jout;   /* neighbour cell for END_PLANE */
    int32_t list_pos;    /* position in the tile list (O3), else -1 */
    double col[3];       /* segment radiance: rgb_i, or c(x) of the detail sites */
} oc_seg;

static double powd(const double x[3], const float *p, float w)
{
    double a = x[0] - p[0], b = x[1] - p[1], c = x[2] - p[2];
    return a * a + b * b + c * c - (double)w;
}

/* ---- detail sites (NEXT-2) --------------------------------------------- */

static double dot3(const double a[3], const double b[3])
{
    return a[0] * b[0] + a[1] * b[1] + a[2] * b[2];
}

static void cross3(const double a[3], const double b[3], double o[3])
{
    o[0] = a[1] * b[2] - a[2] * b[1];
    o[1] = a[2] * b[0] - a[0] * b[2];
    o[2] = a[0] * b[1] - a[1] * b[0];
}

/* Tangent frame of the face: m = n/|n|; k = the axis of the
 * smallest |n_k| (strictly smaller than the others for x, ties -> the higher
 * index); u = (e_k x m)/|e_k x m|, v = m x u, so (u, v, m) is right-handed and
 * n = (0,0,1) gives u = (1,0,0), v = (0,1,0). */
typedef struct {
    double m[3], u[3], v[3];
    double nn, wl; /* |n|, |e_k x m| */
    int kax;
} oc_frame;

static void tangent_frame(const float *n, oc_frame *F)
{
    F->nn = sqrt((double)n[0] * n[0] + (double)n[1] * n[1] + (double)n[2] * n[2]);
    for (int c = 0; c < 3; ++c) F->m[c] = (double)n[c] / F->nn;
    const float ax = fabsf(n[0]), ay = fabsf(n[1]), az = fabsf(n[2]);
    F->kax = (ax < ay && ax < az) ? 0 : (ay <= az ? 1 : 2);
    double e[3] = {0, 0, 0}, w[3];
    e[F->kax] = 1.0;
    cross3(e, F->m, w);
    F->wl = sqrt(dot3(w, w));
    for (int c = 0; c < 3; ++c) F->u[c] = w[c] / F->wl;
    cross3(F->m, F->u, F->v);
}

/* soft-Voronoi weights (Eqs. svdisp/svrad): w_k = exp(-tau rho_k) /
 * sum_j exp(-tau rho_j), rho_k = |q - s_k|, with max-subtraction */
static void soft_voronoi(const double q[2], const float *uv, int K, double tau, double rho[],
                         double w[])
{
    double zmax = -HUGE_VAL, z[OC_MAX_DETAIL], sum = 0.0;
    for (int k = 0; k < K; ++k) {
        double a = q[0] - uv[2 * k], b = q[1] - uv[2 * k + 1];
        rho[k] = sqrt(a * a + b * b);
        z[k] = -tau * rho[k];
        if (z[k] > zmax) zmax = z[k];
    }
    for (int k = 0; k < K; ++k) {
        w[k] = exp(z[k] - zmax);
        sum += w[k];
    }
    for (int k = 0; k < K; ++k) w[k] /= sum;
}

/* Everything the detail evaluation of one (ray, cell) computes, in the order of
 * P:284-293.  Vectors from p_i: c = p - Q, y = x_bar - p, ys = x - p. */
typedef struct {
    oc_frame F;
    double c[3], A, B;         /* A = d.m, B = c.m */
    int parallel;              /* A == 0: no base-face hit (reading R6e) */
    double tb, y[3], qb[2], rho[OC_MAX_DETAIL], w[OC_MAX_DETAIL];
    double dr, delta;          /* sum_k w_k d_k and its clamp to [-r, r] */
    int clamp;                 /* 0, +1 (delta = r), -1 (delta = -r) */
    double ts, ys[3], qs[2], rhos[OC_MAX_DETAIL], ws[OC_MAX_DETAIL];
    double om[OC_SV_AXES];     /* softmax_a(gamma d.a_a) */
    double ck[OC_MAX_DETAIL][3], col[3];
} oc_dstate;

/* steps 1-3 of P:284-289: base-face hit, displacement, displaced-face hit t* */
static void detail_geometry(const oc_scene *S, int64_t i, const double Q[3], const double d[3],
                            oc_dstate *D)
{
    const oc_detail *X = S->det;
    const float *p = S->sites + 3 * i;
    const int K = X->K;
    tangent_frame(S->normals + 3 * i, &D->F);
    for (int c = 0; c < 3; ++c) D->c[c] = (double)p[c] - Q[c];
    D->A = dot3(d, D->F.m);
    D->B = dot3(D->c, D->F.m);
    D->parallel = (D->A == 0.0);
    D->delta = 0.0;
    D->clamp = 0;
    if (D->parallel) return;
    /* x_bar: (Q + t d - p).m = 0 */
    D->tb = D->B / D->A;
    for (int c = 0; c < 3; ++c) D->y[c] = D->tb * d[c] - D->c[c];
    D->qb[0] = dot3(D->y, D->F.u);
    D->qb[1] = dot3(D->y, D->F.v);
    soft_voronoi(D->qb, X->uv + (size_t)2 * K * i, K, (double)X->tau, D->rho, D->w);
    D->dr = 0.0;
    for (int k = 0; k < K; ++k) D->dr += D->w[k] * (double)X->disp[(size_t)K * i + k];
    const double r = (double)S->radii[i];
    D->delta = D->dr;
    if (D->dr > r) {
        D->delta = r;
        D->clamp = 1;
    } else if (D->dr < -r) {
        D->delta = -r;
        D->clamp = -1;
    }
    /* x on the displaced face (Q + t d - p).m = delta */
    D->ts = (D->B + D->delta) / D->A;
}

/* step 4 (Eq. svrad): the radiance at x = p + ys (the parallel case uses the
 * interval's entry point, reading R6e) */
static void detail_radiance(const oc_scene *S, int64_t i, const double d[3], double t_entry,
                            oc_dstate *D)
{
    const oc_detail *X = S->det;
    const int K = X->K;
    const double t = D->parallel ? t_entry : D->ts;
    for (int c = 0; c < 3; ++c) D->ys[c] = t * d[c] - D->c[c];
    D->qs[0] = dot3(D->ys, D->F.u);
    D->qs[1] = dot3(D->ys, D->F.v);
    soft_voronoi(D->qs, X->uv + (size_t)2 * K * i, K, (double)X->tau, D->rhos, D->ws);
    double z[OC_SV_AXES], zmax = -HUGE_VAL, sum = 0.0;
    for (int a = 0; a < OC_SV_AXES; ++a) {
        z[a] = (double)X->gamma * (d[0] * X->axes[a][0] + d[1] * X->axes[a][1] +
                                   d[2] * X->axes[a][2]);
        if (z[a] > zmax) zmax = z[a];
    }
    for (int a = 0; a < OC_SV_AXES; ++a) {
        D->om[a] = exp(z[a] - zmax);
        sum += D->om[a];
    }
    for (int a = 0; a < OC_SV_AXES; ++a) D->om[a] /= sum;
    D->col[0] = D->col[1] = D->col[2] = 0.0;
    for (int k = 0; k < K; ++k) {
        const float *vk = X->sv + ((size_t)K * i + k) * OC_SV_AXES * 3;
        for (int c = 0; c < 3; ++c) {
            D->ck[k][c] = 0.0;
            for (int a = 0; a < OC_SV_AXES; ++a) D->ck[k][c] += D->om[a] * (double)vk[3 * a + c];
            D->col[c] += D->ws[k] * D->ck[k][c];
        }
    }
}

/* Interval of cell i along the ray.  Returns 1 (and fills *s) if the ray meets
 * the sphere of i after t_near (a "hit"), 0 otherwise; s->t_out > s->t_in iff
 * the bounded power cell has a non-empty intersection with the ray.
 * mode O1: planes against every j != i (index order); O2/O3: against i's list.
 * *nplanes receives the number of plane evaluations (counter X_p). */
static int cell_interval(const oc_scene *S, int mode, int64_t i, const double Q[3],
                         const double d[3], double t_near, oc_seg *s, int64_t *nplanes)
{
    const float *p = S->sites + 3 * i;
    double c[3] = {p[0] - Q[0], p[1] - Q[1], p[2] - Q[2]};
    /* |Q + t d - p|^2 <= r^2  <=>  (t - tc)^2 <= r^2 - |c - tc d|^2 */
    double tc = d[0] * c[0] + d[1] * c[1] + d[2] * c[2];
    double e[3] = {c[0] - tc * d[0], c[1] - tc * d[1], c[2] - tc * d[2]};
    double r = (double)S->radii[i];
    double h = r * r - (e[0] * e[0] + e[1] * e[1] + e[2] * e[2]);
    if (!(h > 0.0)) return 0;
    double sq = sqrt(h);
    if (!(tc + sq > t_near)) return 0;
    s->cell = (int32_t)i;
    s->list_pos = -1;
    for (int c = 0; c < 3; ++c) s->col[c] = S->rgb ? (double)S->rgb[3 * i + c] : 0.0;
    s->t_in = tc - sq;
    s->kin = END_SPHERE;
    s->jin = -1;
    s->t_out = tc + sq;
    s->kout = END_SPHERE;
    s->jout = -1;
    if (t_near > s->t_in) {
        s->t_in = t_near;
        s->kin = END_NEAR;
    }
    double powQi = powd(Q, p, S->weights[i]);
    int64_t jb, je;
    if (mode == O1_ALL_PAIRS) {
        jb = 0;
        je = S->N;
    } else {
        jb = S->nbr_off[i];
        je = S->nbr_off[i + 1];
    }
    int empty = 0;
    for (int64_t q = jb; q < je; ++q) {
        int64_t j = (mode == O1_ALL_PAIRS) ? q : (int64_t)S->nbr_idx[q];
        if (j == i) continue;
        const float *pj = S->sites + 3 * j;
        ++*nplanes;
        /* pow(x(t),i) <= pow(x(t),j)  <=>  A t <= B */
        double A = 2.0 * (d[0] * ((double)pj[0] - p[0]) + d[1] * ((double)pj[1] - p[1]) +
                          d[2] * ((double)pj[2] - p[2]));
        double B = powd(Q, pj, S->weights[j]) - powQi;
        if (A > 0.0) {
            double t = B / A;
            if (t < s->t_out) {
                s->t_out = t;
                s->kout = END_PLANE;
                s->jout = (int32_t)j;
            }
        } else if (A < 0.0) {
            double t = B / A;
            if (t > s->t_in) {
                s->t_in = t;
                s->kin = END_PLANE;
                s->jin = (int32_t)j;
            }
        } else if (B < 0.0) {
            empty = 1; /* ray parallel to the plane, on j's side (C14) */
        }
    }
    if (S->det && S->det->K > 0) {
        /* detail sites (NEXT-2): the occupied half is (x - p).m <= delta, delta
         * from the soft-Voronoi displacement at the base-face hit */
        oc_dstate D;
        detail_geometry(S, i, Q, d, &D);
        if (D.parallel) {
            if (D.B < 0.0) empty = 1; /* (x - p).m = -B > 0 = delta everywhere */
        } else if (D.A > 0.0) {
            if (D.ts < s->t_out) {
                s->t_out = D.ts;
                s->kout = END_DIPOLE;
                s->jout = -1;
            }
        } else if (D.ts > s->t_in) {
            s->t_in = D.ts;
            s->kin = END_DIPOLE;
            s->jin = -1;
        }
        detail_radiance(S, i, d, s->t_in, &D);
        for (int c = 0; c < 3; ++c) s->col[c] = D.col[c];
    } else if (S->normals) {
        /* oriented-point dipole: only the half-space the normal points
         * away from is occupied, (x - p_i).n_i <= 0 (SPEC S:242 convention);
         * (x(t) - p_i).n_i = (Q - p_i).n_i + t d.n_i  ->  A t <= B */
        const float *n = S->normals + 3 * i;
        double A = d[0] * n[0] + d[1] * n[1] + d[2] * n[2];
        double B = ((double)p[0] - Q[0]) * n[0] + ((double)p[1] - Q[1]) * n[1] +
                   ((double)p[2] - Q[2]) * n[2];
        if (A > 0.0) {
            double t = B / A;
            if (t < s->t_out) {
                s->t_out = t;
                s->kout = END_DIPOLE;
                s->jout = -1;
            }
        } else if (A < 0.0) {
            double t = B / A;
            if (t > s->t_in) {
                s->t_in = t;
                s->kin = END_DIPOLE;
                s->jin = -1;
            }
        } else if (B < 0.0) {
            empty = 1;
        }
    }
    if (empty) s->t_out = s->t_in;
    return 1;
}

static int cmp_seg(const void *a, const void *b)
{
    const oc_seg *x = (const oc_seg *)a, *y = (const oc_seg *)b;
    if (x->t_in != y->t_in) return x->t_in < y->t_in ? -1 : 1;
    return x->cell < y->cell ? -1 : (x->cell > y->cell);
}

/* per-thread scratch */
typedef struct {
    oc_seg *segs;
    int64_t cap;
} oc_scratch;

static void scratch_reserve(oc_scratch *s, int64_t n)
{
    if (n > s->cap) {
        free(s->segs);
        s->cap = n;
        s->segs = (oc_seg *)malloc(sizeof(oc_seg) * (size_t)n);
    }
}

/* binning products needed by O3 */
typedef struct {
    int32_t tiles_x, tiles_y;
    uint32_t *vals;   /* sorted cell ids */
    uint32_t *ranges; /* [T][2] */
} oc_bins;

static int build_bins(const oc_scene *S, const oc_camera *cam, oc_bins *B)
{
    int64_t N = S->N;
    B->tiles_x = (cam->width + 15) / 16;
    B->tiles_y = (cam->height + 15) / 16;
    int32_t T = B->tiles_x * B->tiles_y;
    int32_t *rect = (int32_t *)malloc(sizeof(int32_t) * 4 * (size_t)N);
    int32_t *count = (int32_t *)malloc(sizeof(int32_t) * (size_t)N);
    uint32_t *kb = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)N);
    oracle_bin_cells(N, S->sites, S->weights, S->radii, cam, rect, count, kb);
    int64_t P = oracle_emit_sort(N, rect, count, kb, B->tiles_x, NULL, NULL, cam, S->sites,
                                 S->radii);
    uint64_t *keys = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(P > 0 ? P : 1));
    B->vals = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)(P > 0 ? P : 1));
    oracle_emit_sort(N, rect, count, kb, B->tiles_x, keys, B->vals, cam, S->sites, S->radii);
    B->ranges = (uint32_t *)malloc(sizeof(uint32_t) * 2 * (size_t)T);
    oracle_tile_ranges(P, keys, T, B->ranges);
    free(rect);
    free(count);
    free(kb);
    free(keys);
    return 0;
}

static void free_bins(oc_bins *B)
{
    free(B->vals);
    free(B->ranges);
}

/* Collects the non-empty segments of one pixel ray, sorted by entry t.
 * counters (O3 only, list order):
 *   cnt[0] = X_s list entries examined up to termination,
 *   cnt[1] = X_h sphere hits among them, cnt[2] = X_p plane evaluations of
 *   those hits, cnt[3] = X_c composited segments; *viol = number of segment
 *   pairs whose key (list) order disagrees with entry order (Theorem 2). */
static int64_t collect_segments(const oc_scene *S, int mode, const oc_bins *B, int x, int y,
                                const double Q[3], const double d[3], double t_near,
                                oc_scratch *scr, int64_t *hits_planes, int64_t *viol)
{
    int64_t nseg = 0, np = 0;
    if (mode == O3_TILE_LISTS) {
        int t = (y / 16) * B->tiles_x + (x / 16);
        uint32_t b = B->ranges[2 * t], e = B->ranges[2 * t + 1];
        scratch_reserve(scr, (int64_t)(e - b) + 1);
        for (uint32_t q = b; q < e; ++q) {
            oc_seg s;
            int64_t npc = 0;
            if (cell_interval(S, mode, B->vals[q], Q, d, t_near, &s, &npc)) {
                s.list_pos = (int32_t)(q - b);
                /* record every hit (even empty ones) for the counters */
                scr->segs[nseg++] = s;
            }
            np += npc;
        }
    } else {
        scratch_reserve(scr, S->N + 1);
        for (int64_t i = 0; i < S->N; ++i) {
            oc_seg s;
            if (cell_interval(S, mode, i, Q, d, t_near, &s, &np)) scr->segs[nseg++] = s;
        }
    }
    (void)hits_planes;
    /* keep non-empty intervals (dt > 0) */
    int64_t k = 0;
    for (int64_t q = 0; q < nseg; ++q)
        if (scr->segs[q].t_out > scr->segs[q].t_in) scr->segs[k++] = scr->segs[q];
    qsort(scr->segs, (size_t)k, sizeof(oc_seg), cmp_seg);
    if (viol && mode == O3_TILE_LISTS)
        for (int64_t q = 1; q < k; ++q)
            if (scr->segs[q].list_pos < scr->segs[q - 1].list_pos) ++*viol;
    return k;
}

/* Front-to-back compositing; returns K (number of composited segments, the
 * termination index).  out[4] = (C + T bg, T). */
static int64_t composite(const oc_scene *S, const oc_seg *segs, int64_t n, double out[4])
{
    double T = 1.0, C[3] = {0, 0, 0};
    int64_t k = 0;
    for (; k < n;) {
        const oc_seg *s = segs + k;
        double sig = (double)S->density[s->cell];
        double tau = sig * (s->t_out - s->t_in);
        double alpha = 1.0 - exp(-tau);
        for (int c = 0; c < 3; ++c) C[c] += T * alpha * s->col[c];
        T *= exp(-tau);
        ++k;
        if (T < T_STOP) break;
    }
    for (int c = 0; c < 3; ++c) out[c] = C[c] + T * S->bg[c];
    out[3] = T;
    return k;
}

static uint64_t mix64(uint64_t h, uint64_t v)
{
    h ^= v + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
    return h;
}

static void pixel_counters(const oc_scene *S, const oc_bins *B, int x, int y, const double Q[3],
                           const double d[3], double t_near, const oc_seg *segs, int64_t K,
                           int terminated, int64_t *cnt)
{
    /* list-order counters of the tile walk up to the terminating entry */
    int t = (y / 16) * B->tiles_x + (x / 16);
    uint32_t b = B->ranges[2 * t], e = B->ranges[2 * t + 1];
    int64_t last = (int64_t)(e - b) - 1;
    if (terminated && K > 0) last = segs[K - 1].list_pos;
    int64_t xs = 0, xh = 0, xp = 0;
    for (int64_t q = 0; q <= last; ++q) {
        oc_seg s;
        int64_t npc = 0;
        ++xs;
        if (cell_interval(S, O3_TILE_LISTS, B->vals[b + q], Q, d, t_near, &s, &npc)) {
            ++xh;
            xp += npc;
        }
    }
    cnt[0] = xs;
    cnt[1] = xh;
    cnt[2] = xp;
    cnt[3] = K;
}

static void make_scene(oc_scene *S, int64_t N, const float *sites, const float *weights,
                       const float *radii, const float *density, const float *rgb,
                       const int64_t *nbr_off, const int32_t *nbr_idx, const float *bg,
                       const float *normals, const oc_detail *det)
{
    S->normals = normals;
    S->det = (det && det->K > 0 && normals) ? det : NULL;
    S->N = N;
    S->sites = sites;
    S->weights = weights;
    S->radii = radii;
    S->density = density;
    S->rgb = rgb;
    S->nbr_off = nbr_off;
    S->nbr_idx = nbr_idx;
    for (int c = 0; c < 3; ++c) S->bg[c] = bg ? (double)bg[c] : 0.0;
}

/*
 * Render npix pixels (pix_xy = int32 pairs (x,y); NULL = the full image,
 * row-major).  out: double[npix*4].  Optional outputs (may be NULL):
 *   counters int64[npix*4] (O3 only), sig uint64[npix] (hash of the active-set
 *   signature: cells, end kinds, plane ids, termination index), nseg int64[npix],
 *   viol int64[1] (Theorem-2 order violations, O3 only).
 */
int oracle_render(int mode, int64_t N, const float *sites, const float *weights,
                  const float *radii, const float *density, const float *rgb,
                  const int64_t *nbr_off, const int32_t *nbr_idx, const float *bg,
                  const float *normals, const oc_detail *det, const oc_camera *cam, int64_t npix, const int32_t *pix_xy, double *out,
                  int64_t *counters, uint64_t *sig, int64_t *nseg_out, int64_t *viol,
                  int nthreads)
{
    oc_scene S;
    make_scene(&S, N, sites, weights, radii, density, rgb, nbr_off, nbr_idx, bg, normals, det);
    oc_bins B;
    memset(&B, 0, sizeof(B));
    if (mode == O3_TILE_LISTS || counters) build_bins(&S, cam, &B);
    if (!pix_xy) npix = (int64_t)cam->width * cam->height;
    int64_t total_viol = 0;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel reduction(+ : total_viol)
    {
        oc_scratch scr = {NULL, 0};
#pragma omp for schedule(dynamic, 16)
        for (int64_t q = 0; q < npix; ++q) {
            int x = pix_xy ? pix_xy[2 * q] : (int)(q % cam->width);
            int y = pix_xy ? pix_xy[2 * q + 1] : (int)(q / cam->width);
            double Q[3], d[3], tn;
            const int pv = pixel_ray(cam, x + 0.5, y + 0.5, Q, d, &tn);
            int64_t v = 0;
            int64_t n = pv ? collect_segments(&S, mode, &B, x, y, Q, d, tn, &scr, NULL, &v) : 0;
            total_viol += v;
            int64_t K = composite(&S, scr.segs, n, out + 4 * q);
            if (counters) {
                if (pv)
                    pixel_counters(&S, &B, x, y, Q, d, tn, scr.segs, K, out[4 * q + 3] < T_STOP,
                                   counters + 4 * q);
                else
                    counters[4 * q] = counters[4 * q + 1] = counters[4 * q + 2] = counters[4 * q + 3] = 0;
            }
            if (nseg_out) nseg_out[q] = K;
            if (sig) {
                uint64_t h = 1469598103934665603ull;
                for (int64_t k = 0; k < K; ++k) {
                    const oc_seg *s = scr.segs + k;
                    h = mix64(h, (uint64_t)s->cell);
                    h = mix64(h, (uint64_t)(s->kin * 4 + s->kout));
                    h = mix64(h, (uint64_t)(uint32_t)s->jin);
                    h = mix64(h, (uint64_t)(uint32_t)s->jout);
                }
                h = mix64(h, (uint64_t)K);
                sig[q] = h;
            }
        }
        free(scr.segs);
    }
    if (viol) *viol = total_viol;
    if (B.vals) free_bins(&B);
    return 0;
}

/*
 * Per-cell by-products of the forward (NEXT-1; P:308 pruning statistic, P:728
 * L_sparse, P:718 L_normal): over the given pixels and their composited
 * segments k (termination as in composite()),
 *   contrib[i]     += T_k alpha_k
 *   normal_term[i] += T_k alpha_k max(n_i . d, 0)^2      (needs dipole normals)
 * Accumulates (+=) into double arrays; normal_term may be NULL.
 */
int oracle_cell_stats(int mode, int64_t N, const float *sites, const float *weights,
                      const float *radii, const float *density, const float *rgb,
                      const int64_t *nbr_off, const int32_t *nbr_idx, const float *bg,
                      const float *normals, const oc_detail *det, const oc_camera *cam, int64_t npix,
                      const int32_t *pix_xy, double *contrib, double *normal_term, int nthreads)
{
    oc_scene S;
    make_scene(&S, N, sites, weights, radii, density, rgb, nbr_off, nbr_idx, bg, normals, det);
    oc_bins B;
    memset(&B, 0, sizeof(B));
    if (mode == O3_TILE_LISTS) build_bins(&S, cam, &B);
    if (!pix_xy) npix = (int64_t)cam->width * cam->height;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel
    {
        oc_scratch scr = {NULL, 0};
#pragma omp for schedule(dynamic, 16)
        for (int64_t q = 0; q < npix; ++q) {
            int x = pix_xy ? pix_xy[2 * q] : (int)(q % cam->width);
            int y = pix_xy ? pix_xy[2 * q + 1] : (int)(q / cam->width);
            double Q[3], d[3], tn, out[4];
            const int pv = pixel_ray(cam, x + 0.5, y + 0.5, Q, d, &tn);
            int64_t n = pv ? collect_segments(&S, mode, &B, x, y, Q, d, tn, &scr, NULL, NULL) : 0;
            int64_t K = composite(&S, scr.segs, n, out);
            double T = 1.0;
            for (int64_t k = 0; k < K; ++k) {
                const oc_seg *sg = scr.segs + k;
                int64_t i = sg->cell;
                double tau = (double)S.density[i] * (sg->t_out - sg->t_in);
                double w = T * (1.0 - exp(-tau));
#pragma omp atomic
                contrib[i] += w;
                if (normal_term && normals) {
                    const float *nn = normals + 3 * i;
                    double nd = nn[0] * d[0] + nn[1] * d[1] + nn[2] * d[2];
                    double m = nd > 0.0 ? nd : 0.0;
#pragma omp atomic
                    normal_term[i] += w * m * m;
                }
                T *= exp(-tau);
            }
        }
        free(scr.segs);
    }
    if (B.vals) free_bins(&B);
    return 0;
}

/* ======================================================================== */
/* (2) backward                                                             */
/* ======================================================================== */

/* d t_end / d theta for one interval end (absolute t), SURVEY App. A.
 *   sphere end:  dt/dp_i = (x*-p_i)/(d.(x*-p_i)),  dt/dr_i = r_i/(d.(x*-p_i))
 *   plane end (i,j): dt/dp_i = (x*-p_i)/a, dt/dp_j = (p_j-x*)/a,
 *                    dt/dw_i = 1/(2a),   dt/dw_j = -1/(2a),  a = d.(p_j-p_i)
 *   near end: 0.
 * Adds sgn * gdt * (those) into the gradient arrays. */
static void end_grad(const oc_scene *S, int kind, int64_t i, int64_t j, double t,
                     const double Q[3], const double d[3], double sgn_gdt, double *g_sites,
                     double *g_w, double *g_r, double *g_normals)
{
    if (kind == END_NEAR) return;
    const float *p = S->sites + 3 * i;
    double x[3] = {Q[0] + t * d[0], Q[1] + t * d[1], Q[2] + t * d[2]};
    double xp[3] = {x[0] - p[0], x[1] - p[1], x[2] - p[2]};
    if (kind == END_DIPOLE) {
        /* t* = (p - Q).n / (d.n):  dt/dp_i = n/a,  dt/dn_i = (p_i - x*)/a,  a = d.n */
        const float *n = S->normals + 3 * i;
        double a = d[0] * n[0] + d[1] * n[1] + d[2] * n[2];
        for (int m = 0; m < 3; ++m) {
#pragma omp atomic
            g_sites[3 * i + m] += sgn_gdt * (double)n[m] / a;
            if (g_normals) {
#pragma omp atomic
                g_normals[3 * i + m] -= sgn_gdt * xp[m] / a;
            }
        }
        return;
    }
    if (kind == END_SPHERE) {
        double den = d[0] * xp[0] + d[1] * xp[1] + d[2] * xp[2];
        for (int m = 0; m < 3; ++m) {
#pragma omp atomic
            g_sites[3 * i + m] += sgn_gdt * xp[m] / den;
        }
#pragma omp atomic
        g_r[i] += sgn_gdt * (double)S->radii[i] / den;
        return;
    }
    const float *pj = S->sites + 3 * j;
    double a = d[0] * ((double)pj[0] - p[0]) + d[1] * ((double)pj[1] - p[1]) +
               d[2] * ((double)pj[2] - p[2]);
    for (int m = 0; m < 3; ++m) {
#pragma omp atomic
        g_sites[3 * i + m] += sgn_gdt * xp[m] / a;
#pragma omp atomic
        g_sites[3 * j + m] += sgn_gdt * ((double)pj[m] - x[m]) / a;
    }
#pragma omp atomic
    g_w[i] += sgn_gdt * 0.5 / a;
#pragma omp atomic
    g_w[j] -= sgn_gdt * 0.5 / a;
}

/* Reverse-mode derivative of one detail segment (NEXT-2), step by step back
 * through detail_radiance and detail_geometry.  g_ts = dL/dt* from the
 * interval ends the displaced face binds; gC = dL/dc(x) = T_k alpha_k G. */
static void detail_backward(const oc_scene *S, int64_t i, const double Q[3], const double d[3],
                            const oc_seg *s, double g_ts, const double gC[3], double *g_sites,
                            double *g_r, double *g_normals, double *g_uv, double *g_disp,
                            double *g_sv)
{
    const oc_detail *X = S->det;
    const int K = X->K;
    const float *uv = X->uv + (size_t)2 * K * i;
    const double tau = (double)X->tau;
    oc_dstate D;
    detail_geometry(S, i, Q, d, &D);
    detail_radiance(S, i, d, s->t_in, &D);
    const oc_frame *F = &D.F;
    double gm[3] = {0, 0, 0}, gc[3] = {0, 0, 0}, gu[3] = {0, 0, 0}, gv[3] = {0, 0, 0};
    /* Eq. svrad: col = sum_k ws_k c_k,  c_k = sum_a om_a v_{k,a} */
    double gws[OC_MAX_DETAIL], sw = 0.0;
    for (int k = 0; k < K; ++k) {
        double *gvk = g_sv + ((size_t)K * i + k) * OC_SV_AXES * 3;
        for (int a = 0; a < OC_SV_AXES; ++a)
            for (int c = 0; c < 3; ++c) {
#pragma omp atomic
                gvk[3 * a + c] += D.ws[k] * D.om[a] * gC[c];
            }
        gws[k] = dot3(D.ck[k], gC);
        sw += D.ws[k] * gws[k];
    }
    /* softmax of z_k = -tau rho_k, rho_k = |qs - s_k| */
    double gqs[2] = {0, 0};
    for (int k = 0; k < K; ++k) {
        const double grho = -tau * D.ws[k] * (gws[k] - sw);
        if (D.rhos[k] > 0.0) {
            const double ex = (D.qs[0] - uv[2 * k]) / D.rhos[k], ey = (D.qs[1] - uv[2 * k + 1]) / D.rhos[k];
            gqs[0] += grho * ex;
            gqs[1] += grho * ey;
#pragma omp atomic
            g_uv[(size_t)2 * K * i + 2 * k] -= grho * ex;
#pragma omp atomic
            g_uv[(size_t)2 * K * i + 2 * k + 1] -= grho * ey;
        }
    }
    if (!D.parallel) {
        /* qs = (ys.u, ys.v) */
        double gys[3];
        for (int c = 0; c < 3; ++c) {
            gys[c] = gqs[0] * F->u[c] + gqs[1] * F->v[c];
            gu[c] += gqs[0] * D.ys[c];
            gv[c] += gqs[1] * D.ys[c];
        }
        /* ys = ts d - c */
        g_ts += dot3(gys, d);
        for (int c = 0; c < 3; ++c) gc[c] -= gys[c];
        /* ts = (c.m + delta) / (d.m) */
        const double f = g_ts / D.A;
        for (int c = 0; c < 3; ++c) {
            gc[c] += f * F->m[c];
            gm[c] -= f * D.ys[c];
        }
        double gdr = 0.0;
        if (D.clamp) {
#pragma omp atomic
            g_r[i] += f * (double)D.clamp;
        } else {
            gdr = f;
        }
        /* Eq. svdisp: dr = sum_k w_k d_k, w = softmax(-tau rho), rho_k = |qb - s_k| */
        double gqb[2] = {0, 0};
        for (int k = 0; k < K; ++k) {
            const double dk = (double)X->disp[(size_t)K * i + k];
#pragma omp atomic
            g_disp[(size_t)K * i + k] += D.w[k] * gdr;
            const double grho = -tau * D.w[k] * gdr * (dk - D.dr);
            if (D.rho[k] > 0.0) {
                const double ex = (D.qb[0] - uv[2 * k]) / D.rho[k], ey = (D.qb[1] - uv[2 * k + 1]) / D.rho[k];
                gqb[0] += grho * ex;
                gqb[1] += grho * ey;
#pragma omp atomic
                g_uv[(size_t)2 * K * i + 2 * k] -= grho * ex;
#pragma omp atomic
                g_uv[(size_t)2 * K * i + 2 * k + 1] -= grho * ey;
            }
        }
        /* qb = (y.u, y.v), y = tb d - c, tb = c.m / (d.m) */
        double gy[3];
        for (int c = 0; c < 3; ++c) {
            gy[c] = gqb[0] * F->u[c] + gqb[1] * F->v[c];
            gu[c] += gqb[0] * D.y[c];
            gv[c] += gqb[1] * D.y[c];
        }
        const double f2 = dot3(gy, d) / D.A;
        for (int c = 0; c < 3; ++c) {
            gc[c] += f2 * F->m[c] - gy[c];
            gm[c] -= f2 * D.y[c];
        }
    }
    /* frame: v = m x u, u = w/|w|, w = e_k x m, m = n/|n| */
    double t3[3], e[3] = {0, 0, 0}, gw[3];
    cross3(F->u, gv, t3);
    for (int c = 0; c < 3; ++c) gm[c] += t3[c];
    cross3(gv, F->m, t3);
    for (int c = 0; c < 3; ++c) gu[c] += t3[c];
    const double ug = dot3(F->u, gu);
    for (int c = 0; c < 3; ++c) gw[c] = (gu[c] - F->u[c] * ug) / F->wl;
    e[F->kax] = 1.0;
    cross3(gw, e, t3);
    for (int c = 0; c < 3; ++c) gm[c] += t3[c];
    const double mg = dot3(F->m, gm);
    for (int c = 0; c < 3; ++c) {
#pragma omp atomic
        g_sites[3 * i + c] += gc[c];
#pragma omp atomic
        g_normals[3 * i + c] += (gm[c] - F->m[c] * mg) / F->nn;
    }
}

/*
 * Gradients of L = sum_pixels <grad_out[pixel], out[pixel]> for npix pixels
 * (same pixel convention as oracle_render; grad_out float[npix*4]).
 * Accumulates (+=) into double arrays g_sites[N*3], g_w[N], g_r[N], g_sigma[N],
 * g_rgb[N*3].  Compositing derivative: with
 * S_k = sum_{m>k} T_m a_m c_m + T_{K+1} bg,
 *   dL/dc_k = T_k a_k G,  dL/dtau_k = G.(T_{k+1} c_k - S_k) - G_T T_{K+1},
 *   dL/dsigma_k = dL/dtau_k dt_k,  dL/ddt_k = dL/dtau_k sigma_k.
 */
int oracle_backward(int mode, int64_t N, const float *sites, const float *weights,
                    const float *radii, const float *density, const float *rgb,
                    const int64_t *nbr_off, const int32_t *nbr_idx, const float *bg,
                    const float *normals, const oc_detail *det, const oc_camera *cam, int64_t npix,
                    const int32_t *pix_xy, const float *grad_out, double *g_sites, double *g_w,
                    double *g_r, double *g_sigma, double *g_rgb, double *g_normals,
                    double *g_uv, double *g_disp, double *g_sv, int nthreads)
{
    oc_scene S;
    make_scene(&S, N, sites, weights, radii, density, rgb, nbr_off, nbr_idx, bg, normals, det);
    oc_bins B;
    memset(&B, 0, sizeof(B));
    if (mode == O3_TILE_LISTS) build_bins(&S, cam, &B);
    if (!pix_xy) npix = (int64_t)cam->width * cam->height;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel
    {
        oc_scratch scr = {NULL, 0};
        double *Tk = NULL, *Ak = NULL;
        int64_t capk = 0;
#pragma omp for schedule(dynamic, 16)
        for (int64_t q = 0; q < npix; ++q) {
            int x = pix_xy ? pix_xy[2 * q] : (int)(q % cam->width);
            int y = pix_xy ? pix_xy[2 * q + 1] : (int)(q / cam->width);
            double Q[3], d[3], tn;
            const int pv = pixel_ray(cam, x + 0.5, y + 0.5, Q, d, &tn);
            int64_t n = pv ? collect_segments(&S, mode, &B, x, y, Q, d, tn, &scr, NULL, NULL) : 0;
            double out[4];
            int64_t K = composite(&S, scr.segs, n, out);
            if (K + 1 > capk) {
                free(Tk);
                free(Ak);
                capk = K + 1;
                Tk = (double *)malloc(sizeof(double) * (size_t)capk);
                Ak = (double *)malloc(sizeof(double) * (size_t)capk);
            }
            /* T_k (transmittance before segment k) and alpha_k */
            double T = 1.0;
            for (int64_t k = 0; k < K; ++k) {
                const oc_seg *s = scr.segs + k;
                double tau = (double)S.density[s->cell] * (s->t_out - s->t_in);
                Tk[k] = T;
                Ak[k] = 1.0 - exp(-tau);
                T *= exp(-tau);
            }
            double Tend = T; /* T_{K+1} */
            const float *g = grad_out + 4 * q;
            double G[3] = {g[0], g[1], g[2]}, GT = g[3];
            for (int64_t k = 0; k < K; ++k) {
                const oc_seg *s = scr.segs + k;
                int64_t i = s->cell;
                double dt = s->t_out - s->t_in;
                double sig = (double)S.density[i];
                double Tnext = Tk[k] * exp(-sig * dt);
                /* S_k = sum_{m>k} T_m a_m c_m + T_{K+1} bg */
                double Sk[3];
                for (int c = 0; c < 3; ++c) Sk[c] = Tend * S.bg[c];
                for (int64_t m = k + 1; m < K; ++m)
                    for (int c = 0; c < 3; ++c)
                        Sk[c] += Tk[m] * Ak[m] * scr.segs[m].col[c];
                double dtau = -GT * Tend;
                for (int c = 0; c < 3; ++c) {
                    dtau += G[c] * (Tnext * s->col[c] - Sk[c]);
                    if (!S.det) {
#pragma omp atomic
                        g_rgb[3 * i + c] += Tk[k] * Ak[k] * G[c];
                    }
                }
#pragma omp atomic
                g_sigma[i] += dtau * dt;
                double gdt = dtau * sig;
                if (S.det) {
                    /* the displaced face's end goes through the detail chain */
                    double g_ts = 0.0, gC[3];
                    if (s->kout == END_DIPOLE) g_ts += gdt;
                    if (s->kin == END_DIPOLE) g_ts -= gdt;
                    if (s->kout != END_DIPOLE)
                        end_grad(&S, s->kout, i, s->jout, s->t_out, Q, d, gdt, g_sites, g_w, g_r,
                                 g_normals);
                    if (s->kin != END_DIPOLE)
                        end_grad(&S, s->kin, i, s->jin, s->t_in, Q, d, -gdt, g_sites, g_w, g_r,
                                 g_normals);
                    for (int c = 0; c < 3; ++c) gC[c] = Tk[k] * Ak[k] * G[c];
                    detail_backward(&S, i, Q, d, s, g_ts, gC, g_sites, g_r, g_normals, g_uv,
                                    g_disp, g_sv);
                } else if (gdt != 0.0) {
                    end_grad(&S, s->kout, i, s->jout, s->t_out, Q, d, gdt, g_sites, g_w, g_r,
                             g_normals);
                    end_grad(&S, s->kin, i, s->jin, s->t_in, Q, d, -gdt, g_sites, g_w, g_r,
                             g_normals);
                }
            }
        }
        free(scr.segs);
        free(Tk);
        free(Ak);
    }
    if (B.vals) free_bins(&B);
    return 0;
}

/* ======================================================================== */
/* debug entry points for the pins                                          */
/* ======================================================================== */

/* Interval of cell i along an arbitrary ray (Q, d unit, t_near).  mode O1 or O2.
 * res[0..1] = t_in, t_out (absolute); kinds[0..3] = kin, kout, jin, jout.
 * Returns 1 on a sphere hit, 0 otherwise. */
int oracle_cell_interval(int mode, int64_t N, const float *sites, const float *weights,
                         const float *radii, const int64_t *nbr_off, const int32_t *nbr_idx,
                         const float *normals, const oc_detail *det, int64_t i,
                         const double *Q, const double *d,
                         double t_near, double *res, int32_t *kinds)
{
    oc_scene S;
    make_scene(&S, N, sites, weights, radii, NULL, NULL, nbr_off, nbr_idx, NULL, normals, det);
    oc_seg s;
    int64_t np = 0;
    int hit = cell_interval(&S, mode, i, Q, d, t_near, &s, &np);
    if (!hit) return 0;
    res[0] = s.t_in;
    res[1] = s.t_out;
    kinds[0] = s.kin;
    kinds[1] = s.kout;
    kinds[2] = s.jin;
    kinds[3] = s.jout;
    return 1;
}

/* The composited segments of one pixel (mode O1/O2/O3), in compositing order:
 * seg[8k..8k+7] = (cell, t_in, t_out, kin, kout, jin, jout, list_pos).
 * Returns the number of segments written (<= cap). */
int64_t oracle_pixel_segments(int mode, int64_t N, const float *sites, const float *weights,
                              const float *radii, const float *density, const float *rgb,
                              const int64_t *nbr_off, const int32_t *nbr_idx, const float *bg,
                              const float *normals, const oc_detail *det, const oc_camera *cam, int32_t x, int32_t y,
                              double *seg, int64_t cap)
{
    oc_scene S;
    make_scene(&S, N, sites, weights, radii, density, rgb, nbr_off, nbr_idx, bg, normals, det);
    oc_bins B;
    memset(&B, 0, sizeof(B));
    if (mode == O3_TILE_LISTS) build_bins(&S, cam, &B);
    oc_scratch scr = {NULL, 0};
    double Q[3], d[3], tn, out[4];
    const int pv = pixel_ray(cam, x + 0.5, y + 0.5, Q, d, &tn);
    int64_t n = pv ? collect_segments(&S, mode, &B, x, y, Q, d, tn, &scr, NULL, NULL) : 0;
    int64_t K = composite(&S, scr.segs, n, out);
    int64_t m = K < cap ? K : cap;
    for (int64_t k = 0; k < m; ++k) {
        const oc_seg *g = scr.segs + k;
        double *o = seg + 8 * k;
        o[0] = g->cell; o[1] = g->t_in; o[2] = g->t_out; o[3] = g->kin;
        o[4] = g->kout; o[5] = g->jin; o[6] = g->jout; o[7] = g->list_pos;
    }
    free(scr.segs);
    if (B.vals) free_bins(&B);
    return m;
}

/* The ray of pixel (x, y): Q[3], d[3], t_near. */
int oracle_pixel_ray(const oc_camera *cam, int32_t x, int32_t y, double *Q, double *d,
                     double *t_near)
{
    pixel_ray(cam, x + 0.5, y + 0.5, Q, d, t_near);
    return 0;
}

/* Front-to-back compositing of explicit segments (sigma[k], dt[k], rgb[3k]):
 * out[4] = (C + T bg, T); returns the termination index. */
int64_t oracle_composite(int64_t n, const double *sigma, const double *dt, const double *rgb,
                         const double *bg, double *out)
{
    double T = 1.0, C[3] = {0, 0, 0};
    int64_t k = 0;
    for (; k < n;) {
        double tau = sigma[k] * dt[k];
        double alpha = 1.0 - exp(-tau);
        for (int c = 0; c < 3; ++c) C[c] += T * alpha * rgb[3 * k + c];
        T *= exp(-tau);
        ++k;
        if (T < T_STOP) break;
    }
    for (int c = 0; c < 3; ++c) out[c] = C[c] + T * bg[c];
    out[3] = T;
    return k;
}

int oracle_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ======================================================================== */
/* NEXT-4: the adjacency-walk ray tracer (§3.1, §3.2,        */
/* P:687-689 App. C)                                                        */
/* ======================================================================== */
/*
 * The paper traces by walking from cell to cell: "the adjacency information
 * ... allows a ray to walk from one cell to the next by checking all faces"
 * (P:157), with the Delaunay graph "replaced with the dual graph of the power
 * diagram, in addition to considering the sphere bounds in the computation of
 * intersection lengths".  Reading R7: the paper walks
 * the UNBOUNDED diagram's dual (the regular triangulation), which is out
 * of scope; a bounded cell's interval, however, only ends on a radical plane of
 * a Čech neighbour (the face's owner is the next cell) or on its own
 * bounding sphere.  With the paper's weights w = r^2 no other ball
 * contains a sphere-exit point (there pow_c = 0 <= pow_k), so the ray is in a
 * gap of the union of balls and the walk resumes at the next point of the union
 * (a "gap jump"; here by brute force over every ball).  Step by step:
 *   t <- t_near;  c <- locate(t)
 *   loop:  walk interval [t_in, t_out] of c (sphere, near, c's list planes;
 *          O2 semantics) and the constraint that ends it;
 *          the occupied segment (the dipole / detail clip applied, exactly the
 *          interval the rasterizer composites) -> front-to-back compositing,
 *          stop after the segment that makes T < 1e-4;
 *          exit on the plane of neighbour j: c <- j, t <- t_out;
 *          exit on the sphere: t <- t_out, c <- locate(t, excluding c).
 *   locate(t): among the balls whose chord ends after t, the smallest
 *          max(t_entry, t); ties by the smaller power pow(x, b) at that point
 *          (a point inside several balls belongs to the argmin-power cell), then
 *          by the lower index.
 * A step that makes no progress (a degenerate crossing through an edge or a
 * vertex, measure zero) falls back to locate(t, excluding c); a step budget
 * of 4N + 64 guards termination.
 * Per pixel the stats are (cells visited, locate calls, composited segments).
 */
static int64_t trace_locate(const oc_scene *S, const double Q[3], const double d[3], double t,
                            int64_t excl, double *t_at)
{
    int64_t best = -1;
    double bt = 0.0, bp = 0.0;
    for (int64_t b = 0; b < S->N; ++b) {
        if (b == excl) continue;
        const float *p = S->sites + 3 * b;
        double c[3] = {p[0] - Q[0], p[1] - Q[1], p[2] - Q[2]};
        double tc = d[0] * c[0] + d[1] * c[1] + d[2] * c[2];
        double e[3] = {c[0] - tc * d[0], c[1] - tc * d[1], c[2] - tc * d[2]};
        double r = (double)S->radii[b];
        double h = r * r - (e[0] * e[0] + e[1] * e[1] + e[2] * e[2]);
        if (!(h > 0.0)) continue;
        double sq = sqrt(h);
        if (!(tc + sq > t)) continue;
        double tt = tc - sq > t ? tc - sq : t;
        double x[3] = {Q[0] + tt * d[0], Q[1] + tt * d[1], Q[2] + tt * d[2]};
        double pw = powd(x, p, S->weights[b]);
        if (best < 0 || tt < bt || (tt == bt && pw < bp)) {
            best = b;
            bt = tt;
            bp = pw;
        }
    }
    *t_at = bt;
    return best;
}

static void trace_pixel(const oc_scene *S, const double Q[3], const double d[3], double tn,
                        double out[4], int64_t st[3])
{
    oc_scene W = *S; /* the walk's geometry: the power cell inside the ball, no dipole clip */
    W.normals = NULL;
    W.det = NULL;
    double T = 1.0, C[3] = {0.0, 0.0, 0.0};
    int64_t visited = 0, located = 0, nseg = 0;
    double t = tn, tl;
    int64_t c = trace_locate(S, Q, d, t, -1, &tl);
    ++located;
    const int64_t budget = 4 * S->N + 64;
    for (int64_t step = 0; c >= 0 && step < budget; ++step) {
        oc_seg w, o;
        int64_t np = 0;
        const int hit = cell_interval(&W, O2_LIST_PLANES, c, Q, d, tn, &w, &np);
        if (!hit || !(w.t_out > w.t_in) || !(w.t_out > t)) {
            /* no progress in c (degenerate crossing): locate past it */
            const int64_t prev = c;
            c = trace_locate(S, Q, d, t, prev, &tl);
            ++located;
            continue;
        }
        ++visited;
        if (cell_interval(S, O2_LIST_PLANES, c, Q, d, tn, &o, &np) && o.t_out > o.t_in) {
            const double sig = (double)S->density[c];
            const double tau = sig * (o.t_out - o.t_in);
            const double alpha = 1.0 - exp(-tau);
            for (int k = 0; k < 3; ++k) C[k] += T * alpha * o.col[k];
            T *= exp(-tau);
            ++nseg;
            if (T < T_STOP) break;
        }
        t = w.t_out;
        if (w.kout == END_PLANE) {
            c = w.jout;
        } else {
            const int64_t prev = c;
            c = trace_locate(S, Q, d, t, prev, &tl);
            ++located;
        }
    }
    for (int k = 0; k < 3; ++k) out[k] = C[k] + T * S->bg[k];
    out[3] = T;
    st[0] = visited;
    st[1] = located;
    st[2] = nseg;
}

/* Trace npix pixels (pix_xy = int32 (x,y) pairs; NULL = the full image).
 * out double[npix*4] = (C + T bg, T); stats int64[npix*3] (may be NULL). */
int oracle_trace(int64_t N, const float *sites, const float *weights, const float *radii,
                 const float *density, const float *rgb, const int64_t *nbr_off,
                 const int32_t *nbr_idx, const float *bg, const float *normals,
                 const oc_detail *det, const oc_camera *cam, int64_t npix, const int32_t *pix_xy,
                 double *out, int64_t *stats, int nthreads)
{
    oc_scene S;
    make_scene(&S, N, sites, weights, radii, density, rgb, nbr_off, nbr_idx, bg, normals, det);
    if (!pix_xy) npix = (int64_t)cam->width * cam->height;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t q = 0; q < npix; ++q) {
        int x = pix_xy ? pix_xy[2 * q] : (int)(q % cam->width);
        int y = pix_xy ? pix_xy[2 * q + 1] : (int)(q / cam->width);
        double Q[3], d[3], tn;
        int64_t st[3] = {0, 0, 0};
        if (pixel_ray(cam, x + 0.5, y + 0.5, Q, d, &tn)) {
            trace_pixel(&S, Q, d, tn, out + 4 * q, st);
        } else {
            for (int k = 0; k < 3; ++k) out[4 * q + k] = S.bg[k];
            out[4 * q + 3] = 1.0;
        }
        if (stats)
            for (int k = 0; k < 3; ++k) stats[3 * q + k] = st[k];
    }
    return 0;
}

/* The walk of one ray (Q, d, t_near): the visited cells in order (up to cap),
 * returns their number (the sequence test against the argmin-power sampler). */
int64_t oracle_trace_cells(int64_t N, const float *sites, const float *weights,
                           const float *radii, const int64_t *nbr_off, const int32_t *nbr_idx,
                           const double *Q, const double *d, double tn, int32_t *cells,
                           int64_t cap)
{
    oc_scene S;
    make_scene(&S, N, sites, weights, radii, NULL, NULL, nbr_off, nbr_idx, NULL, NULL, NULL);
    int64_t n = 0;
    double t = tn, tl;
    int64_t c = trace_locate(&S, Q, d, t, -1, &tl);
    const int64_t budget = 4 * N + 64;
    for (int64_t step = 0; c >= 0 && step < budget; ++step) {
        oc_seg w;
        int64_t np = 0;
        if (!cell_interval(&S, O2_LIST_PLANES, c, Q, d, tn, &w, &np) || !(w.t_out > w.t_in) ||
            !(w.t_out > t)) {
            c = trace_locate(&S, Q, d, t, c, &tl);
            continue;
        }
        if (n < cap) cells[n] = (int32_t)c;
        ++n;
        t = w.t_out;
        c = (w.kout == END_PLANE) ? w.jout : trace_locate(&S, Q, d, t, c, &tl);
    }
    return n;
}

/* ======================================================================== */
/* NEXT-3: the Čech graph ("the graph of all overlapping spheres")    */
/* ======================================================================== */

/* Edge (i, j), i != j, iff |p_i - p_j| < r_i + r_j (strict),
 * evaluated in double in this fixed order (the inputs are fp32, so every
 * difference is exact):  d2 = (dx*dx + dy*dy) + dz*dz,  s = r_i + r_j,  d2 < s*s. */
static int cech_edge(const float *sites, const float *radii, int64_t i, int64_t j)
{
    double dx = (double)sites[3 * i] - (double)sites[3 * j];
    double dy = (double)sites[3 * i + 1] - (double)sites[3 * j + 1];
    double dz = (double)sites[3 * i + 2] - (double)sites[3 * j + 2];
    double d2 = (dx * dx + dy * dy) + dz * dz;
    double s = (double)radii[i] + (double)radii[j];
    return d2 < s * s;
}

/* Brute-force rows of the Čech graph: for each requested row i (rows[k]), every
 * j in [0, N) in ascending order.  counts[k] = degree; if indices != NULL the
 * neighbours of row k are written at indices[offs[k] ...] (offs = exclusive scan
 * of counts, computed by the caller).  O(nrows * N). */
int oracle_cech_rows(int64_t N, const float *sites, const float *radii, int64_t nrows,
                     const int64_t *rows, int64_t *counts, const int64_t *offs, int32_t *indices,
                     int nthreads)
{
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t k = 0; k < nrows; ++k) {
        int64_t i = rows[k], c = 0;
        for (int64_t j = 0; j < N; ++j) {
            if (j == i || !cech_edge(sites, radii, i, j)) continue;
            if (indices) indices[offs[k] + c] = (int32_t)j;
            ++c;
        }
        counts[k] = c;
    }
    return 0;
}

/* L_connect:  L(P_i) = sum_{j in Cech(i)} max(r_i + r_j - d_ij, 0)^2 for
 * every cell (so the total counts each overlapping pair from both ends), and its
 * gradient: with o = max(r_i + r_j - d_ij, 0), u = (p_i - p_j)/d_ij,
 *   dL(P_i)/dr_i = dL(P_i)/dr_j = 2o,  dL(P_i)/dp_i = -2o u,  dL(P_i)/dp_j = +2o u.
 * g_sites / g_radii accumulate d(sum_i L(P_i)); loss[i] = L(P_i). */
int oracle_connect_loss(int64_t N, const float *sites, const float *radii,
                        const int64_t *nbr_off, const int32_t *nbr_idx, double *loss,
                        double *g_sites, double *g_radii)
{
    for (int64_t i = 0; i < N; ++i) {
        double Li = 0.0;
        for (int64_t q = nbr_off[i]; q < nbr_off[i + 1]; ++q) {
            int64_t j = nbr_idx[q];
            double dv[3], d2 = 0.0;
            for (int m = 0; m < 3; ++m) {
                dv[m] = (double)sites[3 * i + m] - (double)sites[3 * j + m];
                d2 += dv[m] * dv[m];
            }
            double d = sqrt(d2);
            double o = (double)radii[i] + (double)radii[j] - d;
            if (o <= 0.0) continue;
            Li += o * o;
            g_radii[i] += 2.0 * o;
            g_radii[j] += 2.0 * o;
            if (d > 0.0)
                for (int m = 0; m < 3; ++m) {
                    g_sites[3 * i + m] -= 2.0 * o * dv[m] / d;
                    g_sites[3 * j + m] += 2.0 * o * dv[m] / d;
                }
        }
        loss[i] = Li;
    }
    return 0;
}

/* ======================================================================== */
/* detail-site probes (NEXT-2 pins)                                         */
/* ======================================================================== */

/* tangent frame of one normal: out[9] = (u, v, m) */
int oracle_tangent_frame(const float *n, double *out)
{
    oc_frame F;
    tangent_frame(n, &F);
    for (int c = 0; c < 3; ++c) {
        out[c] = F.u[c];
        out[3 + c] = F.v[c];
        out[6 + c] = F.m[c];
    }
    return F.kax;
}

/* soft-Voronoi weights of q against K sites (Eqs. svdisp/svrad) */
int oracle_soft_voronoi(const double *q, const float *uv, int32_t K, double tau, double *w)
{
    double rho[OC_MAX_DETAIL];
    if (K < 1 || K > OC_MAX_DETAIL) return -1;
    soft_voronoi(q, uv, K, tau, rho, w);
    return 0;
}

/* Detail evaluation of cell i along (Q, d) with the interval entry t_entry
 * (used by the parallel case): out = (parallel, tb, dr, delta, ts, col[3],
 * qb[2], qs[2]) -- 12 doubles. */
int oracle_detail_probe(int64_t N, const float *sites, const float *radii, const float *normals,
                        const oc_detail *det, int64_t i, const double *Q, const double *d,
                        double t_entry, double *out)
{
    oc_scene S;
    make_scene(&S, N, sites, NULL, radii, NULL, NULL, NULL, NULL, NULL, normals, det);
    if (!S.det) return -1;
    oc_dstate D;
    detail_geometry(&S, i, Q, d, &D);
    detail_radiance(&S, i, d, t_entry, &D);
    out[0] = D.parallel;
    out[1] = D.parallel ? 0.0 : D.tb;
    out[2] = D.parallel ? 0.0 : D.dr;
    out[3] = D.delta;
    out[4] = D.parallel ? 0.0 : D.ts;
    for (int c = 0; c < 3; ++c) out[5 + c] = D.col[c];
    out[8] = D.parallel ? 0.0 : D.qb[0];
    out[9] = D.parallel ? 0.0 : D.qb[1];
    out[10] = D.qs[0];
    out[11] = D.qs[1];
    return 0;
}
