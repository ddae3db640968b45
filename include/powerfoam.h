/*
 * powerfoam.h -- C ABI of the B200-native Power Foam rasterizer
 * (arXiv 2604.24994: tile-based differentiable rasterization of bounded
 * power-diagram cells, forward and backward).
 *
 * Citations: P:<line> = PAPER.md, S:<line> = SPEC.md, SURVEY §x = SURVEY.md,
 * DESIGN §x = DESIGN.md (the readings of the paper that fix what is left open).
 *
 * Conventions common to every entry point
 * ---------------------------------------
 *  - Every function returns an int status (PF_OK = 0) and never throws.
 *    On a non-zero status pf_last_error() returns a thread-local message.
 *  - Array arguments are DEVICE pointers owned by the caller (in practice
 *    PyTorch tensors); the library stores scene pointers without copying them
 *    and re-reads them at every forward (so in-place optimizer updates between
 *    steps are seen).  Parameters must not change between a forward and its
 *    matching backward.
 *  - Camera arrays (pf_camera) are HOST memory.
 *  - `stream` is a cudaStream_t (declared here as an opaque pointer so this
 *    header does not need the CUDA headers); every call enqueues its work on it
 *    and returns.  The one exception: pf_render_forward reads the pair counts
 *    of all its views back to the host once per call (one stream sync), to size
 *    the per-tile lists.
 *  - A handle is bound to the device that was current at creation; calls on one
 *    handle are not thread-safe; separate handles are independent.
 *  - Pixel (x, y) has its centre at (x + 0.5, y + 0.5); tiles are 16x16 pixels;
 *    images are row-major.
 */
#ifndef POWERFOAM_H
#define POWERFOAM_H

#include <stdint.h>

#if defined(__GNUC__)
#define PF_API __attribute__((visibility("default")))
#else
#define PF_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *pf_stream_t; /* == cudaStream_t */
typedef struct pf_scene pf_scene;        /* opaque; owns workspaces and saved state only */

/* status codes (S:615 exit-code convention: 1 malformed input, 2 render failure) */
enum {
    PF_OK = 0,
    PF_ERR_INVALID_ARGUMENT = 1, /* null pointer, N < 1, W/H < 1 or > 32768, fx/fy <= 0,
                                    non-finite camera, validation failure (PF_VALIDATE) */
    PF_ERR_CUDA = 2,             /* launch / asynchronous CUDA error (message has the text) */
    PF_ERR_OUT_OF_MEMORY = 3,
    PF_ERR_STATE = 4             /* backward without a matching forward (views / sizes differ) */
};

/* scene flags */
enum {
    PF_VALIDATE = 1u << 0,     /* check the scene on the device at creation (finite values,
                                  r > 0, sigma >= 0, neighbour ids in [0,N) and != i) */
    PF_STATIC_SCENE = 1u << 1, /* parameters never change after creation: the edge records
                                  (K0) are built once in pf_create_scene, not per forward */
    PF_INFERENCE = 1u << 2     /* forward only: no per-view state is saved for a backward
                                  (pf_render_backward then returns PF_ERR_STATE) */
};

/*
 * The scene: N bounded power cells and their neighbour lists.
 *   cell i = power site p_i with weight w_i ("squared radius (also known ...
 *   as a weight)"; the paper ties w_i = r_i^2, the ABI takes both),
 *   bounding sphere B_i of radius r_i, density sigma_i >= 0 and constant
 *   linear radiance rgb_i (appearance reading SURVEY C6).
 *   Bounded cell C_i = {x : pow(x,i) <= pow(x,j) for all j} ∩ B_i with
 *   pow(x,i) = |x - p_i|^2 - w_i.
 *   nbr_indices[nbr_offsets[i] .. nbr_offsets[i+1]) must contain every j whose
 *   radical plane can cut B_i: the Čech complex (all overlapping spheres)
 *   suffices when w = r^2; extra neighbours are allowed.
 */
typedef struct {
    int64_t num_cells;          /* N >= 1 */
    int64_t num_edges;          /* E = nbr_offsets[N] (host copy of the last offset) */
    const float *sites;         /* device f32[N,3]  p_i (world units), row-major */
    const float *weights;       /* device f32[N]    w_i */
    const float *radii;         /* device f32[N]    r_i > 0 */
    const float *density;       /* device f32[N]    sigma_i >= 0 (1/world units) */
    const float *rgb;           /* device f32[N,3]  linear radiance */
    const int64_t *nbr_offsets; /* device i64[N+1] CSR offsets, nbr_offsets[0] = 0 */
    const int32_t *nbr_indices; /* device i32[E]   neighbour ids */
    float background[3];        /* constant background radiance */
    uint32_t flags;             /* PF_VALIDATE | PF_STATIC_SCENE | PF_INFERENCE */
    const float *normals;       /* device f32[N,3] or NULL.  Oriented-point dipoles (P:238-249,
                                   NEXT-1): cell i is occupied only on the side its normal points
                                   away from, (x - p_i).n_i <= 0; the other half has
                                   zero density.  Non-zero, finite (not required to be unit). */
    /* Detail sites of the dipole faces (NEXT-2, P:278-297 Eqs. svdisp/svrad);
     * num_detail = 0 disables them.  Requires normals.  Face chart: m = n/|n|, axis k of
     * the smallest |n_k| (ties to the higher index), u = (e_k x m)/|e_k x m|, v = m x u
     * (SPEC S:186-189); chart coordinates q(y) = ((y-p).u, (y-p).v).  Per ray and cell:
     * x_bar = hit of the base face (x-p).m = 0; delta = clamp(sum_k softmax_k(-tau
     * |q(x_bar) - s_k|) d_k, -r, r); occupied half (x-p).m <= delta; x = hit of that
     * face; radiance c(x) = sum_k softmax_k(-tau |q(x) - s_k|) sum_a softmax_a(gamma
     * d.a_a) v_{k,a} replaces rgb_i (readings R6). */
    int32_t num_detail;         /* K: 0, or 1..8 detail sites per cell */
    float sv_gamma;             /* SV sharpness gamma (finite) */
    float sv_tau;               /* soft-Voronoi temperature tau > 0 (1/world units) */
    float sv_axes[8][3];        /* the 8 shared SV axes a_a (unit) */
    const float *detail_uv;     /* device f32[N,K,2] s_{i,k} (world units, face chart), 8-byte aligned */
    const float *detail_disp;   /* device f32[N,K]   d_{i,k} along m */
    const float *detail_sv;     /* device f32[N,K,8,3] v_{i,k,a} (linear radiance), 16-byte aligned */
} pf_scene_desc;

/* Camera, OpenCV axes (x right, y down, z forward).
 * model PF_PINHOLE: d_cam = ((x+0.5-cx)/fx, (y+0.5-cy)/fy, 1), d = normalize(R d_cam),
 *   origin Q; the ray is clipped to camera-space z >= near_plane, i.e.
 *   t >= near_plane * |d_cam|.
 * model PF_FISHEYE (equidistant, NEXT-4): (a, b) = ((x+0.5-cx)/fx,
 *   (y+0.5-cy)/fy), theta = |(a,b)|, d_cam = (sin(theta) a/theta, sin(theta) b/theta,
 *   cos(theta)); pixels with theta > pi lie outside the image circle (output
 *   (background, T = 1)); rays are clipped to t >= near_plane (distance). */
enum { PF_PINHOLE = 0, PF_FISHEYE = 1 };
typedef struct {
    int32_t width, height; /* pixels, 1..32768 */
    float fx, fy, cx, cy;  /* pixel units, fx, fy > 0 */
    float c2w[12];         /* row-major 3x4 [R | Q], world-from-camera */
    float near_plane;      /* > 0 */
    int32_t model;         /* PF_PINHOLE or PF_FISHEYE */
} pf_camera;

/* Creates a handle for the scene described by *desc (pointers are stored, not
 * copied).  With PF_VALIDATE the scene is checked on the device (one sync). */
PF_API int pf_create_scene(const pf_scene_desc *desc, pf_scene **out, pf_stream_t stream);

/*
 * Forward render of num_views >= 1 views (all of the same width x height).
 * out: device f32[V,H,W,4], out[v,y,x] = (R, G, B, T_final).
 * Per view: project every bounding sphere and bin it to 16x16 tiles,
 * key = pow(Q, p_i) (Theorem 2), radix-sort (tile, key) pairs
 * ("global sort by depths ... similar to 3DGS"), then per pixel walk the
 * tile list: interval of the ray in each bounded cell from the sphere and the
 * radical planes of its neighbours (P:228, P:577-585 with the weight sign of
 * SURVEY C1), composite front to back with alpha = 1 - exp(-sigma dt)
 * (SURVEY C4), stop after the segment that makes T < 1e-4 (C7),
 * out = (C + T bg, T).  Forward results are bit-deterministic.
 * Saves per-view state (sorted lists, final colours) for pf_render_backward.
 */
PF_API int pf_render_forward(pf_scene *s, const pf_camera *cams, int32_t num_views, float *out,
                      pf_stream_t stream);

/* Optional per-cell by-products of a forward (NEXT-1), accumulated (+=) over the
 * pixels of all views of the call; device f32[N] arrays, or NULL:
 *   contrib[i]     += sum over composited segments of cell i of T_k alpha_k
 *                     (the pruning statistic, and L_sparse)
 *   normal_term[i] += sum of T_k alpha_k max(n_i . d, 0)^2  (L_normal, P:718;
 *                     only with dipole normals). */
typedef struct {
    float *contrib;
    float *normal_term;
} pf_forward_extras;

/* pf_render_forward plus the by-products above (ex may be NULL). */
PF_API int pf_render_forward_ex(pf_scene *s, const pf_camera *cams, int32_t num_views, float *out,
                                const pf_forward_extras *ex, pf_stream_t stream);

/*
 * Backward of the immediately preceding pf_render_forward with the same cameras
 * (else PF_ERR_STATE).  grad_out: device f32[V,H,W,4] = dL/d(out) (channel 3 =
 * dL/dT_final).  ACCUMULATES (+=) dL/d(param) into the five caller arrays
 * (device f32 [N,3], [N], [N], [N], [N,3]); the caller zeroes them.  Exact
 * derivative of the forward for its active constraints and termination index
 * (SURVEY App. A).  Float atomics: deterministic up to summation order.
 */
PF_API int pf_render_backward(pf_scene *s, const pf_camera *cams, int32_t num_views,
                       const float *grad_out, float *grad_sites, float *grad_weights,
                       float *grad_radii, float *grad_density, float *grad_rgb,
                       pf_stream_t stream);

/* Gradient outputs of pf_render_backward_ex (device arrays, accumulated +=). */
typedef struct {
    float *sites;    /* [N,3] */
    float *weights;  /* [N]   */
    float *radii;    /* [N]   */
    float *density;  /* [N]   */
    float *rgb;      /* [N,3] */
    float *normals;  /* [N,3] dL/dn_i of the dipole normals, or NULL (ignored without dipoles) */
    float *detail_uv;   /* [N,K,2] or NULL (detail scenes; rgb receives no gradient there) */
    float *detail_disp; /* [N,K]   or NULL */
    float *detail_sv;   /* [N,K,8,3] or NULL; 8-byte aligned */
} pf_grads;

/* pf_render_backward with the gradient arrays in a struct (adds dL/d normals).
 * Detail scenes (num_detail > 0): the backward runs as a replay of the forward's
 * records (K7) that emits one work item per detail segment, then the detail chain
 * of P:284-293 over the items (K7D); the item arena is sized from the segment count
 * the forward recorded, read with ONE stream synchronisation at the start of the
 * call.  Limits there: width * height < 2^25 and num_views <= 128
 * (PF_ERR_INVALID_ARGUMENT otherwise).  With PF_VALIDATE the call synchronises once
 * more at its end and checks that every item fitted its arena (PF_ERR_STATE). */
PF_API int pf_render_backward_ex(pf_scene *s, const pf_camera *cams, int32_t num_views,
                                 const float *grad_out, const pf_grads *grads, pf_stream_t stream);

/*
 * NEXT-4: the adjacency-walk ray tracer ("walk from one cell to the
 * next by checking all faces", "the cell-to-cell traversal strategy ...
 * still applies ... in addition to considering the sphere bounds", P:687-689;
 * reading R7 of DESIGN.md).  Renders num_views >= 1 views (same width x height)
 * into out (device f32[V,H,W,4], the layout of pf_render_forward) by walking
 * every pixel ray from cell to cell: inside the union of balls the exit plane
 * names the next cell (the Čech list), at a sphere exit the walk jumps the gap
 * to the next ball on a BVH of the balls (built per call; once with
 * PF_STATIC_SCENE).  The image equals pf_render_forward's up to fp32 rounding
 * (the paper's "same" renderers, Fig. 1) for scenes with w = r^2 (P:184-189:
 * the weight IS the squared radius); no backward state is saved.
 * stats: host int64[5] or NULL (then no sync): rays traced, cells visited,
 * locate (BVH) calls, composited segments, walks stopped by the step budget.
 * Errors: PF_ERR_INVALID_ARGUMENT (NULL / bad camera), PF_ERR_CUDA,
 * PF_ERR_OUT_OF_MEMORY.
 */
PF_API int pf_trace_forward(pf_scene *s, const pf_camera *cams, int32_t num_views, float *out,
                            int64_t *stats, pf_stream_t stream);

/* Frees everything the handle owns (not the caller's arrays).  NULL is a no-op. */
PF_API int pf_destroy(pf_scene *s);

/* Thread-local message for the last non-zero status of this thread. */
PF_API const char *pf_last_error(void);

/* ---------------------------------------------------------------------------
 * Debug / measurement exports (used by the parity tests and bench.py).
 * ------------------------------------------------------------------------- */

/*
 * Binning outputs of one camera, device outputs:
 *   rect i32[N,4] (tx0, ty0, tx1, ty1 half-open), count i32[N], keybits u32[N],
 *   keys u64[P], vals u32[P] (sorted), ranges u32[T,2] ([start,end), (0,0) empty).
 * *num_pairs (host) receives P.  If keys == NULL only rect/count/keybits and P
 * are produced (so the caller can size keys/vals).  Synchronizes the stream.
 * The debug exports reuse the forward's sorted-pair workspace: a following
 * pf_render_backward returns PF_ERR_STATE until the next pf_render_forward.
 */
PF_API int pf_debug_binning(pf_scene *s, const pf_camera *cam, int32_t *rect, int32_t *count,
                     uint32_t *keybits, uint64_t *keys, uint32_t *vals, uint32_t *ranges,
                     int64_t *num_pairs, pf_stream_t stream);

/*
 * Per-pixel work counters of one forward view (counting build of the forward
 * kernel): counters i64[H,W,4] = (X_s list entries examined, X_h sphere hits,
 * X_p plane evaluations, X_c composited segments) -- SURVEY §8(d).
 */
PF_API int pf_debug_counters(pf_scene *s, const pf_camera *cam, int64_t *counters, pf_stream_t stream);

/* Kernel launches issued by this handle since creation (bench "gpu_launches"). */
PF_API int64_t pf_launch_count(const pf_scene *s);

/*
 * Stage timing.  While enabled, CUDA events are recorded (on the call's
 * stream) around each stage's launches of a call; pf_stage_times synchronizes,
 * writes per-stage totals in milliseconds and the number of kernels launched
 * inside them, and clears them.
 * Stages: 0 edge records (K0), 1 preprocess (K1), 2 scan (K2), 3 emit (K3),
 * 4 sort (K4), 5 ranges (K5), 6 forward blend (K6), 7 backward (K7), 8 unpack (K8).
 */
#define PF_NUM_STAGES 9
PF_API int pf_set_profiling(pf_scene *s, int enable);
PF_API int pf_stage_times(pf_scene *s, double *ms /* [PF_NUM_STAGES] */,
                   int64_t *launches /* [PF_NUM_STAGES] */);

/* Pairs P of each view of the last forward (host int64[num_views]). */
PF_API int pf_last_pair_counts(const pf_scene *s, int64_t *pairs, int32_t num_views);

/* ---------------------------------------------------------------------------
 * NEXT-3: the Čech graph on the GPU (the graph of all overlapping
 * spheres, "significantly cheaper to construct using GPU-accelerated collision
 * detection") and the connectivity loss L_connect.
 * ------------------------------------------------------------------------- */
typedef struct pf_cech pf_cech; /* opaque builder; owns grow-only workspaces */

PF_API int pf_cech_create(pf_cech **out);
PF_API int pf_cech_destroy(pf_cech *h);
PF_API const char *pf_cech_last_error(void);

/*
 * Builds the CSR neighbour lists of the Čech complex of N spheres (device
 * sites f32[N,3], radii f32[N]): j is a neighbour of i iff i != j and
 * |p_i - p_j| < r_i + r_j (strict), evaluated in double as
 * ((dx*dx + dy*dy) + dz*dz) < (r_i + r_j)^2.  Writes nbr_offsets (device i64[N+1])
 * and *num_edges (host); if nbr_indices != NULL and capacity >= E, also the
 * indices (device i32[E]), each row ascending (canonical).  Otherwise call again
 * with an array of at least *num_edges entries.  One stream sync per call.
 * The output feeds pf_scene_desc (with w = r^2 the lists are exact).
 */
PF_API int pf_cech_build(pf_cech *h, int64_t num_cells, const float *sites, const float *radii,
                         int64_t *nbr_offsets, int32_t *nbr_indices, int64_t capacity,
                         int64_t *num_edges, pf_stream_t stream);

/*
 * L_connect over given lists: loss[i] = sum_{j in N(i)} max(r_i + r_j - d_ij, 0)^2
 * (device f32[N], or NULL); gradients of sum_i loss[i] are ACCUMULATED (+=) into
 * grad_sites [N,3] / grad_radii [N] (device, or NULL).  Asynchronous.
 */
PF_API int pf_connect_loss(int64_t num_cells, const float *sites, const float *radii,
                           const int64_t *nbr_offsets, const int32_t *nbr_indices, float *loss,
                           float *grad_sites, float *grad_radii, pf_stream_t stream);

PF_API int64_t pf_cech_launch_count(const pf_cech *h);

#ifdef __cplusplus
}
#endif
#endif /* POWERFOAM_H */
