// pf_cech.cu -- NEXT-3: the Čech graph (all overlapping sphere pairs, P:234
// "significantly cheaper to construct using GPU-accelerated collision
// detection") and L_connect, on the GPU.
//
// Collision detection by a linear BVH: 30-bit Morton codes of the sites,
// sorted with the K4 radix sort; Karras' radix-tree construction (one thread
// per internal node); bottom-up box refit with arrival counters; then one
// thread per sphere traverses the tree with the sphere's box (fp32, directed
// rounding outwards) and applies the exact overlap test at the leaves in fp64
// with a fixed op order (edge iff ((dx^2 + dy^2) + dz^2) < (r_i + r_j)^2, strict:
// SPEC S:73).  Two traversals: counts, then indices; rows are then
// sorted ascending (canonical CSR, bit-comparable with the oracle).
#include <cuda_runtime.h>
#include <math.h>
#include <string.h>

#include <string>

#include "pf_bvh.cuh"
#include "pf_internal.cuh"

namespace pf {

cudaError_t exclusive_scan_counts(pf_scene *s, const int *cnt, int64_t n, uint32_t *offs,
                                  long long *d_total, cudaStream_t st);

namespace {

constexpr int kStack = 64;

// spread the low 21 bits of v to every third bit of a 63-bit word
__device__ __forceinline__ unsigned long long expand_bits21(unsigned long long v)
{
    v &= 0x1fffffull;
    v = (v | (v << 32)) & 0x001f00000000ffffull;
    v = (v | (v << 16)) & 0x001f0000ff0000ffull;
    v = (v | (v << 8)) & 0x100f00f00f00f00full;
    v = (v | (v << 4)) & 0x10c30c30c30c30c3ull;
    v = (v | (v << 2)) & 0x1249249249249249ull;
    return v;
}

__global__ void c0_bounds(const float *__restrict__ sites, int64_t N, float *__restrict__ bb)
{
    // bb[0..2] min, bb[3..5] max, as order-preserving ints via atomics on floats' bits
    __shared__ float smin[3][256], smax[3][256];
    float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N;
         i += (int64_t)gridDim.x * blockDim.x)
        for (int m = 0; m < 3; ++m) {
            const float v = sites[3 * i + m];
            lo[m] = fminf(lo[m], v);
            hi[m] = fmaxf(hi[m], v);
        }
    for (int m = 0; m < 3; ++m) {
        smin[m][threadIdx.x] = lo[m];
        smax[m][threadIdx.x] = hi[m];
    }
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if ((int)threadIdx.x < o)
            for (int m = 0; m < 3; ++m) {
                smin[m][threadIdx.x] = fminf(smin[m][threadIdx.x], smin[m][threadIdx.x + o]);
                smax[m][threadIdx.x] = fmaxf(smax[m][threadIdx.x], smax[m][threadIdx.x + o]);
            }
        __syncthreads();
    }
    if (threadIdx.x == 0)
        for (int m = 0; m < 3; ++m) {
            // float min/max via int atomics (sign-aware ordering)
            const float a = smin[m][0], b = smax[m][0];
            int ia = __float_as_int(a), ib = __float_as_int(b);
            if (ia >= 0) atomicMin(reinterpret_cast<int *>(bb) + m, ia);
            else atomicMax(reinterpret_cast<unsigned *>(bb) + m, (unsigned)ia);
            if (ib >= 0) atomicMax(reinterpret_cast<int *>(bb) + 3 + m, ib);
            else atomicMin(reinterpret_cast<unsigned *>(bb) + 3 + m, (unsigned)ib);
        }
}

__global__ void c1_morton(const float *__restrict__ sites, int64_t N, const float *__restrict__ bb,
                          unsigned long long *__restrict__ keys, uint32_t *__restrict__ vals)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    // 63-bit codes (21 bits per axis): scenes with a dense object inside a wide
    // shell (mip360: |p| up to 80, cells of ~0.01 near the centre) would otherwise
    // put thousands of centre cells on one 30-bit code, split by index order only
    unsigned long long q[3];
    for (int m = 0; m < 3; ++m) {
        const double ext = fmax((double)bb[3 + m] - (double)bb[m], 1e-30);
        const double u = fmin(fmax(((double)sites[3 * i + m] - (double)bb[m]) / ext, 0.0), 1.0);
        q[m] = (unsigned long long)fmin(u * 2097152.0, 2097151.0);
    }
    keys[i] = (expand_bits21(q[0]) << 2) | (expand_bits21(q[1]) << 1) | expand_bits21(q[2]);
    vals[i] = (uint32_t)i;
}

// common-prefix length of the unique 96-bit keys (63-bit morton code, then the
// 32-bit sorted position)
__device__ __forceinline__ int delta(const unsigned long long *__restrict__ codes, int64_t n,
                                     int64_t i, int64_t j)
{
    if (j < 0 || j >= n) return -1;
    const unsigned long long a = codes[i], b = codes[j];
    if (a != b) return __clzll(a ^ b);
    return 64 + __clz((uint32_t)i ^ (uint32_t)j);
}

// Karras (2012): internal node i of n-1, children encoded as (idx << 1) | is_leaf
__global__ void c2_radix_tree(const unsigned long long *__restrict__ codes, int64_t n,
                              uint32_t *__restrict__ left, uint32_t *__restrict__ right,
                              uint32_t *__restrict__ parent_int, uint32_t *__restrict__ parent_leaf)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n - 1) return;
    const int d = (delta(codes, n, i, i + 1) - delta(codes, n, i, i - 1)) >= 0 ? 1 : -1;
    const int dmin = delta(codes, n, i, i - d);
    int64_t lmax = 2;
    while (delta(codes, n, i, i + lmax * d) > dmin) lmax <<= 1;
    int64_t l = 0;
    for (int64_t t = lmax >> 1; t >= 1; t >>= 1)
        if (delta(codes, n, i, i + (l + t) * d) > dmin) l += t;
    const int64_t j = i + l * d;
    const int dnode = delta(codes, n, i, j);
    int64_t s = 0;
    for (int64_t t = (l + 1) >> 1;; t = (t + 1) >> 1) {
        if (delta(codes, n, i, i + (s + t) * d) > dnode) s += t;
        if (t == 1) break;
    }
    const int64_t gamma = i + s * d + min(d, 0);
    const int64_t lo = min(i, j), hi = max(i, j);
    const bool lleaf = lo == gamma, rleaf = hi == gamma + 1;
    left[i] = ((uint32_t)gamma << 1) | (lleaf ? 1u : 0u);
    right[i] = ((uint32_t)(gamma + 1) << 1) | (rleaf ? 1u : 0u);
    if (lleaf) parent_leaf[gamma] = (uint32_t)i;
    else parent_int[gamma] = (uint32_t)i;
    if (rleaf) parent_leaf[gamma + 1] = (uint32_t)i;
    else parent_int[gamma + 1] = (uint32_t)i;
}

__device__ __forceinline__ Box sphere_box(const float *__restrict__ sites,
                                          const float *__restrict__ radii, uint32_t i)
{
    Box b;
    const float r = radii[i];
    for (int m = 0; m < 3; ++m) {
        b.lo[m] = __fsub_rd(sites[3 * i + m], r);
        b.hi[m] = __fadd_ru(sites[3 * i + m], r);
    }
    return b;
}

__device__ __forceinline__ Box load_cg(const Box *p)
{
    Box b;
    const float *f = reinterpret_cast<const float *>(p);
    for (int m = 0; m < 3; ++m) {
        b.lo[m] = __ldcg(f + m);
        b.hi[m] = __ldcg(f + 3 + m);
    }
    return b;
}

// bottom-up refit: the second child to arrive at a node merges and climbs
__global__ void c3_refit(const float *__restrict__ sites, const float *__restrict__ radii,
                         const uint32_t *__restrict__ order, int64_t n,
                         const uint32_t *__restrict__ left, const uint32_t *__restrict__ right,
                         const uint32_t *__restrict__ parent_int,
                         const uint32_t *__restrict__ parent_leaf, Box *__restrict__ boxes_int,
                         Box *__restrict__ boxes_leaf, int *__restrict__ arrive)
{
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    boxes_leaf[k] = sphere_box(sites, radii, order[k]);
    if (n == 1) return;
    uint32_t node = parent_leaf[k];
    while (true) {
        __threadfence();
        if (atomicAdd(arrive + node, 1) == 0) return;   // first arrival: the sibling finishes
        __threadfence();
        const uint32_t L = left[node], R = right[node];
        // the sibling's box was written by another thread: read it from L2
        const Box a = load_cg((L & 1u) ? boxes_leaf + (L >> 1) : boxes_int + (L >> 1));
        const Box b = load_cg((R & 1u) ? boxes_leaf + (R >> 1) : boxes_int + (R >> 1));
        Box u;
        for (int m = 0; m < 3; ++m) {
            u.lo[m] = fminf(a.lo[m], b.lo[m]);
            u.hi[m] = fmaxf(a.hi[m], b.hi[m]);
        }
        boxes_int[node] = u;
        if (node == 0) return;
        node = parent_int[node];
    }
}

__device__ __forceinline__ bool overlap(const Box &a, const Box &b)
{
    return a.lo[0] <= b.hi[0] && b.lo[0] <= a.hi[0] && a.lo[1] <= b.hi[1] && b.lo[1] <= a.hi[1] &&
           a.lo[2] <= b.hi[2] && b.lo[2] <= a.hi[2];
}

__device__ __forceinline__ bool cech_edge(const float *__restrict__ sites,
                                          const float *__restrict__ radii, uint32_t i, uint32_t j)
{
    const double dx = __dsub_rn((double)sites[3 * i], (double)sites[3 * j]);
    const double dy = __dsub_rn((double)sites[3 * i + 1], (double)sites[3 * j + 1]);
    const double dz = __dsub_rn((double)sites[3 * i + 2], (double)sites[3 * j + 2]);
    const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
    const double s = __dadd_rn((double)radii[i], (double)radii[j]);
    return d2 < __dmul_rn(s, s);
}

// one thread per sorted leaf k (sphere i = order[k]); kWrite: emit, else count
template <bool kWrite>
__global__ void __launch_bounds__(128)
c4_query(const float *__restrict__ sites, const float *__restrict__ radii,
         const uint32_t *__restrict__ order, int64_t n, const uint32_t *__restrict__ left,
         const uint32_t *__restrict__ right, const Box *__restrict__ boxes_int,
         const Box *__restrict__ boxes_leaf, int *__restrict__ counts,
         const int64_t *__restrict__ offs, int32_t *__restrict__ out, int *__restrict__ overflow)
{
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const uint32_t i = order[k];
    const Box q = boxes_leaf[k];
    int c = 0;
    int64_t o = kWrite ? offs[i] : 0;
    if (n == 1) {
        if (!kWrite) counts[i] = 0;
        return;
    }
    uint32_t stack[kStack];
    int sp = 0;
    stack[sp++] = 0u << 1;   // root: internal node 0
    while (sp > 0) {
        const uint32_t nd = stack[--sp];
        const uint32_t idx = nd >> 1;
        if (nd & 1u) {
            const uint32_t j = order[idx];
            if (j != i && overlap(q, boxes_leaf[idx]) && cech_edge(sites, radii, i, j)) {
                if (kWrite) out[o + c] = (int32_t)j;
                ++c;
            }
            continue;
        }
        if (!overlap(q, boxes_int[idx])) continue;
        if (sp + 2 > kStack) {   // cannot happen for n < 2^30 with a balanced-enough tree
            atomicExch(overflow, 1);
            continue;
        }
        stack[sp++] = right[idx];
        stack[sp++] = left[idx];
    }
    if (!kWrite) counts[i] = c;
}

__global__ void c5_offsets(const uint32_t *__restrict__ offs32, const int *__restrict__ counts,
                           int64_t n, int64_t *__restrict__ offs)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) offs[i] = (int64_t)offs32[i];
    if (i == n - 1) offs[n] = (int64_t)offs32[i] + counts[i];
}

// canonical order: each row ascending (insertion sort; rows are short)
__global__ void c6_sort_rows(const int64_t *__restrict__ offs, int64_t n, int32_t *__restrict__ idx)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t b = offs[i], e = offs[i + 1];
    for (int64_t p = b + 1; p < e; ++p) {
        const int32_t v = idx[p];
        int64_t q = p - 1;
        while (q >= b && idx[q] > v) {
            idx[q + 1] = idx[q];
            --q;
        }
        idx[q + 1] = v;
    }
}

// L_connect: per cell i, sum over its Čech neighbours of
// o^2 with o = max(r_i + r_j - d_ij, 0); gradient of the total: the two ends get
// dr = 2o each, dp_i = -2o u, dp_j = +2o u (u = (p_i - p_j)/d).
__global__ void c7_connect(const float *__restrict__ sites, const float *__restrict__ radii,
                           const int64_t *__restrict__ offs, const int32_t *__restrict__ idx,
                           int64_t n, float *__restrict__ loss, float *__restrict__ gs,
                           float *__restrict__ gr)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float px = sites[3 * i], py = sites[3 * i + 1], pz = sites[3 * i + 2], ri = radii[i];
    float L = 0.0f, gxi = 0.0f, gyi = 0.0f, gzi = 0.0f, gri = 0.0f;
    for (int64_t q = offs[i]; q < offs[i + 1]; ++q) {
        const int j = idx[q];
        const float dx = px - sites[3 * j], dy = py - sites[3 * j + 1], dz = pz - sites[3 * j + 2];
        const float d = sqrtf(dx * dx + dy * dy + dz * dz);
        const float o = ri + radii[j] - d;
        if (!(o > 0.0f)) continue;
        L += o * o;
        if (gr) {
            gri += 2.0f * o;
            atomicAdd(gr + j, 2.0f * o);
        }
        if (gs && d > 0.0f) {
            const float f = 2.0f * o / d;
            gxi -= f * dx;
            gyi -= f * dy;
            gzi -= f * dz;
            atomicAdd(gs + 3 * j, f * dx);
            atomicAdd(gs + 3 * j + 1, f * dy);
            atomicAdd(gs + 3 * j + 2, f * dz);
        }
    }
    if (loss) loss[i] = L;
    if (gr) atomicAdd(gr + i, gri);
    if (gs) {
        atomicAdd(gs + 3 * i, gxi);
        atomicAdd(gs + 3 * i + 1, gyi);
        atomicAdd(gs + 3 * i + 2, gzi);
    }
}

}  // namespace
}  // namespace pf

namespace pf {

cudaError_t build_ball_bvh(pf_scene *scratch, BallBVH &B, int64_t N, const float *sites,
                           const float *radii, cudaStream_t st)
{
    const size_t n = (size_t)N;
    cudaError_t e;
#define PF_BV(x)                    \
    if ((e = (x)) != cudaSuccess)   \
        return e;
    PF_BV(B.keys.reserve(8 * n));
    PF_BV(B.keys_alt.reserve(8 * n));
    PF_BV(B.vals.reserve(4 * n));
    PF_BV(B.vals_alt.reserve(4 * n));
    PF_BV(B.bb.reserve(64));
    PF_BV(B.left.reserve(4 * n));
    PF_BV(B.right.reserve(4 * n));
    PF_BV(B.pint.reserve(4 * n));
    PF_BV(B.pleaf.reserve(4 * n));
    PF_BV(B.bint.reserve(sizeof(Box) * n));
    PF_BV(B.bleaf.reserve(sizeof(Box) * n));
    PF_BV(B.arrive.reserve(4 * n));
    // bounds (init min = +inf bits, max = -inf bits)
    static const float init[6] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY};
    PF_BV(cudaMemcpyAsync(B.bb.ptr, init, sizeof(init), cudaMemcpyHostToDevice, st));
    c0_bounds<<<min(ceil_div(N, 256), 1184), 256, 0, st>>>(sites, N, B.bb.as<float>());
    c1_morton<<<ceil_div(N, 256), 256, 0, st>>>(sites, N, B.bb.as<float>(),
                                                 B.keys.as<unsigned long long>(), B.vals.as<uint32_t>());
    bool alt = false;
    PF_BV(radix_sort_pairs(scratch, B.keys.as<uint64_t>(), B.vals.as<uint32_t>(),
                           B.keys_alt.as<uint64_t>(), B.vals_alt.as<uint32_t>(), N, 63, &alt, st));
    const unsigned long long *codes = (alt ? B.keys_alt : B.keys).as<unsigned long long>();
    B.order = (alt ? B.vals_alt : B.vals).as<uint32_t>();
    B.n = N;
    if (N > 1)
        c2_radix_tree<<<ceil_div(N - 1, 256), 256, 0, st>>>(codes, N, B.left.as<uint32_t>(),
                                                             B.right.as<uint32_t>(), B.pint.as<uint32_t>(),
                                                             B.pleaf.as<uint32_t>());
    PF_BV(cudaMemsetAsync(B.arrive.ptr, 0, 4 * n, st));
    c3_refit<<<ceil_div(N, 256), 256, 0, st>>>(sites, radii, B.order, N, B.left.as<uint32_t>(),
                                                B.right.as<uint32_t>(), B.pint.as<uint32_t>(),
                                                B.pleaf.as<uint32_t>(), B.bint.as<Box>(),
                                                B.bleaf.as<Box>(), B.arrive.as<int>());
    scratch->launches += 4;
#undef PF_BV
    return cudaGetLastError();
}

}  // namespace pf

struct pf_cech {
    pf_scene scratch;   // sort / scan workspaces and launch counter (reused machinery)
    pf::BallBVH bvh;
    pf::DevBuf counts, offs32, flag;
};

namespace {
thread_local std::string g_cech_err;
int cfail(int code, const std::string &m)
{
    g_cech_err = m;
    return code;
}
#define PF_CC(expr)                                                                           \
    do {                                                                                      \
        cudaError_t _e = (expr);                                                              \
        if (_e != cudaSuccess)                                                                \
            return cfail(_e == cudaErrorMemoryAllocation ? PF_ERR_OUT_OF_MEMORY : PF_ERR_CUDA, \
                         std::string(#expr) + ": " + cudaGetErrorString(_e));                \
    } while (0)
}  // namespace

extern "C" {

const char *pf_cech_last_error(void) { return g_cech_err.c_str(); }

int pf_cech_create(pf_cech **out)
{
    if (!out) return cfail(PF_ERR_INVALID_ARGUMENT, "NULL out");
    *out = new (std::nothrow) pf_cech();
    if (!*out) return cfail(PF_ERR_OUT_OF_MEMORY, "host allocation failed");
    cudaGetDevice(&(*out)->scratch.device);
    return PF_OK;
}

int pf_cech_destroy(pf_cech *h)
{
    if (!h) return PF_OK;
    cudaDeviceSynchronize();
    h->bvh.release();
    pf::DevBuf *bufs[] = {&h->counts, &h->offs32, &h->flag, &h->scratch.sort_hist,
                          &h->scratch.scan_tmp};
    for (auto *b : bufs) b->release();
    delete h;
    return PF_OK;
}

int pf_cech_build(pf_cech *h, int64_t N, const float *sites, const float *radii,
                  int64_t *nbr_offsets, int32_t *nbr_indices, int64_t capacity,
                  int64_t *num_edges, pf_stream_t stream)
{
    using namespace pf;
    if (!h || !sites || !radii || !nbr_offsets || !num_edges)
        return cfail(PF_ERR_INVALID_ARGUMENT, "NULL argument");
    if (N < 1 || N >= ((int64_t)1 << 30)) return cfail(PF_ERR_INVALID_ARGUMENT, "N must be in [1, 2^30)");
    cudaStream_t st = (cudaStream_t)stream;
    const size_t n = (size_t)N;
    PF_CC(h->counts.reserve(4 * n));
    PF_CC(h->offs32.reserve(4 * n + 16));
    PF_CC(h->flag.reserve(16));
    PF_CC(build_ball_bvh(&h->scratch, h->bvh, N, sites, radii, st));
    const uint32_t *order = h->bvh.order;
    PF_CC(cudaMemsetAsync(h->flag.ptr, 0, 4, st));
    c4_query<false><<<ceil_div(N, 128), 128, 0, st>>>(
        sites, radii, order, N, h->bvh.left.as<uint32_t>(), h->bvh.right.as<uint32_t>(), h->bvh.bint.as<Box>(),
        h->bvh.bleaf.as<Box>(), h->counts.as<int>(), nullptr, nullptr, h->flag.as<int>());
    long long *d_tot = reinterpret_cast<long long *>(h->offs32.as<uint32_t>() + ((n + 3) & ~3ull));
    PF_CC(exclusive_scan_counts(&h->scratch, h->counts.as<int>(), N, h->offs32.as<uint32_t>(), d_tot, st));
    c5_offsets<<<ceil_div(N, 256), 256, 0, st>>>(h->offs32.as<uint32_t>(), h->counts.as<int>(), N,
                                                  nbr_offsets);
    long long E = 0;
    int ovf = 0;
    PF_CC(cudaMemcpyAsync(&E, d_tot, sizeof(E), cudaMemcpyDeviceToHost, st));
    PF_CC(cudaMemcpyAsync(&ovf, h->flag.ptr, sizeof(int), cudaMemcpyDeviceToHost, st));
    PF_CC(cudaStreamSynchronize(st));
    if (ovf) return cfail(PF_ERR_CUDA, "BVH traversal stack overflow");
    if (E >= ((long long)1 << 32)) return cfail(PF_ERR_OUT_OF_MEMORY, "edge count exceeds 2^32");
    *num_edges = E;
    h->scratch.launches += 3;
    if (!nbr_indices || capacity < E) return PF_OK;   // caller sizes the index array
    c4_query<true><<<ceil_div(N, 128), 128, 0, st>>>(
        sites, radii, order, N, h->bvh.left.as<uint32_t>(), h->bvh.right.as<uint32_t>(), h->bvh.bint.as<Box>(),
        h->bvh.bleaf.as<Box>(), nullptr, nbr_offsets, nbr_indices, h->flag.as<int>());
    c6_sort_rows<<<ceil_div(N, 256), 256, 0, st>>>(nbr_offsets, N, nbr_indices);
    h->scratch.launches += 2;
    PF_CC(cudaGetLastError());
    return PF_OK;
}

int pf_connect_loss(int64_t N, const float *sites, const float *radii, const int64_t *nbr_offsets,
                    const int32_t *nbr_indices, float *loss, float *grad_sites, float *grad_radii,
                    pf_stream_t stream)
{
    if (N < 1 || !sites || !radii || !nbr_offsets || !nbr_indices)
        return cfail(PF_ERR_INVALID_ARGUMENT, "NULL argument");
    pf::c7_connect<<<pf::ceil_div(N, 256), 256, 0, (cudaStream_t)stream>>>(
        sites, radii, nbr_offsets, nbr_indices, N, loss, grad_sites, grad_radii);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cfail(PF_ERR_CUDA, cudaGetErrorString(e));
    return PF_OK;
}

int64_t pf_cech_launch_count(const pf_cech *h) { return h ? h->scratch.launches : -1; }

}  // extern "C"
