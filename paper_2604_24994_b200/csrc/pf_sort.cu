// pf_sort.cu -- K4: stable LSD radix sort of (u64 or u32 key, u32 value) pairs,
// 9-bit (u64) / 8-bit (u32) digits, only over the significant low `end_bit` bits (32 key bits + the tile
// bits, "global sort ... similar to 3DGS").
//
// Per pass:  (1) per-block digit histograms (digit-major [256][nblocks]),
//            (2) exclusive scan of that array (the K2 scan kernels),
//            (3) stable scatter: warp-level multisplit ranking with
//                one ballot per digit bit (PF_SORT_BALLOT; __match_any_sync measured
//                6% slower), per-warp digit counters in shared memory,
//                block prefix over warps, then a block-local shuffle through
//                shared memory so each digit's run is stored contiguously.
// Stability: warp w of block b owns keys [b*TILE + w*32*I, +32*I) in I rounds of
// 32 consecutive keys; ranks follow (round, lane) = input order.
#include <cuda_runtime.h>

#include "pf_internal.cuh"

namespace pf {

cudaError_t exclusive_scan_counts(pf_scene *s, const int *cnt, int64_t n, uint32_t *offs,
                                  long long *d_total, cudaStream_t st);

#ifndef PF_SORT_THREADS
#define PF_SORT_THREADS 512
#endif
#ifndef PF_SORT_TILE
#define PF_SORT_TILE 4096
#endif
constexpr int kSortThreads = PF_SORT_THREADS, kSortItems = PF_SORT_TILE / PF_SORT_THREADS,
              kSortTile = kSortThreads * kSortItems, kSortWarps = kSortThreads / 32;
// digit bits of the 64-bit-key sorts: the visible cells' 35-bit (view, depth) keys in 4
// passes instead of 5 (measured K4 0.717 -> 0.690 ms per train8_1m step; the Cech
// build's 63-bit Morton codes in 7 instead of 8)
#ifndef PF_SORT_BITS_WIDE
#define PF_SORT_BITS_WIDE 9
#endif

// Lanes of the warp holding the same digit d (d in [0, 2^kBits], kRadix = the invalid
// sentinel): with PF_SORT_BALLOT one ballot per digit bit (kBits + 1 ballots, full-rate
// vote and logic ops) instead of __match_any_sync.
#ifndef PF_SORT_BALLOT
#define PF_SORT_BALLOT 1
#endif
template <int kBits>
__device__ __forceinline__ unsigned digit_peers(int d)
{
    if (!PF_SORT_BALLOT) return __match_any_sync(0xffffffffu, d);
    unsigned peers = 0xffffffffu;
#pragma unroll
    for (int b = 0; b <= kBits; ++b) {
        const bool bit = (d >> b) & 1;
        const unsigned v = __ballot_sync(0xffffffffu, bit);
        peers &= bit ? v : ~v;
    }
    return peers;
}

template <class KeyT, int kRadixBits>
__global__ void __launch_bounds__(kSortThreads)
k4_histogram(const KeyT *__restrict__ keys, int64_t n, int shift, int nb, int *__restrict__ hist)
{
    constexpr int kRadix = 1 << kRadixBits;
    __shared__ int h[kSortWarps][kRadix];
    const int warp = threadIdx.x >> 5;
    for (int q = threadIdx.x; q < kSortWarps * kRadix; q += kSortThreads) (&h[0][0])[q] = 0;
    __syncthreads();
    int64_t base = (int64_t)blockIdx.x * kSortTile;
#pragma unroll 4
    for (int k = 0; k < kSortItems; ++k) {
        int64_t idx = base + (int64_t)k * kSortThreads + threadIdx.x;
        if (idx < n) {
            int d = (int)((keys[idx] >> shift) & (kRadix - 1));
            atomicAdd(&h[warp][d], 1);
        }
    }
    __syncthreads();
    for (int d = threadIdx.x; d < kRadix; d += kSortThreads) {
        int t = 0;
#pragma unroll
        for (int w = 0; w < kSortWarps; ++w) t += h[w][d];
        hist[(int64_t)d * nb + blockIdx.x] = t;
    }
}

// Scatter with a block-local shuffle: every key gets its position inside the
// block's digit-sorted tile (digit start + warp prefix + rank), the tile is
// staged in shared memory, and the threads then write it out in tile order, so
// each digit's run (about 16 keys per block) goes to consecutive addresses:
// coalesced stores instead of one scattered 8-byte store per key.
template <class KeyT, int kRadixBits>
constexpr size_t scatter_smem()
{
    constexpr int kRadix = 1 << kRadixBits;
    return (size_t)kSortTile * (sizeof(KeyT) + sizeof(uint32_t)) +
           (size_t)kSortWarps * kRadix * sizeof(uint32_t) + 2 * kRadix * sizeof(uint32_t);
}

// Onesweep mode (kOne): the block takes its partition from a ticket counter (so a
// partition only ever waits on partitions already running), publishes its digit counts,
// and finds each digit's exclusive prefix over the earlier partitions by decoupled
// look-back on `status` ([partition][digit]: count | flag; kAgg = this partition's
// count, kPre = inclusive prefix); the digit's global start comes from the one
// upfront histogram of every pass (k4_hist_all).  Without kOne: per-pass histogram +
// scan offsets (digit_offs[digit * nb + block]).
constexpr uint32_t kAgg = 1u << 30, kPre = 2u << 30, kValMask = kAgg - 1u;

template <class KeyT, int kRadixBits, bool kOne = false>
__global__ void __launch_bounds__(kSortThreads)
k4_scatter(const KeyT *__restrict__ kin, const uint32_t *__restrict__ vin, KeyT *__restrict__ kout,
           uint32_t *__restrict__ vout, int64_t n, int shift, int nb,
           const uint32_t *__restrict__ digit_offs, uint32_t *status = nullptr,
           uint32_t *ticket = nullptr)
{
    constexpr int kRadix = 1 << kRadixBits;
    extern __shared__ __align__(16) unsigned char sort_smem[];
    KeyT *sk = reinterpret_cast<KeyT *>(sort_smem);
    uint32_t *sv = reinterpret_cast<uint32_t *>(sk + kSortTile);
    uint32_t(*wh)[kRadix] = reinterpret_cast<uint32_t(*)[kRadix]>(sv + kSortTile);
    uint32_t *dstart = reinterpret_cast<uint32_t *>(wh + kSortWarps);
    uint32_t *gbase = dstart + kRadix;
    __shared__ int part_s;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (kOne && threadIdx.x == 0) part_s = (int)atomicAdd(ticket, 1u);
    for (int q = threadIdx.x; q < kSortWarps * kRadix; q += kSortThreads) (&wh[0][0])[q] = 0;
    __syncthreads();
    const int part = kOne ? part_s : (int)blockIdx.x;
    const unsigned lt_mask = (1u << lane) - 1u;
    const int64_t bbase = (int64_t)part * kSortTile;
    const int64_t wbase = bbase + (int64_t)warp * (32 * kSortItems);
    KeyT key[kSortItems];
    uint32_t val[kSortItems], rank[kSortItems];
    int dig[kSortItems];
#pragma unroll
    for (int r = 0; r < kSortItems; ++r) {
        int64_t idx = wbase + r * 32 + lane;
        bool valid = idx < n;
        key[r] = valid ? kin[idx] : KeyT(0);
        val[r] = valid ? vin[idx] : 0u;
    }
#pragma unroll
    for (int r = 0; r < kSortItems; ++r) {
        int64_t idx = wbase + r * 32 + lane;
        bool valid = idx < n;
        int d = valid ? (int)((key[r] >> shift) & (kRadix - 1)) : kRadix;
        unsigned peers = digit_peers<kRadixBits>(d);
        uint32_t before = valid ? wh[warp][d] : 0u;
        __syncwarp();
        if (valid && lane == __ffs(peers) - 1) wh[warp][d] = before + __popc(peers);
        __syncwarp();
        rank[r] = before + __popc(peers & lt_mask);
        dig[r] = d;
    }
    __syncthreads();
    // per digit: warp prefixes, block total, global base of this block's run
    for (int d = threadIdx.x; d < kRadix; d += kSortThreads) {
        uint32_t run = 0;
#pragma unroll
        for (int w = 0; w < kSortWarps; ++w) {
            const uint32_t c = wh[w][d];
            wh[w][d] = run;
            run += c;
        }
        dstart[d] = run;
        if (kOne) {
            uint32_t *st = status + (size_t)part * kRadix + d;
            if (part == 0) {
                atomicExch(st, run | kPre);
                gbase[d] = digit_offs[d];
            } else {
                atomicExch(st, run | kAgg);
                uint32_t excl = 0;
                for (int j = part - 1; j >= 0;) {
                    const uint32_t v = __ldcv(status + (size_t)j * kRadix + d);
                    if (!(v & (kAgg | kPre))) continue;   // partition j not published yet
                    excl += v & kValMask;
                    if (v & kPre) break;
                    --j;
                }
                atomicExch(st, (excl + run) | kPre);
                gbase[d] = digit_offs[d] + excl;
            }
        } else {
            gbase[d] = digit_offs[(int64_t)d * nb + blockIdx.x];
        }
    }
    __syncthreads();
    if (warp == 0) {   // exclusive scan of the digit totals (kRadix / 32 per lane)
        uint32_t v[kRadix / 32], sum = 0;
#pragma unroll
        for (int q = 0; q < kRadix / 32; ++q) {
            v[q] = dstart[lane * (kRadix / 32) + q];
            sum += v[q];
        }
        uint32_t incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        uint32_t run = incl - sum;
#pragma unroll
        for (int q = 0; q < kRadix / 32; ++q) {
            dstart[lane * (kRadix / 32) + q] = run;
            run += v[q];
        }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kSortItems; ++r) {
        if (dig[r] < kRadix) {
            const uint32_t lp = dstart[dig[r]] + wh[warp][dig[r]] + rank[r];
            sk[lp] = key[r];
            sv[lp] = val[r];
        }
    }
    __syncthreads();
    const int nvalid = (int)min((int64_t)kSortTile, n - bbase);
    for (int q = threadIdx.x; q < nvalid; q += kSortThreads) {
        const KeyT k = sk[q];
        const int d = (int)((k >> shift) & (kRadix - 1));
        const uint32_t pos = gbase[d] + ((uint32_t)q - dstart[d]);
        kout[pos] = k;
        vout[pos] = sv[q];
    }
}

// Onesweep: the digit histograms of every pass in one read of the keys
template <class KeyT, int kRadixBits>
__global__ void __launch_bounds__(kSortThreads)
k4_hist_all(const KeyT *__restrict__ keys, int64_t n, int npass, uint32_t *__restrict__ ghist)
{
    constexpr int kRadix = 1 << kRadixBits, kMaxPass = (int)(8 * sizeof(KeyT) + kRadixBits - 1) / kRadixBits;
    __shared__ uint32_t h[kMaxPass][kRadix];
    for (int q = threadIdx.x; q < kMaxPass * kRadix; q += kSortThreads) (&h[0][0])[q] = 0u;
    __syncthreads();
    // warp-aggregated: the high digits take few values (view bits, float order
    // bits), so per-key shared atomics would serialise on a handful of bins
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int64_t base = ((int64_t)blockIdx.x * kSortWarps + warp) * 32; base < n;
         base += (int64_t)gridDim.x * kSortThreads) {
        const int64_t i = base + lane;
        const bool valid = i < n;
        const KeyT k = valid ? keys[i] : KeyT(0);
        for (int p = 0; p < npass; ++p) {
            const int d = valid ? (int)((k >> (p * kRadixBits)) & (kRadix - 1)) : -1;
            const unsigned peers = digit_peers<kRadixBits>(d < 0 ? kRadix : d);
            if (valid && lane == __ffs(peers) - 1) atomicAdd(&h[p][d], (uint32_t)__popc(peers));
        }
    }
    __syncthreads();
    for (int q = threadIdx.x; q < npass * kRadix; q += kSortThreads) {
        const uint32_t c = (&h[0][0])[q];
        if (c) atomicAdd(ghist + q, c);
    }
}

// exclusive scan of each pass's kRadix digit counts (block p = pass p, in place)
template <int kRadixBits>
__global__ void __launch_bounds__(kSortThreads) k4_scan_digits(uint32_t *__restrict__ ghist)
{
    constexpr int kRadix = 1 << kRadixBits, kPer = (kRadix + kSortThreads - 1) / kSortThreads;
    __shared__ uint32_t ws[kSortWarps];
    uint32_t *g = ghist + (size_t)blockIdx.x * kRadix;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t v[kPer], sum = 0;
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
        const int d = threadIdx.x * kPer + q;
        v[q] = d < kRadix ? g[d] : 0u;
        sum += v[q];
    }
    uint32_t inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) ws[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < kSortWarps ? ws[lane] : 0u, wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += y;
        }
        if (lane < kSortWarps) ws[lane] = wi - w;
    }
    __syncthreads();
    uint32_t run = inc - sum + ws[warp];
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
        const int d = threadIdx.x * kPer + q;
        if (d < kRadix) g[d] = run;
        run += v[q];
    }
}

// 1: upfront histograms of every pass + a decoupled look-back scatter per pass (no
// per-pass histogram / scan launches).  Bit-exact (binning and Cech tests pass) but
// measured slower on B200: train8_1m sort 0.69 -> 0.94 ms per step (one thread per
// digit walks the look-back partition by partition; ~150-400 partitions are in flight
// at once, so most walks are long), nerfsynth200k 0.32 -> 0.38 ms.  Off.
#ifndef PF_SORT_ONESWEEP
#define PF_SORT_ONESWEEP 0
#endif

template <class KeyT, int kRadixBits>
static cudaError_t radix_sort_t(pf_scene *s, KeyT *keys, uint32_t *vals, KeyT *keys_alt,
                                uint32_t *vals_alt, int64_t n, int end_bit, bool *result_in_alt,
                                cudaStream_t st)
{
    constexpr int kRadix = 1 << kRadixBits;
    *result_in_alt = false;
    if (n <= 1) return cudaSuccess;
    int nb = ceil_div(n, kSortTile);
    size_t hist_n = (size_t)kRadix * nb;
    cudaError_t err = s->sort_hist.reserve(hist_n * (sizeof(int) + sizeof(uint32_t)) + 64);
    if (err != cudaSuccess) return err;
    int *hist = s->sort_hist.as<int>();
    uint32_t *offs = reinterpret_cast<uint32_t *>(hist + hist_n);
    long long *dummy_total = reinterpret_cast<long long *>(
        (reinterpret_cast<uintptr_t>(offs + hist_n) + 15) & ~uintptr_t(15));
    KeyT *ka = keys, *kb = keys_alt;
    uint32_t *va = vals, *vb = vals_alt;
    bool alt = false;
    cudaEvent_t ev;
    constexpr size_t smem = scatter_smem<KeyT, kRadixBits>();
    cudaFuncSetAttribute(k4_scatter<KeyT, kRadixBits>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    const int npass = (end_bit + kRadixBits - 1) / kRadixBits;
    if (PF_SORT_ONESWEEP && n < (int64_t)kValMask) {
        // ghist [npass][kRadix] | tickets [npass] | status [npass][nb][kRadix], zeroed at once
        const size_t words = (size_t)npass * kRadix + npass + (size_t)npass * nb * kRadix;
        err = s->sort_status.reserve(words * sizeof(uint32_t));
        if (err != cudaSuccess) return err;
        uint32_t *ghist = s->sort_status.as<uint32_t>(), *tick = ghist + (size_t)npass * kRadix,
                 *status = tick + npass;
        cudaFuncSetAttribute(k4_scatter<KeyT, kRadixBits, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        stage_begin(s, 4, st, &ev);
        err = cudaMemsetAsync(ghist, 0, words * sizeof(uint32_t), st);
        if (err != cudaSuccess) return err;
        const int hb = nb < 1184 ? nb : 1184;   // 8 blocks per SM, grid-stride
        k4_hist_all<KeyT, kRadixBits><<<hb, kSortThreads, 0, st>>>(keys, n, npass, ghist);
        k4_scan_digits<kRadixBits><<<npass, kSortThreads, 0, st>>>(ghist);
        s->launches += 2;
        for (int p = 0; p < npass; ++p) {
            k4_scatter<KeyT, kRadixBits, true><<<nb, kSortThreads, smem, st>>>(
                ka, va, kb, vb, n, p * kRadixBits, nb, ghist + (size_t)p * kRadix,
                status + (size_t)p * nb * kRadix, tick + p);
            ++s->launches;
            err = cudaGetLastError();
            if (err != cudaSuccess) return err;
            KeyT *tk = ka; ka = kb; kb = tk;
            uint32_t *tv = va; va = vb; vb = tv;
            alt = !alt;
        }
        stage_end(s, 4, st, ev);
        *result_in_alt = alt;
        return cudaGetLastError();
    }
    stage_begin(s, 4, st, &ev);
    for (int shift = 0; shift < end_bit; shift += kRadixBits) {
        k4_histogram<KeyT, kRadixBits><<<nb, kSortThreads, 0, st>>>(ka, n, shift, nb, hist);
        ++s->launches;
        err = exclusive_scan_counts(s, hist, (int64_t)hist_n, offs, dummy_total, st);
        if (err != cudaSuccess) return err;
        k4_scatter<KeyT, kRadixBits><<<nb, kSortThreads, smem, st>>>(ka, va, kb, vb, n, shift, nb, offs);
        ++s->launches;
        err = cudaGetLastError();
        if (err != cudaSuccess) return err;
        KeyT *tk = ka; ka = kb; kb = tk;
        uint32_t *tv = va; va = vb; vb = tv;
        alt = !alt;
    }
    stage_end(s, 4, st, ev);
    *result_in_alt = alt;
    return cudaGetLastError();
}

cudaError_t radix_sort_pairs(pf_scene *s, uint64_t *keys, uint32_t *vals, uint64_t *keys_alt,
                             uint32_t *vals_alt, int64_t n, int end_bit, bool *result_in_alt,
                             cudaStream_t st)
{
    return radix_sort_t<unsigned long long, PF_SORT_BITS_WIDE>(s, (unsigned long long *)keys, vals,
                                            (unsigned long long *)keys_alt, vals_alt, n, end_bit,
                                            result_in_alt, st);
}

cudaError_t radix_sort_pairs32(pf_scene *s, uint32_t *keys, uint32_t *vals, uint32_t *keys_alt,
                               uint32_t *vals_alt, int64_t n, int end_bit, bool *result_in_alt,
                               cudaStream_t st)
{
    return radix_sort_t<uint32_t, 8>(s, keys, vals, keys_alt, vals_alt, n, end_bit, result_in_alt, st);
}

}  // namespace pf
