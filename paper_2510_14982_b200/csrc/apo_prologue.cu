// apo_prologue.cu -- the device loop's iteration prologue for small populations.
//
// The prologue is the stable sort by fitness (core.py:504-513) and the
// coordinator's Dr set (core.py:263-278).  At ps = 10^6 it runs as CUB
// onesweep passes + the parallel Fisher-Yates kernels (apo_kernels.cu); for
// ps <= kSmallPrologueMax those are ~12 launches of a few microseconds each
// and dominate the iteration.  Here it is one or two launches:
//   * ps <= kCountMax: ONE kernel; every CTA stages all keys (8 B) and Dr
//     targets (4 B) in shared memory and ranks by counting: the new rank of
//     element e is #(k_q < k_e) + #(k_q == k_e, q < e) -- exactly the stable
//     order by (key, previous rank); S lanes per element split the count.
//   * larger: tiles of kTile ranks are count-sorted locally (k_prologue_tiles),
//     then every element adds, per other tile, a binary search of its key in
//     that tile's sorted keys (upper bound for earlier tiles, lower bound for
//     later ones -- stability) (k_prologue_merge).
// Dr set: step j's target r_j is resolved by walking "the latest earlier step
// with the same target" (k_dr_resolve's rule) by a backward scan of the staged
// targets instead of a binary search in sorted draws.  The order is written to
// a second buffer (the caller swaps them).  Results are bit-identical to the
// CUB prologue (tests/test_gpu_parity.py).
#include "apo_kernels.cuh"

namespace apo {

constexpr int kPrologueThreads = 512;
constexpr int kCountMax = 2048;           // O(ps^2) compares: a few microseconds up to here
constexpr int kSmallPrologueMax = 24576;  // k_prologue_merge stages 8 B x ps <= 192 KB of shared memory
constexpr int kTile = 256;

__device__ __forceinline__ int dr_target(const Key& base, int j, int n) {  // k_dr_draw
    const double u = uniform(base, 1ull + (uint64_t)j);
    const int r = j + (int)(u * (double)(n - j));
    return r > n - 1 ? n - 1 : r;
}

// Mark the element Dr step j finally selects (k_dr_resolve), one warp per step: the lanes scan 32
// earlier steps per round for the latest one that also targeted p (its swap brought position q's
// element to p) -- a serial scan would wait on one shared-memory load per step.
__device__ __forceinline__ void dr_mark_warp(int j, const int* tgt, unsigned* dr_bits, int lane) {
    int p = tgt[j];
    int t = j;
    for (;;) {
        int found = -1;
        for (int hi = t; hi > 0; hi -= 32) {  // steps [hi - 32, hi), newest first
            const int q = hi - 1 - lane;
            const unsigned b = __ballot_sync(0xFFFFFFFFu, q >= 0 && tgt[q] == p);
            if (b) {
                found = hi - __ffs(b);  // lowest lane = latest step
                break;
            }
        }
        if (found < 0) break;
        p = found;
        t = found;
    }
    if (lane == 0) atomicOr(&dr_bits[p >> 5], 1u << (p & 31));
}

// dst[i] = src[i] for i < n by the CTA, eight loads in flight per thread.
__device__ __forceinline__ void stage_u64(unsigned long long* dst, const unsigned long long* __restrict__ src, int n) {
    constexpr int U = 8;
    for (int base = 0; base < n; base += U * (int)blockDim.x) {
        unsigned long long v[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int i = base + u * (int)blockDim.x + (int)threadIdx.x;
            if (i < n) v[u] = src[i];
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int i = base + u * (int)blockDim.x + (int)threadIdx.x;
            if (i < n) dst[i] = v[u];
        }
    }
}

template <int S>
__global__ void __launch_bounds__(kPrologueThreads)
    k_prologue_small(int ps, const double* __restrict__ fit, const int* __restrict__ order_in,
                     int* __restrict__ order_out, int count, Key cbase, unsigned* __restrict__ dr_bits) {
    extern __shared__ __align__(16) unsigned char smem[];
    unsigned long long* keys = reinterpret_cast<unsigned long long*>(smem);
    int* tgt = reinterpret_cast<int*>(smem + 8 * (size_t)ps);
    for (int r = threadIdx.x; r < ps; r += blockDim.x) keys[r] = sort_key(fit[order_in[r]]);
    for (int j = threadIdx.x; j < count; j += blockDim.x) tgt[j] = dr_target(cbase, j, ps);
    __syncthreads();

    // 1. stable rank by counting (S lanes per element; S divides 32)
    const int lane = threadIdx.x & 31, sub = lane & (S - 1);
    const long long nthreads = (long long)gridDim.x * blockDim.x;
    const long long first = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long span = ((long long)ps * S + 31) / 32 * 32;  // whole warps so the shuffles are uniform
    for (long long gt = first; gt < span; gt += nthreads) {
        const int e = (int)(gt / S);
        int cnt = 0;
        if (e < ps) {
            const unsigned long long ke = keys[e];
            for (int q = sub; q < ps; q += S) {
                const unsigned long long kq = keys[q];
                cnt += (kq < ke) || (kq == ke && q < e);
            }
        }
#pragma unroll
        for (int o = 1; o < S; o <<= 1) cnt += __shfl_xor_sync(0xFFFFFFFFu, cnt, o);
        if (e < ps && sub == 0) order_out[cnt] = order_in[e];
    }

    // 2. Dr set (dr_bits zeroed by the caller), one warp per step
    const int gw = (int)(first >> 5), nw = (int)(nthreads >> 5);
    for (int j = gw; j < count; j += nw) dr_mark_warp(j, tgt, dr_bits, lane);
}

// Local stable rank within a tile of kTile consecutive ranks, the tile's sorted keys, and the Dr set.
__global__ void __launch_bounds__(kTile)
    k_prologue_tiles(int ps, const double* __restrict__ fit, const int* __restrict__ order_in,
                     unsigned long long* __restrict__ tkeys, int* __restrict__ trank, int count, Key cbase,
                     unsigned* __restrict__ dr_bits) {
    extern __shared__ __align__(16) unsigned char smem[];
    unsigned long long* keys = reinterpret_cast<unsigned long long*>(smem);
    int* tgt = reinterpret_cast<int*>(smem + 8 * kTile);
    const int base = blockIdx.x * kTile, n = min(kTile, ps - base), t = threadIdx.x;
    if (t < n) keys[t] = sort_key(fit[order_in[base + t]]);
    for (int j = t; j < count; j += kTile) tgt[j] = dr_target(cbase, j, ps);
    __syncthreads();
    if (t < n) {
        const unsigned long long ke = keys[t];
        int cnt = 0;
        for (int q = 0; q < n; q++) {
            const unsigned long long kq = keys[q];
            cnt += (kq < ke) || (kq == ke && q < t);
        }
        tkeys[base + cnt] = ke;
        trank[base + t] = cnt;
    }
    const int nw = kTile / 32;
    for (int j = blockIdx.x * nw + (t >> 5); j < count; j += gridDim.x * nw) dr_mark_warp(j, tgt, dr_bits, t & 31);
}

// Global rank = local rank + per other tile the number of its keys ordered before this one; kMergeLanes
// lanes per element split the tiles and fold their counts.
constexpr int kMergeLanes = 8;
__global__ void __launch_bounds__(kPrologueThreads)
    k_prologue_merge(int ps, const unsigned long long* __restrict__ tkeys, const int* __restrict__ trank,
                     const int* __restrict__ order_in, int* __restrict__ order_out) {
    extern __shared__ __align__(16) unsigned char smem[];
    unsigned long long* keys = reinterpret_cast<unsigned long long*>(smem);
    stage_u64(keys, tkeys, ps);
    __syncthreads();
    const int ntiles = (ps + kTile - 1) / kTile;
    const int sub = threadIdx.x & (kMergeLanes - 1);
    const long long span = ((long long)ps * kMergeLanes + 31) / 32 * 32;
    for (long long gt = (long long)blockIdx.x * blockDim.x + threadIdx.x; gt < span;
         gt += (long long)gridDim.x * blockDim.x) {
        const int e = (int)(gt / kMergeLanes);
        int rank = 0;
        if (e < ps) {
            const int te = e / kTile, local = trank[e];
            const unsigned long long ke = keys[te * kTile + local];
            if (sub == 0) rank = local;
            for (int T = sub; T < ntiles; T += kMergeLanes) {
                if (T == te) continue;
                const unsigned long long* k = keys + T * kTile;
                const int n = min(kTile, ps - T * kTile);
                const bool before = T < te;  // earlier tile: keys <= ke count (ties rank first); later: keys < ke
                int c = 0;
#pragma unroll
                for (int step = kTile / 2; step > 0; step >>= 1) {
                    const int probe = c + step;
                    if (probe <= n) {
                        const unsigned long long kp = k[probe - 1];
                        if (before ? kp <= ke : kp < ke) c = probe;
                    }
                }
                // the halvings reach kTile - 1; a full tile's last key decides kTile
                if (c == kTile - 1 && n == kTile && (before ? k[kTile - 1] <= ke : k[kTile - 1] < ke)) c = kTile;
                rank += c;
            }
        }
#pragma unroll
        for (int o = 1; o < kMergeLanes; o <<= 1) rank += __shfl_xor_sync(0xFFFFFFFFu, rank, o);
        if (e < ps && sub == 0) order_out[rank] = order_in[e];
    }
}

bool prologue_small_fits(long long ps) { return ps >= 1 && ps <= kSmallPrologueMax; }

cudaError_t launch_prologue_small(int ps, const double* fit, const int* order_in, int* order_out, int count,
                                  Key cbase, unsigned* dr_bits, unsigned long long* scratch_keys, int* scratch_rank,
                                  int num_sms, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(dr_bits, 0, 4 * (size_t)((ps + 31) / 32), st);
    if (e != cudaSuccess) return e;
    const size_t tbytes = 4 * (size_t)(count > 0 ? count : 0);
    if (ps > kCountMax) {
        const int ntiles = (ps + kTile - 1) / kTile;
        const size_t b1 = 8 * kTile + tbytes, b2 = 8 * (size_t)ps;
        if ((e = cudaFuncSetAttribute(k_prologue_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)b1)))
            return e;
        if ((e = cudaFuncSetAttribute(k_prologue_merge, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)b2)))
            return e;
        k_prologue_tiles<<<ntiles, kTile, b1, st>>>(ps, fit, order_in, scratch_keys, scratch_rank, count, cbase,
                                                      dr_bits);
        const int g2 = (int)(((long long)ps * kMergeLanes + kPrologueThreads - 1) / kPrologueThreads);
        k_prologue_merge<<<g2 < num_sms ? g2 : num_sms, kPrologueThreads, b2, st>>>(ps, scratch_keys, scratch_rank,
                                                                                     order_in, order_out);
        return cudaGetLastError();
    }
    const size_t bytes = 8 * (size_t)ps + tbytes;
    // lanes per element: enough threads to cover the GPU once, at most a warp per element
    const int S = ps >= 1024 ? 16 : 32;
    const long long want = ((long long)ps * S + kPrologueThreads - 1) / kPrologueThreads;
    const int grid = (int)(want < num_sms ? (want < 1 ? 1 : want) : num_sms);
    auto launch = [&](auto fn) {
        cudaError_t err = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
        if (err != cudaSuccess) return err;
        fn<<<grid, kPrologueThreads, bytes, st>>>(ps, fit, order_in, order_out, count, cbase, dr_bits);
        return cudaGetLastError();
    };
    if (S == 16) return launch(k_prologue_small<16>);
    return launch(k_prologue_small<32>);
}

}  // namespace apo
