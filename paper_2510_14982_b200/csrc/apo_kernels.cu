// apo_kernels.cu -- the small kernels and the C ABI of libapo_b200.so.
//
// Built with --fmad=false (oracle-exact arithmetic).
// Kernels defined here:
//   k_init              iteration-0 draws + evaluation (engine.py:116-139)
//   k_evaluate          batch fitness (objectives.py:222-228)
//   k_make_keys         fitness -> order-preserving u64 keys for the stable
//                       radix sort (core.py:504-513)
//   k_dr_draw/resolve   coordinator Dr set (core.py:263-278) as a parallel
//                       partial Fisher-Yates (see apo_update.cuh:build_mask)
//   k_threshold_tables  multilevel Otsu/Kapur prefix tables
//   k_histogram_u8      shared-memory privatised 256-bin histogram
// The hot kernels are templates in apo_kernels.cuh, instantiated in their own
// TUs and reached through pick_* getters:
//   k_update_group / k_update   the fused per-protozoon update (apo_update_*.cu)
//   k_cec_eval                  CEC2022 DMMA evaluation + select (apo_cec_eval.cu)
//   k_run_batch                 one CTA per independent run (apo_batch_*.cu)
//   k_cec_prep/k_dgemm_nn/k_cec_finish   large-D GEMM path (apo_cec_gemm.cu)
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <string>
#include <utility>
#include <vector>

#include "apo_b200.h"
#include "apo_kernels.cuh"

using namespace apo;

namespace apo_philox {  // apo_update_sel.cu / apo_update_dense.cu built with APO_PHILOX_VARIANT
const void* pick_update_sel(int dim, bool cand_only, bool cec, bool many);
const void* pick_update_dense(int dim, bool cand_only, bool cec, bool many);
}

static_assert(sizeof(apo_draw_table) == sizeof(DrawTable) && offsetof(apo_draw_table, miss) == offsetof(DrawTable, miss),
              "apo_draw_table (include/apo_b200.h) and DrawTable (apo_device.cuh) must share one layout");

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    if (code == APO_ECUDA) (void)cudaGetLastError();  // a failed launch must not fail the next call's check
    return code;
}

#define APO_CUDA(call)                                                                             \
    do {                                                                                           \
        cudaError_t e_ = (call);                                                                   \
        if (e_ != cudaSuccess) return fail(APO_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

#define APO_CHECK(cond, msg)                         \
    do {                                             \
        if (!(cond)) return fail(APO_EINVAL, (msg)); \
    } while (0)


// Scratch from cudaMallocAsync stays in the device's stream-ordered pool once freed: with the default
// release threshold (0) every synchronisation hands it back and the next step re-maps it, which at the
// C4 shape cost 50-100 ms spikes in step() (tools/e2e_probe.py).
void keep_mempool() {
    static const bool done = [] {
        int dev = 0;
        cudaMemPool_t pool;
        if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t keep = ~0ull;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
        return true;
    }();
    (void)done;
}

inline cudaStream_t as_stream(void* s) {
    keep_mempool();
    return reinterpret_cast<cudaStream_t>(s);
}

int num_sms() {
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

// Warps per CTA for a given dim so the per-warp scratch fits comfortably.
// Largest dimension the update, initialise and evaluate kernels take: ONE warp's warp-path scratch
// (candidate, terms and auxiliary rows, permutation) must fit a CTA's opt-in shared memory
// (6403 on a B200's 227 KB).
int smem_optin();
int64_t max_dim_supported() {
    static int64_t m = 0;
    if (m == 0) {
        int64_t d = 8192;
        while (d > 1 && warp_scratch_bytes((int)d) + 1024 > (size_t)smem_optin()) d--;
        m = d;
    }
    return m;
}

int warps_for_dim(int64_t dim) {
    size_t per = warp_scratch_bytes((int)dim);
    int w = kWarps;
    while (w > 1 && per * (size_t)w > 96 * 1024) w >>= 1;
    return w;
}

// Per-launch host work is cached per (kernel, device): cudaFuncSetAttribute only when a launch needs
// more dynamic shared memory than already granted, occupancy queried once per launch shape (the
// device loop at ps ~ 1e5 was host-bound on these calls).
std::mutex g_attr_mu;
std::map<std::pair<const void*, int>, size_t> g_smem_set;
std::map<std::tuple<const void*, int, int, size_t>, int> g_occ;

int set_smem(const void* fn, size_t bytes) {
    // always (the first time): the 48 KB default covers static + dynamic shared memory, so a request just
    // under 48 KB still fails to launch once the kernel's own static arrays are added (k_run_batch,
    // ps = 48, D = 6)
    if (bytes == 0) return APO_OK;
    int dev = 0;
    APO_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_attr_mu);
    size_t& have = g_smem_set[{fn, dev}];
    if (have >= bytes) return APO_OK;
    APO_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    have = bytes;
    return APO_OK;
}

int occupancy(int* per_sm, const void* fn, int threads, size_t smem) {
    int dev = 0;
    APO_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_attr_mu);
    const auto key = std::make_tuple(fn, dev, threads, smem);
    auto it = g_occ.find(key);
    if (it == g_occ.end()) {
        int v = 0;
        APO_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, fn, threads, smem));
        it = g_occ.emplace(key, v).first;
    }
    *per_sm = it->second;
    return APO_OK;
}

ObjDesc to_desc(const apo_objective* o) {
    ObjDesc d;
    d.code = o->code;
    d.table_len = o->table_len;
    d.table = o->table;
    d.cec.fn = o->code >= APO_OBJ_CEC2022_BASE ? o->code - APO_OBJ_CEC2022_BASE : 0;
    d.cec.shift = o->shift;
    d.cec.rot_t = o->rot_t;
    d.cec.shuffle = o->shuffle;
    d.cec.rot_pad = o->rot_pad;
    d.cec.rot_gemm = o->rot_gemm;
    d.flags = o->flags;
    return d;
}

int check_objective(const apo_objective* o, int64_t dim) {
    APO_CHECK(o != nullptr, "objective descriptor is NULL");
    const bool cec = o->code > APO_OBJ_CEC2022_BASE && o->code <= APO_OBJ_CEC2022_BASE + 12;
    APO_CHECK(cec || (o->code >= APO_OBJ_SPHERE && o->code <= APO_OBJ_KAPUR_ML), "unsupported objective code");
    if (o->code == APO_OBJ_OTSU_ML || o->code == APO_OBJ_KAPUR_ML) {
        APO_CHECK(o->table && o->table_len >= APO_THRESHOLD_TABLE_LEN, "threshold objective needs the 515-entry table");
        APO_CHECK(dim >= 1 && dim <= kThresholdMaxK, "multilevel thresholding supports 1..32 thresholds");
    }
    if (cec) {
        APO_CHECK(o->shift && o->rot_t, "CEC2022 objectives need shift and rotation data");
        const int fn = o->code - APO_OBJ_CEC2022_BASE;
        APO_CHECK(fn < 6 || fn > 8 || o->shuffle, "CEC2022 hybrid functions need a shuffle");
        APO_CHECK(dim >= ((fn == 7 || fn == 8) ? 5 : 2), "CEC2022 dim too small (F7/F8 need >= 5, others >= 2)");
    }
    if (o->code == APO_OBJ_ELLIPTIC) APO_CHECK(o->table && o->table_len >= dim, "elliptic needs dim weights");
    if (o->code == APO_OBJ_TABLE) APO_CHECK(o->table && o->table_len >= 1, "table objective needs a table");
    return APO_OK;
}



__global__ void __launch_bounds__(kThreads) k_init(int rng, uint64_t seed, int ps, int dim, int ld, double lower,
                                                   double span, ObjDesc O, double* __restrict__ pos,
                                                   double* __restrict__ fit, unsigned long long* trace_key) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ unsigned long long red_min[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const WarpScratch s = warp_scratch(smem + (size_t)warp * warp_scratch_bytes(dim), dim);
    unsigned long long my_min = ~0ull;
    for (int r0 = blockIdx.x * nwarps + warp; r0 < ps; r0 += gridDim.x * nwarps) {
        const Key base = stream_key(rng, seed, 0, (uint64_t)(r0 + 1));
        double* row = pos + (size_t)r0 * ld;
        for (int d = lane; d < dim; d += 32) {
            const double c = lower + uniform(base, (uint64_t)d) * span;
            s.cand[d] = c;
            row[d] = c;
        }
        __syncwarp();
        if (!fit) continue;  // positions only (k_cec_eval evaluates them)
        const double f = eval_warp(O, s.cand, s.terms, dim, lane, s.aux);
        if (lane == 0) fit[r0] = f;
        const unsigned long long k = sort_key(f);
        my_min = k < my_min ? k : my_min;
    }
    if (lane == 0) red_min[warp] = my_min;
    __syncthreads();
    if (threadIdx.x == 0 && trace_key) {
        unsigned long long m = ~0ull;
        for (int k = 0; k < nwarps; k++) m = red_min[k] < m ? red_min[k] : m;
        if (m != ~0ull) atomicMin(trace_key, m);
    }
}

__global__ void __launch_bounds__(kThreads) k_evaluate(const double* __restrict__ x, int n, int dim, int ld, ObjDesc O,
                                                       double* __restrict__ out) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const WarpScratch s = warp_scratch(smem + (size_t)warp * warp_scratch_bytes(dim), dim);
    for (int r0 = blockIdx.x * nwarps + warp; r0 < n; r0 += gridDim.x * nwarps) {
        const double* row = x + (size_t)r0 * ld;
        for (int d = lane; d < dim; d += 32) s.cand[d] = row[d];
        __syncwarp();
        const double f = eval_warp(O, s.cand, s.terms, dim, lane, s.aux);
        if (lane == 0) out[r0] = f;
    }
}

__global__ void k_make_keys(int n, const double* __restrict__ fit, const int* __restrict__ order,
                            unsigned long long* __restrict__ keys, int* __restrict__ vals) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
        const int slot = order ? order[r] : r;
        keys[r] = sort_key(fit[slot]);
        vals[r] = slot;
    }
}

__global__ void k_iota(int n, int* __restrict__ v) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) v[r] = r;
}

// Coordinator Dr set, parallel partial Fisher-Yates (rng.py:137-156 on
// counters 1.., core.py:271-278).  Step j's target r_j is packed with j so a
// radix sort groups same-target steps in step order; resolution then walks
// "latest earlier step with the same target" by binary search.
__global__ void k_dr_draw(int count, int n, Key base, unsigned long long* __restrict__ keys) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < count; j += gridDim.x * blockDim.x) {
        const double u = uniform(base, 1ull + (uint64_t)j);
        int r = j + (int)(u * (double)(n - j));
        if (r > n - 1) r = n - 1;
        keys[j] = ((unsigned long long)r << 32) | (unsigned)j;
    }
}

__device__ __forceinline__ int latest_before(const unsigned long long* keys, int count, unsigned p, unsigned t) {
    // largest index q with keys[q] < (p<<32 | t); -1 if none or target differs
    const unsigned long long probe = ((unsigned long long)p << 32) | t;
    int lo = 0, hi = count;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (keys[mid] < probe) lo = mid + 1;
        else hi = mid;
    }
    const int q = lo - 1;
    if (q < 0 || (unsigned)(keys[q] >> 32) != p) return -1;
    return (int)(keys[q] & 0xFFFFFFFFull);
}

__global__ void k_dr_resolve(int count, int n, Key base, const unsigned long long* __restrict__ keys,
                             unsigned* __restrict__ bits, uint8_t* __restrict__ bytes) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < count; j += gridDim.x * blockDim.x) {
        const double u = uniform(base, 1ull + (uint64_t)j);
        int p = j + (int)(u * (double)(n - j));
        if (p > n - 1) p = n - 1;
        int t = j;
        for (;;) {
            const int q = latest_before(keys, count, (unsigned)p, (unsigned)t);
            if (q < 0) break;
            p = q;
            t = q;
        }
        if (bits) atomicOr(&bits[p >> 5], 1u << (p & 31));
        if (bytes) bytes[p] = 1;
    }
}

__global__ void k_gather_rows(int n, int dim, int ld, const double* __restrict__ pos0,
                              const double* __restrict__ pos1, const uint8_t* __restrict__ sel,
                              const double* __restrict__ fit, const int* __restrict__ order,
                              double* __restrict__ out_pos, double* __restrict__ out_fit) {
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    for (int r = warp; r < n; r += nw) {
        const int slot = order[r];
        const double* src = (sel[slot] ? pos1 : pos0) + (size_t)slot * ld;
        for (int d = lane; d < dim; d += 32) out_pos[(size_t)r * dim + d] = src[d];
        if (lane == 0 && out_fit) out_fit[r] = fit[slot];
    }
}

__global__ void k_histogram_u8(const uint8_t* __restrict__ px, long long n, unsigned long long* __restrict__ counts) {
    __shared__ unsigned h[kWarps][256];
    const int warp = threadIdx.x >> 5;
    for (int k = threadIdx.x; k < kWarps * 256; k += blockDim.x) (&h[0][0])[k] = 0u;
    __syncthreads();
    const long long nvec = n / 16;
    const uint4* v = reinterpret_cast<const uint4*>(px);
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < nvec;
         q += (long long)gridDim.x * blockDim.x) {
        const uint4 w = v[q];
        const unsigned words[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int a = 0; a < 4; a++) {
#pragma unroll
            for (int b = 0; b < 4; b++) atomicAdd(&h[warp][(words[a] >> (8 * b)) & 0xFFu], 1u);
        }
    }
    for (long long q = nvec * 16 + blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n;
         q += (long long)gridDim.x * blockDim.x)
        atomicAdd(&h[warp][px[q]], 1u);
    __syncthreads();
    for (int b = threadIdx.x; b < 256; b += blockDim.x) {
        unsigned long long s = 0;
        for (int w = 0; w < kWarps; w++) s += h[w][b];
        if (s) atomicAdd(&counts[b], s);
    }
}

// Prefix tables for the multilevel threshold objectives, one thread in
// histogram order (the order oracle/threshold_oracle.c sums in).
__global__ void k_threshold_tables(const long long* __restrict__ counts, int method, double* __restrict__ tab) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    long long n = 0;
    for (int v = 0; v < 256; v++) n += counts[v];
    tab[0] = (double)n;
    long long c = 0;
    double s = 0.0;
    tab[1] = 0.0;
    tab[258] = 0.0;
    for (int v = 0; v < 256; v++) {
        c += counts[v];
        tab[2 + v] = (double)c;
        if (method == 0) {
            s += (double)v * (double)counts[v];
        } else if (counts[v] > 0) {
            const double p = (double)counts[v] / (double)n;
            s += p * log(p);
        }
        tab[259 + v] = s;
    }
}

__global__ void k_debug_cos(const double* x, double* out, long long n) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x)
        out[k] = cos_glibc(x[k]);
}

__global__ void k_debug_exp(const double* x, double* out, long long n) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x)
        out[k] = exp_glibc(x[k]);
}



int smem_optin() {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess) optin = 227 * 1024;
    return optin;
}

// Fused update launch.  CEC2022 objectives with dim <= kCecEvalMaxDim and a
// cand_ok scratch run as two kernels: k_update_group writes the candidates,
// k_cec_eval evaluates them in DMMA tiles and finishes the update.
// mid_event (nullable) is recorded between the two.

int launch_cec_eval(bool sel_mode, const UpdArgs& a, cudaStream_t st, uint8_t* cand_ok, unsigned* tile_counter,
                    int init);

// Which kernels an update launch runs (apo_run_update_path): 0 one fused kernel (basic objectives,
// or CEC2022 without DMMA tables), 1 CEC2022 split (k_update_group candidates + k_cec_eval), 2 fused
// CEC2022 (k_update_cec), 3 CEC2022 GEMM (candidates + k_dgemm_nn + k_cec_finish), 4 the reference's
// objectives split (candidates + k_basic_eval).
int update_path(bool sel_mode, const UpdArgs& a0, bool have_cand_ok, bool have_counter) {
    UpdArgs a = a0;
    const int dim = a.P.dim;
    if ((a.O.flags & APO_OBJ_FMA_SMALL_D) && dim <= 32) a.O.cec.rot_pad = nullptr;  // launch_update does the same
    const int fn_id = a.O.code - APO_OBJ_CEC2022_BASE;
    const bool cec = have_cand_ok && a.O.code > APO_OBJ_CEC2022_BASE;
    if (cec && dim <= kGroupMaxDim && dim <= kCecEvalMaxDim && a.O.cec.rot_pad != nullptr) {
        // APO_CEC_FUSED: 0 split (two kernels, the default: measured faster), 1 one kernel
        const int env_fused = getenv("APO_CEC_FUSED") ? atoi(getenv("APO_CEC_FUSED")) : 0;
        size_t fsmem = 0;
        int fss = 0;
        if (sel_mode && env_fused == 1 && have_counter && fused_cec_shape(a, smem_optin(), &fsmem, &fss) > 0) return 2;
        return 1;
    }
    if (cec && dim > kCecEvalMaxDim && a.O.cec.rot_gemm != nullptr && (fn_id <= 8 || fn_id == 10)) return 3;
    const int bs = getenv("APO_BASIC_SPLIT_MIN_DIM") ? atoi(getenv("APO_BASIC_SPLIT_MIN_DIM")) : 33;
    if (have_cand_ok && basic_split_code(a.O.code) && bs > 0 && dim >= bs && dim <= kGroupMaxDim) return 4;
    return 0;
}

constexpr int kCecFmaMaxDim = 32;  // the fused FMA rotation beats the DMMA split up to here (device loop)

int launch_update(bool sel_mode, const UpdArgs& A0, cudaStream_t st, uint8_t* cand_ok = nullptr,
                  cudaEvent_t mid_event = nullptr, unsigned* tile_counter = nullptr, bool scripted = false) {
    UpdArgs a = A0;
    const int dim = a.P.dim;
    if ((a.O.flags & APO_OBJ_FMA_SMALL_D) && dim <= kCecFmaMaxDim) a.O.cec.rot_pad = nullptr;  // FMA rotation
    const bool group = dim <= kGroupMaxDim;
    const int fn_id = a.O.code - APO_OBJ_CEC2022_BASE;
    const bool split = group && cand_ok && a.O.code > APO_OBJ_CEC2022_BASE && dim <= kCecEvalMaxDim &&
                       a.O.cec.rot_pad != nullptr;
    // D > 104: candidates, then the rotation of every candidate as one DMMA GEMM (apo_cec_gemm.cu)
    const bool gemm = !split && cand_ok && a.O.code > APO_OBJ_CEC2022_BASE && dim > kCecEvalMaxDim &&
                      a.O.cec.rot_gemm != nullptr && (fn_id <= 8 || fn_id == 10);
    // the reference's objectives at D > 32: candidates, then lane-per-protozoon evaluation (k_basic_eval)
    const bool bsplit = group && cand_ok && update_path(sel_mode, a, true, true) == 4;
    if (split || gemm || bsplit) {
        a.cand_ok = cand_ok;
        a.cec_bufs = 0;
    }
    // SEL rows (device loop): candidates, DMMA evaluation and select as one kernel (apo_update_fused.cu)
    const int path = split ? update_path(sel_mode, a, true, tile_counter != nullptr) : 0;
    if (path == 2) {
        if (a.rank_hi <= 0) a.rank_hi = a.P.ps;
        APO_CUDA(launch_update_cec_fused(a, st, tile_counter, smem_optin(), num_sms()));
        if (mid_event) APO_CUDA(cudaEventRecord(mid_event, st));
        return APO_OK;
    }
    int w = group ? kWarps : warps_for_dim(dim);
    const bool stage = sel_mode && dim <= APO_STAGE_MAX_DIM;
    const size_t per_warp = group ? group_scratch_bytes(dim, stage, a.cec_bufs) : warp_scratch_bytes(dim);
    while (w > 1 && per_warp * (size_t)w + 1024 > (size_t)smem_optin()) w--;  // e.g. fused CEC at D ~ 150-256
    const size_t smem = per_warp * (size_t)w;
    const bool cec = a.O.code > APO_OBJ_CEC2022_BASE;
    // the keyed builds carry no Philox call site; Philox runs (device loop, shards) take their own build
    const bool co = split || gemm || bsplit;
    const bool philox = a.P.rng == RNG_PHILOX;
    const bool many = a.P.npairs > 1;
    const void* fn = scripted ? pick_update_scripted(dim, co, cec, many)
                     : philox ? (sel_mode ? apo_philox::pick_update_sel(dim, co, cec, many)
                                          : apo_philox::pick_update_dense(dim, co, cec, many))
                              : (sel_mode ? pick_update_sel(dim, co, cec, many) : pick_update_dense(dim, co, cec, many));
    if (int rc = set_smem(fn, smem)) return rc;
    int per_sm = 1;
    if (int rc = occupancy(&per_sm, fn, 32 * w, smem)) return rc;
    if (per_sm < 1) per_sm = 1;
    if (a.rank_hi <= 0) a.rank_hi = a.P.ps;  // default: every rank
    const long long cap = (long long)per_sm * num_sms();
    if (group) {
        // 32 ranks per warp, or fewer when that leaves warp slots empty: a small population is
        // latency-bound and each warp walks its group's ranks partly in sequence
        const long long ranks = a.rank_hi - a.rank_lo, slots = cap * w;
        static const int env_g = getenv("APO_GROUP_SIZE") ? atoi(getenv("APO_GROUP_SIZE")) : 0;
        long long G = env_g > 0 ? env_g : (ranks + slots - 1) / slots;
        a.gsize = (int)(G < 1 ? 1 : G > 32 ? 32 : G);
    }
    const long long units = group ? ((long long)(a.rank_hi - a.rank_lo) + a.gsize - 1) / a.gsize
                                  : (long long)(a.rank_hi - a.rank_lo);
    const long long need = (units + w - 1) / w;
    const int grid = (int)(need < cap ? need : cap);
    {
        void* args[] = {(void*)&a};
        APO_CUDA(cudaLaunchKernel(fn, dim3(grid), dim3(32 * w), args, smem, st));
    }
    if (mid_event) APO_CUDA(cudaEventRecord(mid_event, st));
    if (bsplit) {
        BasicEvalArgs B{};
        B.n_rows = a.rank_hi - a.rank_lo;
        B.row0 = a.rank_lo;
        B.dim = dim;
        B.ld = a.P.ld;
        B.order = sel_mode ? nullptr : a.order;
        B.O = a.O;
        B.pos0 = a.pos0;
        B.pos1 = a.pos1;
        B.sel = a.sel;
        B.sel_next = a.sel_next;
        B.pos = a.pos;
        B.out_pos = a.out_pos;
        B.out_acc = a.out_acc;
        B.out_warn = a.out_warn;
        B.fit = a.fit;
        B.out_fit = a.out_fit;
        B.cand_ok = cand_ok;
        B.warn_count = a.warn_count;
        B.trace_key = a.trace_key;
        // even row strides: each lane streams its row with 16-byte loads (APO_BASIC_EVAL=1 forces the
        // staged form); odd strides: 32 x 32 blocks through cp.async, double-buffered.  (Whole rows by
        // TMA measured slower: the fold of one group cannot overlap the copy of the next.)
        static const int env_be = getenv("APO_BASIC_EVAL") ? atoi(getenv("APO_BASIC_EVAL")) : 0;
        const bool direct = (B.ld % 2) == 0 && env_be != 1;
        const void* fb = direct ? (sel_mode ? (const void*)k_basic_eval_direct<true> : (const void*)k_basic_eval_direct<false>)
                                : (sel_mode ? (const void*)k_basic_eval<true> : (const void*)k_basic_eval<false>);
        const int bw = direct ? kBasicDirectWarps : kBasicEvalWarps;
        const size_t bsmem = direct ? 0 : kBasicEvalSmem;
        if (int rc = set_smem(fb, bsmem)) return rc;
        int bper = 1;
        if (int rc = occupancy(&bper, fb, 32 * bw, bsmem)) return rc;
        if (bper < 1) bper = 1;
        const long long groups = ((long long)B.n_rows + 31) / 32;
        const long long bneed = (groups + bw - 1) / bw;
        const long long bcap = (long long)bper * num_sms();
        void* bargs[] = {(void*)&B};
        APO_CUDA(cudaLaunchKernel(fb, dim3((unsigned)(bneed < bcap ? bneed : bcap)), dim3(32 * bw), bargs, bsmem, st));
        return APO_OK;
    }
    if (gemm) {
        CecGemmArgs G{};
        G.row0 = a.rank_lo;
        G.n_rows = a.rank_hi - a.rank_lo;
        G.dim = dim;
        G.ld = a.P.ld;
        G.kp = gemm_kp(dim);
        G.np = gemm_np(dim);
        G.comp = fn_id == 10 ? 1 : 0;  // F10: the one rotated component (kCecSpec rflag {0, 1, 0})
        G.O = a.O;
        G.pos0 = a.pos0;
        G.pos1 = a.pos1;
        G.sel = sel_mode ? a.sel : nullptr;
        G.sel_next = a.sel_next;
        G.pos = a.pos;
        G.out_pos = a.out_pos;
        G.order = sel_mode ? nullptr : a.order;
        G.out_acc = a.out_acc;
        G.out_warn = a.out_warn;
        G.fit = a.fit;
        G.out_fit = a.out_fit;
        G.cand_ok = cand_ok;
        G.warn_count = a.warn_count;
        G.trace_key = a.trace_key;
        const int rc = cec_gemm_finish(G, st, num_sms());
        if (rc) return fail(APO_ECUDA, "cec_gemm_finish failed");
        return APO_OK;
    }
    if (!split) return APO_OK;
    return launch_cec_eval(sel_mode, a, st, cand_ok, tile_counter, 0);
}

// k_cec_eval over ranks [rank_lo, rank_hi) of an update (init = 0) or over every slot of pos0 at
// iteration 0 (init = 1).
int launch_cec_eval(bool sel_mode, const UpdArgs& a, cudaStream_t st, uint8_t* cand_ok, unsigned* tile_counter,
                    int init) {
    const int dim = a.P.dim;
    const int fn_id = a.O.code - APO_OBJ_CEC2022_BASE;
    CecEvalArgs E{};
    E.init = init;
    E.row0 = a.rank_lo;
    E.n_rows = a.rank_hi - a.rank_lo;
    E.order = sel_mode ? nullptr : a.order;
    E.dim = dim;
    E.ld = a.P.ld;
    E.O = a.O;
    E.bufs = 0;  // hybrids permute inside rot_pad, compositions re-read the candidate per component
    static const int kNcomp[12] = {1, 1, 1, 1, 1, 1, 1, 1, 5, 3, 5, 6};
    static const int kFirstRot[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 1, 0, 0};  // first rflag = 1 (apo_cec.cuh kCecSpec)
    E.ncomp = kNcomp[fn_id - 1];
    E.bsm_comp = kFirstRot[fn_id - 1];
    E.pos0 = a.pos0;
    E.pos1 = a.pos1;
    E.sel = a.sel;
    E.sel_next = a.sel_next;
    E.pos = a.pos;
    E.out_pos = a.out_pos;
    E.out_acc = a.out_acc;
    E.out_warn = a.out_warn;
    E.fit = a.fit;
    E.out_fit = a.out_fit;
    E.cand_ok = cand_ok;
    E.warn_count = a.warn_count;
    E.trace_key = a.trace_key;
    // the (first) rotation + shift vectors staged in SMEM per CTA, as many warps as fit (<= 16, a
    // multiple of 4), X double-buffered only if that does not cost warps; further composition
    // rotations are read through L1
    const bool fast = true;
    const void* fe = pick_cec_eval(sel_mode, dim, fast);
    int ewarps = kWarps;
    E.prefetch = 0;
    size_t esmem = cec_eval_warp_bytes(dim, E.bufs, false) * kWarps;
    if (fast) {
        int dev = 0, optin = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess)
            optin = 227 * 1024;
        static const int env_pf = getenv("APO_CEC_PREFETCH") ? atoi(getenv("APO_CEC_PREFETCH")) : -1;
        const size_t bsm = cec_bsm_bytes(dim, cec_nt(dim), E.ncomp);
        auto fit_warps = [&](bool pf) {
            int w = (int)(((size_t)optin - bsm) / cec_eval_warp_bytes(dim, E.bufs, pf));
            if (w > 16) w = 16;
            if (w >= 4) w &= ~3;  // equal warps per SM sub-partition (they share its DMMA pipe)
            return w;
        };
        // prefetch (double-buffered X) unless dropping it buys more warps per SM
        E.prefetch = env_pf >= 0 ? env_pf : (fit_warps(false) > fit_warps(true) ? 0 : 1);
        ewarps = fit_warps(E.prefetch != 0);
        APO_CHECK(ewarps >= 1, "k_cec_eval: dim too large for the shared-memory rotation");
        esmem = bsm + cec_eval_warp_bytes(dim, E.bufs, E.prefetch != 0) * (size_t)ewarps;
    }
    if (int rc = set_smem(fe, esmem)) return rc;
    int eper = 1;
    if (int rc = occupancy(&eper, fe, 32 * ewarps, esmem)) return rc;
    if (eper < 1) eper = 1;
    const long long tiles = ((long long)E.n_rows + kCecRows - 1) / kCecRows;
    const long long eneed = (tiles + ewarps - 1) / ewarps;
    const long long ecap = (long long)eper * num_sms();
    APO_CHECK(tile_counter != nullptr, "k_cec_eval needs a tile counter");
    E.tile_counter = tile_counter;
    APO_CUDA(cudaMemsetAsync(tile_counter, 0, sizeof(unsigned), st));
    void* eargs[] = {(void*)&E};
    APO_CUDA(cudaLaunchKernel(fe, dim3((unsigned)(eneed < ecap ? eneed : ecap)), dim3(32 * ewarps), eargs, esmem, st));
    return APO_OK;
}

int grid_for(long long n, int threads) {
    long long g = (n + threads - 1) / threads;
    long long cap = 16LL * num_sms();
    if (g < 1) g = 1;
    return (int)(g < cap ? g : cap);
}

int nbits_for(long long n) {
    int b = 1;
    while ((1LL << b) < n) b++;
    return b;
}

uint64_t coord_count(int rng, uint64_t seed, uint64_t key_iteration, int64_t ps, double pf_max) {
    const Key cbase = stream_key(rng, seed, key_iteration, kCoordinator);
    const double pf = pf_max * uniform(cbase, 0);
    return (uint64_t)ceil((double)ps * pf);
}

// Coordinator Dr on device given scratch (keys + sorted keys + CUB temp).
int dr_device(int rng, uint64_t seed, uint64_t key_iteration, int64_t ps, int64_t count, unsigned long long* keys,
              unsigned long long* keys_sorted, void* tmp, size_t tmp_bytes, unsigned* bits, uint8_t* bytes,
              cudaStream_t st) {
    if (bits) APO_CUDA(cudaMemsetAsync(bits, 0, 4 * (size_t)((ps + 31) / 32), st));
    if (bytes) APO_CUDA(cudaMemsetAsync(bytes, 0, (size_t)ps, st));
    if (count <= 0) return APO_OK;
    const Key cbase = stream_key(rng, seed, key_iteration, kCoordinator);
    k_dr_draw<<<grid_for(count, 256), 256, 0, st>>>((int)count, (int)ps, cbase, keys);
    APO_CUDA(cudaGetLastError());
    size_t bytes_needed = tmp_bytes;
    // only the target bits: the step half is already in step order and the radix sort is stable
    APO_CUDA(cub::DeviceRadixSort::SortKeys(tmp, bytes_needed, keys, keys_sorted, (int)count, 32,
                                            32 + nbits_for(ps), st));
    k_dr_resolve<<<grid_for(count, 256), 256, 0, st>>>((int)count, (int)ps, cbase, keys_sorted, bits, bytes);
    APO_CUDA(cudaGetLastError());
    return APO_OK;
}


// Shared-memory extras of a batch: CEC2022 scratch rows (one X tile when the quad evaluator can
// run -- rot_pad present, dim <= 104 -- else the fallback's 2-3 buffers) and threshold tables.
void batch_smem_needs(const apo_objective* objs, int64_t n, int64_t dim, int* cec_bufs, int* tab_smem) {
    *cec_bufs = 0;
    *tab_smem = 0;
    for (int64_t k = 0; k < n; k++) {
        int cb = cec_bufs_for(objs[k].code);
        if (cb > 0 && objs[k].rot_pad && dim <= kCecQuadMaxDim) cb = 1;
        if (cb > *cec_bufs) *cec_bufs = cb;
        if (objs[k].code == APO_OBJ_OTSU_ML || objs[k].code == APO_OBJ_KAPUR_ML) *tab_smem = APO_THRESHOLD_TABLE_LEN;
    }
}

size_t dr_tmp_bytes(int64_t cap, int64_t ps) {
    size_t b = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, b, (unsigned long long*)nullptr, (unsigned long long*)nullptr,
                                   (int)(cap > 0 ? cap : 1), 32, 32 + nbits_for(ps));
    return b;
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================

struct apo_run {
    int64_t ps, dim, ld, T;
    int rng;  // RngMode
    uint64_t seed;
    int64_t npairs;
    double pf_max, lower, upper, eps;
    ObjDesc obj;
    cudaStream_t stream;
    double* pos[2];  // two row buffers; sel[cur][slot] picks the current one
    uint8_t* sel[2];
    double* fit[2];
    int cur;
    int* order;
    unsigned long long* keys_in;
    unsigned long long* keys_out;
    int* vals_in;
    unsigned long long* dr_keys;
    unsigned long long* dr_sorted;
    unsigned* dr_bits;
    int64_t dr_cap;
    void* tmp;
    size_t tmp_bytes;
    double* p_dr;
    uint8_t* cand_ok;  // CEC2022 split update: per-slot candidate finiteness
    unsigned* tile_counter;
    std::vector<double> sched;
    unsigned long long* trace_keys;  // [T+1]
    unsigned long long* warn;
    int64_t iters;
    bool initialized;
    // optional CUDA-event timing of the fused update launch (bench.py roofline)
    bool profile;
    std::vector<cudaEvent_t> prof_events;
    // the coordinator's Dr draws (their own sort) run on a side stream beside the fitness sort
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    void* dr_tmp = nullptr;
    size_t dr_tmp_bytes = 0;
};

extern "C" {

int64_t apo_max_dim(void) { return max_dim_supported(); }

int apo_abi_version(void) { return 4; }  // 4: scripted draws; 3: apo_objective.flags, apo_run_updates_ordered; 2: rng, shard/load/threshold

const char* apo_last_error(void) { return g_err.c_str(); }

int apo_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

int apo_run_updates_obj(const double* positions, const double* fitness, const uint8_t* in_dr, double* out_pos,
                        double* out_fit, uint8_t* out_acc, uint8_t* out_warn, int64_t ps, int64_t dim, uint64_t seed,
                        uint64_t key_iteration, int64_t npairs, double lower, double upper, double eps, double p_ah,
                        double f_mult, double decay, const apo_objective* objective_host, const double* p_dr,
                        unsigned long long* warn_count, void* stream) {
    if (warn_count) APO_CUDA(cudaMemsetAsync(warn_count, 0, sizeof(unsigned long long), as_stream(stream)));
    return apo_run_updates_range(positions, fitness, in_dr, out_pos, out_fit, out_acc, out_warn, ps, dim, seed,
                                 key_iteration, npairs, lower, upper, eps, p_ah, f_mult, decay, objective_host, p_dr,
                                 warn_count, 0, ps, stream);
}

namespace {
int updates_range(const double* positions, const double* fitness, const int32_t* order, const uint8_t* in_dr,
                  double* out_pos, double* out_fit, uint8_t* out_acc, uint8_t* out_warn, int64_t ps, int64_t dim,
                  uint64_t seed, uint64_t key_iteration, int64_t npairs, double lower, double upper, double eps,
                  double p_ah, double f_mult, double decay, const apo_objective* objective_host, const double* p_dr,
                  unsigned long long* warn_count, int64_t rank_lo, int64_t rank_hi, void* stream,
                  int rng = RNG_KEYED);
}

int apo_run_updates_range(const double* positions, const double* fitness, const uint8_t* in_dr, double* out_pos,
                          double* out_fit, uint8_t* out_acc, uint8_t* out_warn, int64_t ps, int64_t dim,
                          uint64_t seed, uint64_t key_iteration, int64_t npairs, double lower, double upper,
                          double eps, double p_ah, double f_mult, double decay, const apo_objective* objective_host,
                          const double* p_dr, unsigned long long* warn_count, int64_t rank_lo, int64_t rank_hi,
                          void* stream) {
    return updates_range(positions, fitness, nullptr, in_dr, out_pos, out_fit, out_acc, out_warn, ps, dim, seed,
                         key_iteration, npairs, lower, upper, eps, p_ah, f_mult, decay, objective_host, p_dr,
                         warn_count, rank_lo, rank_hi, stream);
}

int apo_run_updates_ordered(const double* positions, const double* fitness, const int32_t* order,
                            const uint8_t* in_dr, double* out_pos, double* out_fit, uint8_t* out_acc,
                            uint8_t* out_warn, int64_t ps, int64_t dim, uint64_t seed, uint64_t key_iteration,
                            int64_t npairs, double lower, double upper, double eps, double p_ah, double f_mult,
                            double decay, const apo_objective* objective_host, const double* p_dr,
                            unsigned long long* warn_count, int64_t rank_lo, int64_t rank_hi, void* stream) {
    APO_CHECK(order != nullptr, "order is NULL");
    APO_CHECK(dim <= kGroupMaxDim, "apo_run_updates_ordered: dim > 256 (gather the snapshot, use _range)");
    return updates_range(positions, fitness, order, in_dr, out_pos, out_fit, out_acc, out_warn, ps, dim, seed,
                         key_iteration, npairs, lower, upper, eps, p_ah, f_mult, decay, objective_host, p_dr,
                         warn_count, rank_lo, rank_hi, stream);
}

namespace {
int updates_range(const double* positions, const double* fitness, const int32_t* order, const uint8_t* in_dr,
                  double* out_pos, double* out_fit, uint8_t* out_acc, uint8_t* out_warn, int64_t ps, int64_t dim,
                  uint64_t seed, uint64_t key_iteration, int64_t npairs, double lower, double upper, double eps,
                  double p_ah, double f_mult, double decay, const apo_objective* objective_host, const double* p_dr,
                  unsigned long long* warn_count, int64_t rank_lo, int64_t rank_hi, void* stream, int rng) {
    APO_CHECK(ps >= 1 && ps < (1LL << 31), "ps out of range");
    APO_CHECK(0 <= rank_lo && rank_lo < rank_hi && rank_hi <= ps, "rank range must satisfy 0 <= lo < hi <= ps");
    APO_CHECK(dim >= 1 && dim <= max_dim_supported(), "dim out of range (1..apo_max_dim())");
    APO_CHECK(npairs >= 1, "npairs must be >= 1");
    APO_CHECK(positions && fitness && in_dr && out_pos && out_fit && p_dr, "NULL buffer");
    APO_CHECK(out_pos != positions && out_fit != fitness, "outputs must not alias inputs");
    if (int rc = check_objective(objective_host, dim)) return rc;
    IterParams P;
    P.seed = seed;
    P.key_iteration = key_iteration;
    P.ps = (int)ps;
    P.dim = (int)dim;
    P.npairs = (int)npairs;
    P.ld = (int)dim;
    P.lower = lower;
    P.upper = upper;
    P.span = upper - lower;
    P.eps = eps;
    P.p_ah = p_ah;
    P.f_mult = f_mult;
    P.decay = decay;
    P.rng = rng;  // the reference-facing boundary: the keyed stream, or scripted draws (RNG_TABLE)
    if (rng == RNG_KEYED) set_iteration_base(P);
    else P.has_base_it = 0;
    UpdArgs A{};
    A.P = P;
    A.rank_lo = (int)rank_lo;
    A.rank_hi = (int)rank_hi;
    A.O = to_desc(objective_host);
    A.pos = positions;
    A.out_pos = out_pos;
    A.fit = fitness;
    A.out_fit = out_fit;
    A.in_dr_bytes = in_dr;
    A.p_dr = p_dr;
    A.out_acc = out_acc;
    A.out_warn = out_warn;
    A.warn_count = warn_count;
    A.order = order;  // rows of positions/fitness read at order[rank]; outputs by rank
    A.cec_bufs = cec_bufs_for(A.O.code);
    uint8_t* cand_ok = nullptr;
    // CEC2022 and the split basic objectives need the per-row candidate finiteness scratch
    const bool cec = A.O.code > APO_OBJ_CEC2022_BASE || basic_split_code(A.O.code);
    const size_t ok_bytes = ((size_t)ps + 15) & ~(size_t)15;  // cand_ok, then the k_cec_eval tile counter
    if (cec) APO_CUDA(cudaMallocAsync((void**)&cand_ok, ok_bytes + 16, as_stream(stream)));
    unsigned* counter = cec ? reinterpret_cast<unsigned*>(cand_ok + ok_bytes) : nullptr;
    const int rc = launch_update(false, A, as_stream(stream), cand_ok, nullptr, counter, rng == RNG_TABLE);
    if (cec) cudaFreeAsync(cand_ok, as_stream(stream));
    return rc;
}
}  // namespace

int apo_run_updates_scripted(const double* positions, const double* fitness, const uint8_t* in_dr, double* out_pos,
                             double* out_fit, uint8_t* out_acc, uint8_t* out_warn, int64_t ps, int64_t dim,
                             const apo_draw_table* table, int64_t npairs, double lower, double upper, double eps,
                             double p_ah, double f_mult, double decay, const apo_objective* objective_host,
                             const double* p_dr, unsigned long long* warn_count, void* stream) {
    APO_CHECK(table != nullptr, "table is NULL");
    if (warn_count) APO_CUDA(cudaMemsetAsync(warn_count, 0, sizeof(unsigned long long), as_stream(stream)));
    return updates_range(positions, fitness, nullptr, in_dr, out_pos, out_fit, out_acc, out_warn, ps, dim,
                         (uint64_t)(uintptr_t)table, 0, npairs, lower, upper, eps, p_ah, f_mult, decay,
                         objective_host, p_dr, warn_count, 0, ps, stream, RNG_TABLE);
}

int apo_run_updates(const double* positions, const double* fitness, const uint8_t* in_dr, double* out_pos,
                    double* out_fit, uint8_t* out_acc, uint8_t* out_warn, int64_t ps, int64_t dim, uint64_t seed,
                    uint64_t key_iteration, int64_t npairs, double lower, double upper, double span, double eps,
                    double p_ah, double f_mult, double decay, int64_t code, const double* table, int64_t table_len,
                    const double* p_dr, unsigned long long* warn_count, void* stream) {
    APO_CHECK(span == upper - lower, "span must equal upper - lower");
    apo_objective o{};
    o.code = (int32_t)code;
    o.table_len = (int32_t)table_len;
    o.table = table;
    return apo_run_updates_obj(positions, fitness, in_dr, out_pos, out_fit, out_acc, out_warn, ps, dim, seed,
                               key_iteration, npairs, lower, upper, eps, p_ah, f_mult, decay, &o, p_dr, warn_count,
                               stream);
}

int apo_evaluate(const double* x, int64_t n, int64_t dim, int64_t ld, const apo_objective* objective_host, double* out,
                 void* stream) {
    APO_CHECK(n >= 0 && dim >= 1 && dim <= max_dim_supported() && ld >= dim, "bad shape (dim > apo_max_dim()?)");
    if (int rc = check_objective(objective_host, dim)) return rc;
    if (n == 0) return APO_OK;
    const int w = warps_for_dim(dim);
    const size_t smem = warp_scratch_bytes((int)dim) * (size_t)w;
    if (int rc = set_smem((const void*)k_evaluate, smem)) return rc;
    const long long need = (n + w - 1) / w;
    const long long cap = 8LL * num_sms();
    k_evaluate<<<(int)(need < cap ? need : cap), 32 * w, smem, as_stream(stream)>>>(x, (int)n, (int)dim, (int)ld,
                                                                                  to_desc(objective_host), out);
    APO_CUDA(cudaGetLastError());
    return APO_OK;
}

int apo_initialize(uint64_t seed, int64_t ps, int64_t dim, int64_t ld, double lower, double span,
                   const apo_objective* objective_host, double* positions, double* fitness, void* stream) {
    APO_CHECK(ps >= 1 && ps < (1LL << 31) && dim >= 1 && dim <= max_dim_supported() && ld >= dim,
              "bad shape (dim > apo_max_dim()?)");
    APO_CHECK(positions && fitness, "NULL buffer");
    if (int rc = check_objective(objective_host, dim)) return rc;
    const int w = warps_for_dim(dim);
    const size_t smem = warp_scratch_bytes((int)dim) * (size_t)w;
    if (int rc = set_smem((const void*)k_init, smem)) return rc;
    const long long need = (ps + w - 1) / w;
    const long long cap = 8LL * num_sms();
    const ObjDesc O = to_desc(objective_host);
    // CEC2022 with DMMA tables: the same evaluator as the device loop's iteration 0 (k_cec_eval, init mode)
    const bool cec_fast = O.code > APO_OBJ_CEC2022_BASE && dim <= kCecEvalMaxDim && O.cec.rot_pad;
    k_init<<<(int)(need < cap ? need : cap), 32 * w, smem, as_stream(stream)>>>(
        RNG_KEYED, seed, (int)ps, (int)dim, (int)ld, lower, span, O, positions, cec_fast ? nullptr : fitness, nullptr);
    APO_CUDA(cudaGetLastError());
    if (cec_fast) {
        unsigned* counter = nullptr;
        APO_CUDA(cudaMallocAsync((void**)&counter, 16, as_stream(stream)));
        UpdArgs A{};
        A.P.ps = (int)ps;
        A.P.dim = (int)dim;
        A.P.ld = (int)ld;
        A.O = O;
        A.pos0 = positions;
        A.pos1 = positions;
        A.out_fit = fitness;
        A.rank_lo = 0;
        A.rank_hi = (int)ps;
        const int rc = launch_cec_eval(true, A, as_stream(stream), nullptr, counter, 1);
        cudaFreeAsync(counter, as_stream(stream));
        if (rc) return rc;
    }
    return APO_OK;
}

int apo_sort_order(const double* fitness, int64_t n, int32_t* order, void* stream) {
    APO_CHECK(n >= 0 && n < (1LL << 31), "n out of range");
    if (n == 0) return APO_OK;
    cudaStream_t st = as_stream(stream);
    unsigned long long *k_in = nullptr, *k_out = nullptr;
    int* v_in = nullptr;
    void* tmp = nullptr;
    size_t tb = 0;
    APO_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, k_in, k_out, v_in, (int*)order, (int)n, 0, 64, st));
    APO_CUDA(cudaMallocAsync((void**)&k_in, 8 * (size_t)n, st));
    APO_CUDA(cudaMallocAsync((void**)&k_out, 8 * (size_t)n, st));
    APO_CUDA(cudaMallocAsync((void**)&v_in, 4 * (size_t)n, st));
    APO_CUDA(cudaMallocAsync(&tmp, tb, st));
    k_make_keys<<<grid_for(n, 256), 256, 0, st>>>((int)n, fitness, nullptr, k_in, v_in);
    APO_CUDA(cudaGetLastError());
    APO_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, k_in, k_out, v_in, (int*)order, (int)n, 0, 64, st));
    cudaFreeAsync(k_in, st);
    cudaFreeAsync(k_out, st);
    cudaFreeAsync(v_in, st);
    cudaFreeAsync(tmp, st);
    return APO_OK;
}

int apo_select_dr(uint64_t seed, uint64_t key_iteration, int64_t ps, double pf_max, uint8_t* in_dr,
                  int64_t* count_host, void* stream) {
    APO_CHECK(ps >= 1 && ps < (1LL << 31) && in_dr, "bad arguments");
    APO_CHECK(pf_max > 0.0 && pf_max <= 1.0, "pf_max must be in (0, 1]");
    cudaStream_t st = as_stream(stream);
    const int64_t count = (int64_t)coord_count(RNG_KEYED, seed, key_iteration, ps, pf_max);
    if (count_host) *count_host = count;
    unsigned long long *keys = nullptr, *sorted = nullptr;
    void* tmp = nullptr;
    size_t tb = dr_tmp_bytes(count, ps);
    if (count > 0) {
        APO_CUDA(cudaMallocAsync((void**)&keys, 8 * (size_t)count, st));
        APO_CUDA(cudaMallocAsync((void**)&sorted, 8 * (size_t)count, st));
        APO_CUDA(cudaMallocAsync(&tmp, tb, st));
    }
    int rc = dr_device(RNG_KEYED, seed, key_iteration, ps, count, keys, sorted, tmp, tb, nullptr, in_dr, st);
    if (count > 0) {
        cudaFreeAsync(keys, st);
        cudaFreeAsync(sorted, st);
        cudaFreeAsync(tmp, st);
    }
    return rc;
}

int apo_select_dr_scripted(const apo_draw_table* table, int64_t ps, int64_t count, uint8_t* in_dr, void* stream) {
    APO_CHECK(table && in_dr && ps >= 1 && ps < (1LL << 31), "bad arguments");
    APO_CHECK(count >= 0 && count <= ps, "count must be in [0, ps]");
    cudaStream_t st = as_stream(stream);
    int* perm = nullptr;
    APO_CUDA(cudaMallocAsync((void**)&perm, 4 * (size_t)ps, st));
    APO_CUDA(launch_dr_scripted((uint64_t)(uintptr_t)table, (int)ps, (int)count, perm, in_dr, st));
    cudaFreeAsync(perm, st);
    return APO_OK;
}

int apo_histogram_u8(const uint8_t* pixels, int64_t n, int64_t* counts, void* stream) {
    APO_CHECK(n >= 0 && counts && (n == 0 || pixels), "bad arguments");
    APO_CHECK(((uintptr_t)pixels & 15) == 0, "pixels must be 16-byte aligned");
    cudaStream_t st = as_stream(stream);
    APO_CUDA(cudaMemsetAsync(counts, 0, 256 * sizeof(int64_t), st));
    if (n == 0) return APO_OK;
    long long g = (n / 16 + kThreads - 1) / kThreads;
    const long long cap = 4LL * num_sms();
    if (g < 1) g = 1;
    k_histogram_u8<<<(int)(g < cap ? g : cap), kThreads, 0, st>>>(pixels, n, (unsigned long long*)counts);
    APO_CUDA(cudaGetLastError());
    return APO_OK;
}

int apo_threshold_tables(const int64_t* counts, int method, double* table, void* stream) {
    APO_CHECK(counts && table && (method == 0 || method == 1), "bad arguments");
    k_threshold_tables<<<1, 32, 0, as_stream(stream)>>>((const long long*)counts, method, table);
    APO_CUDA(cudaGetLastError());
    return APO_OK;
}

void apo_philox4x32_10(const uint32_t* ctr4, const uint32_t* key2, uint32_t* out4) {
    uint32_t c[4] = {ctr4[0], ctr4[1], ctr4[2], ctr4[3]};
    philox4x32_10_block(c, key2[0], key2[1]);
    for (int k = 0; k < 4; k++) out4[k] = c[k];
}

double apo_rng_uniform(int rng, uint64_t seed, uint64_t iteration, uint64_t individual, uint64_t counter) {
    const Key k = stream_key(rng, seed, iteration, individual);
    if (rng == RNG_PHILOX) return philox_draw(k.a, k.b, k.c, counter);  // any iteration, kTableMark included
    if (rng == RNG_TABLE) return NAN;                                    // the table lives in device memory
    return uniform(k, counter);
}

int apo_debug_cos(const double* x, double* out, int64_t n, void* stream) {
    APO_CHECK(n >= 0, "bad n");
    if (n == 0) return APO_OK;
    k_debug_cos<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(x, out, n);
    APO_CUDA(cudaGetLastError());
    return APO_OK;
}

int apo_debug_exp(const double* x, double* out, int64_t n, void* stream) {
    APO_CHECK(n >= 0, "bad n");
    if (n == 0) return APO_OK;
    k_debug_exp<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(x, out, n);
    APO_CUDA(cudaGetLastError());
    return APO_OK;
}

int apo_debug_cec_basic(int basic, const double* z, int64_t rows, int64_t n, const double* ew, double* out,
                        int variant, void* stream) {
    APO_CHECK(basic >= 0 && basic <= 16 && rows >= 0 && n >= 1 && (variant == 0 || variant == 1), "bad arguments");
    if (rows == 0) return APO_OK;
    APO_CUDA(launch_debug_cec_basic(basic, z, rows, (int)n, ew, out, variant, as_stream(stream)));
    return APO_OK;
}

// --------------------------- device-resident run ---------------------------

int apo_run_create(apo_run** out, int64_t ps, int64_t dim, int64_t max_iterations, uint64_t seed, int64_t npairs,
                   double pf_max, double lower, double upper, double eps, const apo_objective* objective_host,
                   const double* sched_host, const double* p_dr_host, int rng, void* stream) {
    APO_CHECK(rng == RNG_KEYED || rng == RNG_PHILOX, "rng must be APO_RNG_KEYED or APO_RNG_PHILOX");
    APO_CHECK(out != nullptr, "out is NULL");
    APO_CHECK(ps >= 1 && ps < (1LL << 31) && dim >= 1 && dim <= max_dim_supported(), "bad shape (dim > apo_max_dim()?)");
    APO_CHECK(max_iterations >= 0 && npairs >= 1 && pf_max > 0.0 && pf_max <= 1.0, "bad config");
    APO_CHECK(max_iterations == 0 || sched_host, "sched_host is NULL");
    APO_CHECK(p_dr_host, "p_dr_host is NULL");
    if (int rc = check_objective(objective_host, dim)) return rc;
    apo_run* r = new apo_run();
    r->ps = ps;
    r->dim = dim;
    r->rng = rng;
    r->ld = (dim + 1) & ~1LL;  // 16-byte aligned rows
    r->T = max_iterations;
    r->seed = seed;
    r->npairs = npairs;
    r->pf_max = pf_max;
    r->lower = lower;
    r->upper = upper;
    r->eps = eps;
    r->obj = to_desc(objective_host);
    r->stream = as_stream(stream);
    r->cur = 0;
    r->iters = 0;
    r->initialized = false;
    r->profile = false;
    r->sched.assign(sched_host, sched_host + 3 * max_iterations);
    r->dr_cap = (int64_t)ceil((double)ps * pf_max) + 1;
    const size_t rows = 8 * (size_t)ps * (size_t)r->ld;
    cudaStream_t st = r->stream;
    size_t tb_sort = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb_sort, (unsigned long long*)nullptr, (unsigned long long*)nullptr,
                                    (int*)nullptr, (int*)nullptr, (int)ps, 0, 64, st);
    const size_t tb_dr = dr_tmp_bytes(r->dr_cap, ps);
    r->tmp_bytes = tb_sort > tb_dr ? tb_sort : tb_dr;
    cudaError_t e = cudaSuccess;
    // stream-ordered allocations: the pool keeps them after apo_run_destroy (keep_mempool), so creating
    // and destroying runs costs no cudaMalloc/cudaFree (hundreds of ms at the C4 shape)
    auto alloc = [&](void** p, size_t b) {
        if (e == cudaSuccess) e = cudaMallocAsync(p, b > 0 ? b : 16, st);
    };
    alloc((void**)&r->pos[0], rows);
    alloc((void**)&r->pos[1], rows);
    alloc((void**)&r->sel[0], (size_t)ps);
    alloc((void**)&r->sel[1], (size_t)ps);
    alloc((void**)&r->fit[0], 8 * (size_t)ps);
    alloc((void**)&r->fit[1], 8 * (size_t)ps);
    alloc((void**)&r->order, 4 * (size_t)ps);
    alloc((void**)&r->keys_in, 8 * (size_t)ps);
    alloc((void**)&r->keys_out, 8 * (size_t)ps);
    alloc((void**)&r->vals_in, 4 * (size_t)ps);
    alloc((void**)&r->dr_keys, 8 * (size_t)r->dr_cap);
    alloc((void**)&r->dr_sorted, 8 * (size_t)r->dr_cap);
    alloc((void**)&r->dr_bits, 4 * (size_t)((ps + 31) / 32));
    alloc(&r->tmp, r->tmp_bytes);
    r->dr_tmp_bytes = tb_dr;
    alloc(&r->dr_tmp, r->dr_tmp_bytes);
    alloc((void**)&r->p_dr, 8 * (size_t)ps);
    alloc((void**)&r->cand_ok, (size_t)ps);
    alloc((void**)&r->tile_counter, 16);
    alloc((void**)&r->trace_keys, 8 * (size_t)(max_iterations + 1));
    alloc((void**)&r->warn, 8);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&r->side, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&r->ev_fork, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&r->ev_join, cudaEventDisableTiming);
    if (e != cudaSuccess) {
        apo_run_destroy(r);
        return fail(APO_ENOMEM, std::string("apo_run_create: ") + cudaGetErrorString(e));
    }
    APO_CUDA(cudaMemcpyAsync(r->p_dr, p_dr_host, 8 * (size_t)ps, cudaMemcpyHostToDevice, st));
    APO_CUDA(cudaMemsetAsync(r->trace_keys, 0xFF, 8 * (size_t)(max_iterations + 1), st));
    APO_CUDA(cudaMemsetAsync(r->warn, 0, 8, st));
    *out = r;
    return APO_OK;
}

int apo_run_initialize(apo_run* r) {
    APO_CHECK(r, "run is NULL");
    cudaStream_t st = r->stream;
    const int w = warps_for_dim(r->dim);
    const size_t smem = warp_scratch_bytes((int)r->dim) * (size_t)w;
    if (int rc = set_smem((const void*)k_init, smem)) return rc;
    int per_sm = 1;
    if (int rc = occupancy(&per_sm, (const void*)k_init, 32 * w, smem)) return rc;
    const long long need = (r->ps + w - 1) / w;
    const long long cap = (long long)(per_sm > 0 ? per_sm : 1) * num_sms();
    APO_CUDA(cudaMemsetAsync(r->trace_keys, 0xFF, 8 * (size_t)(r->T + 1), st));
    APO_CUDA(cudaMemsetAsync(r->warn, 0, 8, st));
    // CEC2022 with DMMA tables: k_init draws the rows, k_cec_eval (init mode) evaluates them
    const bool cec_fast = r->obj.code > APO_OBJ_CEC2022_BASE && r->dim <= kCecEvalMaxDim && r->obj.cec.rot_pad;
    k_init<<<(int)(need < cap ? need : cap), 32 * w, smem, st>>>(r->rng, r->seed, (int)r->ps, (int)r->dim, (int)r->ld,
                                                                  r->lower, r->upper - r->lower, r->obj, r->pos[0],
                                                                  cec_fast ? nullptr : r->fit[0], r->trace_keys);
    APO_CUDA(cudaGetLastError());
    if (cec_fast) {
        UpdArgs A{};
        A.P.ps = (int)r->ps;
        A.P.dim = (int)r->dim;
        A.P.ld = (int)r->ld;
        A.O = r->obj;
        A.pos0 = r->pos[0];
        A.pos1 = r->pos[0];
        A.out_fit = r->fit[0];
        A.trace_key = r->trace_keys;
        A.rank_lo = 0;
        A.rank_hi = (int)r->ps;
        if (int rc = launch_cec_eval(true, A, st, r->cand_ok, r->tile_counter, 1)) return rc;
    }
    k_iota<<<grid_for(r->ps, 256), 256, 0, st>>>((int)r->ps, r->order);
    APO_CUDA(cudaGetLastError());
    APO_CUDA(cudaMemsetAsync(r->sel[0], 0, (size_t)r->ps, st));
    r->cur = 0;
    r->iters = 0;
    r->initialized = true;
    return APO_OK;
}

int apo_run_iterate(apo_run* r, int64_t n) {
    APO_CHECK(r && r->initialized, "run not initialised");
    APO_CHECK(n >= 0 && r->iters + n <= r->T, "iteration budget exceeded");
    cudaStream_t st = r->stream;
    const int ps = (int)r->ps;
    static const char* env_small = getenv("APO_SMALL_PROLOGUE");
    const bool small_prologue = prologue_small_fits(ps) && !(env_small && atoi(env_small) == 0);
    for (int64_t k = 0; k < n; k++) {
        const int64_t t = r->iters;
        const uint64_t key_it = (uint64_t)t + 1;
        const int64_t count = (int64_t)coord_count(r->rng, r->seed, key_it, r->ps, r->pf_max);
        if (small_prologue) {
            // 1 + 2 as one launch (apo_prologue.cu); the new order goes to the spare buffer
            APO_CUDA(launch_prologue_small(ps, r->fit[r->cur], r->order, r->vals_in, (int)count,
                                           stream_key(r->rng, r->seed, key_it, kCoordinator), r->dr_bits,
                                           r->keys_in, (int*)r->keys_out, num_sms(), st));
            std::swap(r->order, r->vals_in);
        } else {
            // 2. coordinator draws, forked onto the side stream (they depend only on the keys and on the
            //    previous update having consumed dr_bits, which the fork event orders)
            APO_CUDA(cudaEventRecord(r->ev_fork, st));
            APO_CUDA(cudaStreamWaitEvent(r->side, r->ev_fork, 0));
            if (int rc = dr_device(r->rng, r->seed, key_it, r->ps, count, r->dr_keys, r->dr_sorted, r->dr_tmp,
                                   r->dr_tmp_bytes, r->dr_bits, nullptr, r->side))
                return rc;
            APO_CUDA(cudaEventRecord(r->ev_join, r->side));
            // 1. stable sort by fitness, ties by previous rank (concurrently with 2.)
            k_make_keys<<<grid_for(ps, 256), 256, 0, st>>>(ps, r->fit[r->cur], r->order, r->keys_in, r->vals_in);
            APO_CUDA(cudaGetLastError());
            size_t tb = r->tmp_bytes;
            APO_CUDA(cub::DeviceRadixSort::SortPairs(r->tmp, tb, r->keys_in, r->keys_out, r->vals_in, r->order, ps, 0,
                                                     64, st));
            APO_CUDA(cudaStreamWaitEvent(st, r->ev_join, 0));
        }
        // 3. fused update
        IterParams P;
        P.seed = r->seed;
        P.key_iteration = key_it;
        P.ps = ps;
        P.dim = (int)r->dim;
        P.npairs = (int)r->npairs;
        P.ld = (int)r->ld;
        P.lower = r->lower;
        P.upper = r->upper;
        P.span = r->upper - r->lower;
        P.eps = r->eps;
        P.p_ah = r->sched[3 * t];
        P.f_mult = r->sched[3 * t + 1];
        P.decay = r->sched[3 * t + 2];
        P.rng = r->rng;
        set_iteration_base(P);
        cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};
        if (r->profile) {
            for (auto& e : ev) {
                APO_CUDA(cudaEventCreate(&e));
                r->prof_events.push_back(e);
            }
            APO_CUDA(cudaEventRecord(ev[0], st));
        }
        UpdArgs A{};
        A.P = P;
        A.O = r->obj;
        A.pos0 = r->pos[0];
        A.pos1 = r->pos[1];
        A.sel = r->sel[r->cur];
        A.sel_next = r->sel[r->cur ^ 1];
        A.fit = r->fit[r->cur];
        A.out_fit = r->fit[r->cur ^ 1];
        A.order = r->order;
        A.in_dr_bits = r->dr_bits;
        A.p_dr = r->p_dr;
        A.warn_count = r->warn;
        A.trace_key = r->trace_keys + t + 1;
        A.cec_bufs = cec_bufs_for(r->obj.code);
        if (int rc = launch_update(true, A, st, r->cand_ok, ev[1], r->tile_counter)) return rc;
        if (r->profile) APO_CUDA(cudaEventRecord(ev[2], st));
        r->cur ^= 1;
        r->iters++;
    }
    return APO_OK;
}

int apo_run_load(apo_run* r, const double* positions, const double* fitness, int is_host, int64_t iteration,
                 int64_t warnings) {
    APO_CHECK(r && positions && fitness, "NULL argument");
    APO_CHECK(iteration >= 0 && iteration <= r->T, "iteration outside [0, max_iterations]");
    cudaStream_t st = r->stream;
    const cudaMemcpyKind kind = is_host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
    // rows in reference row order become slots 0..ps-1 (identity order, buffer 0): exactly the state
    // the device loop would hold, since the next stable sort breaks ties by that order
    APO_CUDA(cudaMemcpy2DAsync(r->pos[0], 8 * (size_t)r->ld, positions, 8 * (size_t)r->dim, 8 * (size_t)r->dim,
                               (size_t)r->ps, kind, st));
    APO_CUDA(cudaMemcpyAsync(r->fit[0], fitness, 8 * (size_t)r->ps, kind, st));
    APO_CUDA(cudaMemsetAsync(r->sel[0], 0, (size_t)r->ps, st));
    k_iota<<<grid_for(r->ps, 256), 256, 0, st>>>((int)r->ps, r->order);
    APO_CUDA(cudaGetLastError());
    APO_CUDA(cudaMemsetAsync(r->trace_keys, 0xFF, 8 * (size_t)(r->T + 1), st));
    const unsigned long long w = (unsigned long long)warnings;
    APO_CUDA(cudaMemcpyAsync(r->warn, &w, 8, cudaMemcpyHostToDevice, st));
    APO_CUDA(cudaStreamSynchronize(st));  // w lives on this stack frame
    r->cur = 0;
    r->iters = iteration;
    r->initialized = true;
    return APO_OK;
}

int apo_run_trace(apo_run* r, double* trace_host, int64_t n) {
    APO_CHECK(r && trace_host && n >= 0 && n <= r->T, "bad arguments");
    std::vector<unsigned long long> k((size_t)n + 1);
    APO_CUDA(cudaMemcpyAsync(k.data(), r->trace_keys, 8 * ((size_t)n + 1), cudaMemcpyDeviceToHost, r->stream));
    APO_CUDA(cudaStreamSynchronize(r->stream));
    for (int64_t a = 0; a <= n; a++) trace_host[a] = key_to_double(k[(size_t)a]);
    return APO_OK;
}

int apo_run_population(apo_run* r, double* positions, double* fitness, int is_host) {
    APO_CHECK(r && r->initialized, "run not initialised");
    cudaStream_t st = r->stream;
    double* dpos = positions;
    double* dfit = fitness;
    if (is_host) {
        APO_CUDA(cudaMallocAsync((void**)&dpos, 8 * (size_t)r->ps * r->dim, st));
        APO_CUDA(cudaMallocAsync((void**)&dfit, 8 * (size_t)r->ps, st));
    }
    k_gather_rows<<<grid_for(r->ps * 32, 256), 256, 0, st>>>((int)r->ps, (int)r->dim, (int)r->ld, r->pos[0],
                                                             r->pos[1], r->sel[r->cur], r->fit[r->cur], r->order,
                                                             dpos, dfit);
    APO_CUDA(cudaGetLastError());
    if (is_host) {
        if (positions)
            APO_CUDA(cudaMemcpyAsync(positions, dpos, 8 * (size_t)r->ps * r->dim, cudaMemcpyDeviceToHost, st));
        if (fitness) APO_CUDA(cudaMemcpyAsync(fitness, dfit, 8 * (size_t)r->ps, cudaMemcpyDeviceToHost, st));
        cudaFreeAsync(dpos, st);
        cudaFreeAsync(dfit, st);
        APO_CUDA(cudaStreamSynchronize(st));
    }
    return APO_OK;
}

int apo_run_best(apo_run* r, double* best_fitness_host, double* best_position_host, int64_t* best_row_host) {
    APO_CHECK(r && r->initialized, "run not initialised");
    std::vector<double> fit((size_t)r->ps);
    std::vector<int> order((size_t)r->ps);
    cudaStream_t st = r->stream;
    APO_CUDA(cudaMemcpyAsync(order.data(), r->order, 4 * (size_t)r->ps, cudaMemcpyDeviceToHost, st));
    APO_CUDA(cudaMemcpyAsync(fit.data(), r->fit[r->cur], 8 * (size_t)r->ps, cudaMemcpyDeviceToHost, st));
    APO_CUDA(cudaStreamSynchronize(st));
    int64_t best = 0;
    for (int64_t a = 1; a < r->ps; a++)
        if (fit[(size_t)order[(size_t)a]] < fit[(size_t)order[(size_t)best]]) best = a;
    const int slot = order[(size_t)best];
    if (best_fitness_host) *best_fitness_host = fit[(size_t)slot];
    if (best_row_host) *best_row_host = best;
    if (best_position_host) {
        uint8_t which = 0;
        APO_CUDA(cudaMemcpyAsync(&which, r->sel[r->cur] + slot, 1, cudaMemcpyDeviceToHost, st));
        APO_CUDA(cudaStreamSynchronize(st));
        APO_CUDA(cudaMemcpyAsync(best_position_host, r->pos[which] + (size_t)slot * r->ld, 8 * (size_t)r->dim,
                                 cudaMemcpyDeviceToHost, st));
        APO_CUDA(cudaStreamSynchronize(st));
    }
    return APO_OK;
}

int apo_run_counters(apo_run* r, int64_t* iterations_run, int64_t* fe_count, int64_t* warnings) {
    APO_CHECK(r, "run is NULL");
    unsigned long long w = 0;
    APO_CUDA(cudaMemcpyAsync(&w, r->warn, 8, cudaMemcpyDeviceToHost, r->stream));
    APO_CUDA(cudaStreamSynchronize(r->stream));
    if (iterations_run) *iterations_run = r->iters;
    if (fe_count) *fe_count = r->ps * (1 + r->iters);
    if (warnings) *warnings = (int64_t)w;
    return APO_OK;
}

static void clear_profile(apo_run* r) {
    for (cudaEvent_t e : r->prof_events) cudaEventDestroy(e);
    r->prof_events.clear();
}

int apo_run_profile(apo_run* r, int enable) {
    APO_CHECK(r, "run is NULL");
    APO_CUDA(cudaStreamSynchronize(r->stream));
    clear_profile(r);
    r->profile = enable != 0;
    return APO_OK;
}

int apo_run_update_path(apo_run* r, int* path_host) {
    APO_CHECK(r && path_host, "NULL argument");
    UpdArgs A{};
    A.P.dim = (int)r->dim;
    A.P.ps = (int)r->ps;
    A.P.npairs = (int)r->npairs;
    A.O = r->obj;
    *path_host = update_path(true, A, true, true);
    return APO_OK;
}

int apo_run_profile_split(apo_run* r, double* candidates_ms_host, double* evaluate_ms_host, int64_t* launches_host) {
    APO_CHECK(r, "run is NULL");
    APO_CUDA(cudaStreamSynchronize(r->stream));
    double a = 0.0, b = 0.0;
    for (size_t k = 0; k + 2 < r->prof_events.size(); k += 3) {
        float m1 = 0.f, m2 = 0.f;
        APO_CUDA(cudaEventElapsedTime(&m1, r->prof_events[k], r->prof_events[k + 1]));
        APO_CUDA(cudaEventElapsedTime(&m2, r->prof_events[k + 1], r->prof_events[k + 2]));
        a += m1;
        b += m2;
    }
    if (candidates_ms_host) *candidates_ms_host = a;
    if (evaluate_ms_host) *evaluate_ms_host = b;
    if (launches_host) *launches_host = (int64_t)(r->prof_events.size() / 3);
    return APO_OK;
}

int apo_run_profile_read(apo_run* r, double* update_ms_host, int64_t* launches_host) {
    double a = 0.0, b = 0.0;
    if (int rc = apo_run_profile_split(r, &a, &b, launches_host)) return rc;
    if (update_ms_host) *update_ms_host = a + b;
    return APO_OK;
}

int apo_run_destroy(apo_run* r) {
    if (!r) return APO_OK;
    clear_profile(r);
    if (r->side) cudaStreamSynchronize(r->side);  // nothing may still run on the side stream
    void* bufs[] = {r->pos[0], r->pos[1], r->sel[0], r->sel[1], r->fit[0], r->fit[1], r->order, r->keys_in, r->keys_out, r->vals_in,
                    r->dr_keys, r->dr_sorted, r->dr_bits, r->tmp, r->p_dr, r->trace_keys, r->warn, r->cand_ok,
                    r->tile_counter, r->dr_tmp};
    for (void* b : bufs)
        if (b) cudaFreeAsync(b, r->stream);
    if (r->ev_fork) cudaEventDestroy(r->ev_fork);
    if (r->ev_join) cudaEventDestroy(r->ev_join);
    if (r->side) cudaStreamDestroy(r->side);
    delete r;
    return APO_OK;
}

int apo_release_cached_memory(void) {
    int dev = 0;
    cudaMemPool_t pool;
    APO_CUDA(cudaGetDevice(&dev));
    APO_CUDA(cudaDeviceSynchronize());
    APO_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
    APO_CUDA(cudaMemPoolTrimTo(pool, 0));
    return APO_OK;
}

// ----------------------------- sharded population -----------------------------
// One huge population split by RANK across processes (BASELINE config 4 on N
// GPUs).  Every process holds the whole population in rank order of the
// previous iteration (rows = "slots"), computes the identical stable sort
// and Dr set, updates only ranks [lo, hi) into the next buffer (rows by
// rank), and the caller exchanges the chunks (NCCL all-gather over NVLink)
// before apo_shard_end.  Position/fitness buffers are the caller's
// (torch tensors registered with NCCL), [ps_pad][ld] and [ps_pad].
struct apo_shard {
    int64_t ps, dim, ld, T;
    int rng;
    uint64_t seed;
    int64_t npairs;
    double pf_max, lower, upper, eps;
    ObjDesc obj;
    cudaStream_t stream;
    double* pos[2];
    double* fit[2];
    int cur;
    int* order;
    unsigned long long *keys_in, *keys_out, *dr_keys, *dr_sorted;
    int* vals_in;
    unsigned* dr_bits;
    int64_t dr_cap;
    void* tmp;
    size_t tmp_bytes;
    double* p_dr;
    uint8_t* cand_ok;
    unsigned* tile_counter;
    unsigned long long* trace_keys;  // [T+1], this process's ranks only (reduce MIN across processes)
    unsigned long long* warn;        // this process's ranks only (reduce SUM)
    std::vector<double> sched;
    int64_t iters;
};

int apo_shard_create(apo_shard** out, int64_t ps, int64_t dim, int64_t ld, int64_t max_iterations, uint64_t seed,
                     int64_t npairs, double pf_max, double lower, double upper, double eps,
                     const apo_objective* objective_host, const double* sched_host, const double* p_dr_host, int rng,
                     double* pos0, double* pos1, double* fit0, double* fit1, void* stream) {
    APO_CHECK(out != nullptr, "out is NULL");
    APO_CHECK(ps >= 1 && ps < (1LL << 31) && dim >= 1 && dim <= kGroupMaxDim && ld >= dim,
              "sharded runs need 1 <= dim <= 256 and ld >= dim");
    APO_CHECK(max_iterations >= 0 && npairs >= 1 && pf_max > 0.0 && pf_max <= 1.0, "bad config");
    APO_CHECK(rng == RNG_KEYED || rng == RNG_PHILOX, "bad rng");
    APO_CHECK((max_iterations == 0 || sched_host) && p_dr_host && pos0 && pos1 && fit0 && fit1, "NULL buffer");
    if (int rc = check_objective(objective_host, dim)) return rc;
    apo_shard* r = new apo_shard();
    r->ps = ps;
    r->dim = dim;
    r->ld = ld;
    r->T = max_iterations;
    r->rng = rng;
    r->seed = seed;
    r->npairs = npairs;
    r->pf_max = pf_max;
    r->lower = lower;
    r->upper = upper;
    r->eps = eps;
    r->obj = to_desc(objective_host);
    r->stream = as_stream(stream);
    r->pos[0] = pos0;
    r->pos[1] = pos1;
    r->fit[0] = fit0;
    r->fit[1] = fit1;
    r->cur = 0;
    r->iters = 0;
    r->sched.assign(sched_host, sched_host + 3 * max_iterations);
    r->dr_cap = (int64_t)ceil((double)ps * pf_max) + 1;
    size_t tb_sort = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb_sort, (unsigned long long*)nullptr, (unsigned long long*)nullptr,
                                    (int*)nullptr, (int*)nullptr, (int)ps, 0, 64, r->stream);
    const size_t tb_dr = dr_tmp_bytes(r->dr_cap, ps);
    r->tmp_bytes = tb_sort > tb_dr ? tb_sort : tb_dr;
    cudaError_t e = cudaSuccess;
    auto alloc = [&](void** p, size_t b) {
        if (e == cudaSuccess) e = cudaMalloc(p, b > 0 ? b : 16);
    };
    alloc((void**)&r->order, 4 * (size_t)ps);
    alloc((void**)&r->keys_in, 8 * (size_t)ps);
    alloc((void**)&r->keys_out, 8 * (size_t)ps);
    alloc((void**)&r->vals_in, 4 * (size_t)ps);
    alloc((void**)&r->dr_keys, 8 * (size_t)r->dr_cap);
    alloc((void**)&r->dr_sorted, 8 * (size_t)r->dr_cap);
    alloc((void**)&r->dr_bits, 4 * (size_t)((ps + 31) / 32));
    alloc(&r->tmp, r->tmp_bytes);
    alloc((void**)&r->p_dr, 8 * (size_t)ps);
    alloc((void**)&r->cand_ok, (size_t)ps);
    alloc((void**)&r->tile_counter, 16);
    alloc((void**)&r->trace_keys, 8 * (size_t)(max_iterations + 1));
    alloc((void**)&r->warn, 8);
    if (e != cudaSuccess) {
        apo_shard_destroy(r);
        return fail(APO_ENOMEM, std::string("apo_shard_create: ") + cudaGetErrorString(e));
    }
    APO_CUDA(cudaMemcpyAsync(r->p_dr, p_dr_host, 8 * (size_t)ps, cudaMemcpyHostToDevice, r->stream));
    APO_CUDA(cudaMemsetAsync(r->trace_keys, 0xFF, 8 * (size_t)(max_iterations + 1), r->stream));
    APO_CUDA(cudaMemsetAsync(r->warn, 0, 8, r->stream));
    *out = r;
    return APO_OK;
}

int apo_shard_initialize(apo_shard* r) {
    APO_CHECK(r, "shard is NULL");
    cudaStream_t st = r->stream;
    const int w = warps_for_dim(r->dim);
    const size_t smem = warp_scratch_bytes((int)r->dim) * (size_t)w;
    if (int rc = set_smem((const void*)k_init, smem)) return rc;
    const long long need = (r->ps + w - 1) / w;
    const long long cap = 8LL * num_sms();
    APO_CUDA(cudaMemsetAsync(r->trace_keys, 0xFF, 8 * (size_t)(r->T + 1), st));
    APO_CUDA(cudaMemsetAsync(r->warn, 0, 8, st));
    // every process builds the identical iteration-0 population (replicated, no exchange), with the
    // same evaluator as the single-GPU device loop (k_cec_eval in init mode for CEC2022)
    const bool cec_fast = r->obj.code > APO_OBJ_CEC2022_BASE && r->dim <= kCecEvalMaxDim && r->obj.cec.rot_pad;
    k_init<<<(int)(need < cap ? need : cap), 32 * w, smem, st>>>(r->rng, r->seed, (int)r->ps, (int)r->dim, (int)r->ld,
                                                                  r->lower, r->upper - r->lower, r->obj, r->pos[0],
                                                                  cec_fast ? nullptr : r->fit[0], r->trace_keys);
    APO_CUDA(cudaGetLastError());
    if (cec_fast) {
        UpdArgs A{};
        A.P.ps = (int)r->ps;
        A.P.dim = (int)r->dim;
        A.P.ld = (int)r->ld;
        A.O = r->obj;
        A.pos0 = r->pos[0];
        A.pos1 = r->pos[0];
        A.out_fit = r->fit[0];
        A.trace_key = r->trace_keys;
        A.rank_lo = 0;
        A.rank_hi = (int)r->ps;
        if (int rc = launch_cec_eval(true, A, st, nullptr, r->tile_counter, 1)) return rc;
    }
    r->cur = 0;
    r->iters = 0;
    return APO_OK;
}

// Sort + coordinator draws of the next iteration (identical on every process).
int apo_shard_begin(apo_shard* r) {
    APO_CHECK(r && r->iters < r->T, "iteration budget exceeded");
    cudaStream_t st = r->stream;
    const int ps = (int)r->ps;
    const uint64_t key_it = (uint64_t)r->iters + 1;
    // rows are in rank order of the previous iteration, so ties keep row order
    k_make_keys<<<grid_for(ps, 256), 256, 0, st>>>(ps, r->fit[r->cur], nullptr, r->keys_in, r->vals_in);
    APO_CUDA(cudaGetLastError());
    size_t tb = r->tmp_bytes;
    APO_CUDA(cub::DeviceRadixSort::SortPairs(r->tmp, tb, r->keys_in, r->keys_out, r->vals_in, r->order, ps, 0, 64, st));
    const int64_t count = (int64_t)coord_count(r->rng, r->seed, key_it, r->ps, r->pf_max);
    return dr_device(r->rng, r->seed, key_it, r->ps, count, r->dr_keys, r->dr_sorted, r->tmp, r->tmp_bytes, r->dr_bits,
                     nullptr, st);
}

// Update ranks [lo, hi) (lo % 32 == 0) into the next buffers (rows by rank).
int apo_shard_update_range(apo_shard* r, int64_t lo, int64_t hi) {
    APO_CHECK(r && lo >= 0 && lo <= hi && hi <= r->ps, "bad rank range");
    if (hi == lo) return APO_OK;
    APO_CHECK((lo & 31) == 0, "rank ranges must start on a multiple of 32");
    const int64_t t = r->iters;
    UpdArgs A{};
    A.P.seed = r->seed;
    A.P.key_iteration = (uint64_t)t + 1;
    A.P.ps = (int)r->ps;
    A.P.dim = (int)r->dim;
    A.P.npairs = (int)r->npairs;
    A.P.ld = (int)r->ld;
    A.P.lower = r->lower;
    A.P.upper = r->upper;
    A.P.span = r->upper - r->lower;
    A.P.eps = r->eps;
    A.P.p_ah = r->sched[3 * t];
    A.P.f_mult = r->sched[3 * t + 1];
    A.P.decay = r->sched[3 * t + 2];
    A.P.rng = r->rng;
    set_iteration_base(A.P);
    A.O = r->obj;
    A.pos = r->pos[r->cur];
    A.fit = r->fit[r->cur];
    A.order = r->order;
    A.out_pos = r->pos[r->cur ^ 1];
    A.out_fit = r->fit[r->cur ^ 1];
    A.in_dr_bits = r->dr_bits;
    A.p_dr = r->p_dr;
    A.warn_count = r->warn;
    A.trace_key = r->trace_keys + t + 1;
    A.cec_bufs = cec_bufs_for(r->obj.code);
    A.rank_lo = (int)lo;
    A.rank_hi = (int)hi;
    return launch_update(false, A, r->stream, r->cand_ok, nullptr, r->tile_counter);
}

int apo_shard_end(apo_shard* r) {
    APO_CHECK(r, "shard is NULL");
    r->cur ^= 1;
    r->iters++;
    return APO_OK;
}

int apo_shard_state(apo_shard* r, double** pos_host, double** fit_host, int64_t* iterations_host) {
    APO_CHECK(r, "shard is NULL");
    if (pos_host) *pos_host = r->pos[r->cur];
    if (fit_host) *fit_host = r->fit[r->cur];
    if (iterations_host) *iterations_host = r->iters;
    return APO_OK;
}

int apo_shard_counters(apo_shard* r, unsigned long long* trace_keys_host, int64_t n, int64_t* warnings_host) {
    APO_CHECK(r && n >= 0 && n <= r->T, "bad arguments");
    if (trace_keys_host)
        APO_CUDA(cudaMemcpyAsync(trace_keys_host, r->trace_keys, 8 * ((size_t)n + 1), cudaMemcpyDeviceToHost,
                                 r->stream));
    unsigned long long w = 0;
    APO_CUDA(cudaMemcpyAsync(&w, r->warn, 8, cudaMemcpyDeviceToHost, r->stream));
    APO_CUDA(cudaStreamSynchronize(r->stream));
    if (warnings_host) *warnings_host = (int64_t)w;
    return APO_OK;
}

int apo_shard_destroy(apo_shard* r) {
    if (!r) return APO_OK;
    void* bufs[] = {r->order, r->keys_in, r->keys_out, r->vals_in, r->dr_keys, r->dr_sorted, r->dr_bits, r->tmp,
                    r->p_dr, r->cand_ok, r->tile_counter, r->trace_keys, r->warn};
    for (void* b : bufs)
        if (b) cudaFree(b);
    delete r;
    return APO_OK;
}

// ------------------------------ batched runs -------------------------------

int apo_run_batch_fits(int64_t ps, int64_t dim, const apo_objective* objectives_host, int64_t nobj) {
    if (ps < 1 || dim < 1 || dim > 8192 || !objectives_host || nobj < 1) return 0;
    int cec_bufs = 0, tab = 0;
    batch_smem_needs(objectives_host, nobj, dim, &cec_bufs, &tab);
    const BatchLayout L = batch_layout((int)ps, (int)dim, (int)((dim + 1) & ~1LL), kWarps, cec_bufs, tab);
    return (int64_t)L.total + 2048 <= smem_optin() ? 1 : 0;
}

int64_t apo_run_batch_max_elems(int64_t ps, int64_t dim) {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess) optin = 227 * 1024;
    const int64_t ld = (dim + 1) & ~1LL;
    const BatchLayout L = batch_layout((int)ps, (int)dim, (int)ld, kWarps, 0);
    return (int64_t)L.total + 2048 <= optin ? ps * dim : 0;
}

int apo_run_batch(int64_t nruns, const uint64_t* seeds, const apo_objective* objectives_host, int64_t ps,
                  int64_t dim, int64_t max_iterations, int64_t n_iters, int64_t npairs, double pf_max, double lower,
                  double upper, double eps, const double* sched, const double* p_dr, double* best_fit,
                  double* best_pos, double* trace, double* final_pos, double* final_fit, int64_t* warnings,
                  int rng, void* stream) {
    return apo_run_batch_shaped(nruns, seeds, objectives_host, ps, dim, max_iterations, n_iters, npairs, pf_max,
                                lower, upper, eps, sched, p_dr, best_fit, best_pos, trace, final_pos, final_fit,
                                warnings, rng, 0, stream);
}

int apo_run_batch_shaped(int64_t nruns, const uint64_t* seeds, const apo_objective* objectives_host, int64_t ps,
                         int64_t dim, int64_t max_iterations, int64_t n_iters, int64_t npairs, double pf_max,
                         double lower, double upper, double eps, const double* sched, const double* p_dr,
                         double* best_fit, double* best_pos, double* trace, double* final_pos, double* final_fit,
                         int64_t* warnings, int rng, int threads_per_run, void* stream) {
    APO_CHECK(rng == RNG_KEYED || rng == RNG_PHILOX, "rng must be APO_RNG_KEYED or APO_RNG_PHILOX");
    APO_CHECK(threads_per_run == 0 || (threads_per_run >= 32 && threads_per_run <= kBatchMaxThreads &&
                                       threads_per_run % 32 == 0),
              "threads_per_run must be 0 or a multiple of 32 in [32, 640]");
    APO_CHECK(nruns >= 1 && nruns < (1LL << 31), "nruns out of range");
    APO_CHECK(ps >= 1 && dim >= 1 && dim <= 8192, "bad shape");
    APO_CHECK(n_iters >= 0 && n_iters <= max_iterations, "n_iters must be in [0, max_iterations]");
    APO_CHECK(npairs >= 1 && pf_max > 0.0 && pf_max <= 1.0, "bad config");
    APO_CHECK(seeds && objectives_host && best_fit && p_dr && (n_iters == 0 || sched), "NULL buffer");
    for (int64_t k = 0; k < nruns; k++)
        if (int rc = check_objective(&objectives_host[k], dim)) return rc;
    APO_CHECK(apo_run_batch_max_elems(ps, dim) > 0, "population too large for the shared-memory batch kernel");
    cudaStream_t st = as_stream(stream);
    // one staging block: descriptors | claim order | claim counter
    const size_t desc_bytes = (sizeof(ObjDesc) * (size_t)nruns + 15) & ~(size_t)15;
    const size_t order_bytes = (4 * (size_t)nruns + 15) & ~(size_t)15;
    std::vector<unsigned char> stage(desc_bytes + order_bytes + 16, 0);
    ObjDesc* descs = reinterpret_cast<ObjDesc*>(stage.data());
    for (int64_t k = 0; k < nruns; k++) descs[k] = to_desc(&objectives_host[k]);
    {
        // costliest runs first (per-objective cost of a D = 20 run relative to ~20 for the basic functions;
        // measured with tools/prof_batch.py): the last claims then go to the cheap runs
        static const float kCecCost[13] = {20, 23, 23, 24, 28, 24, 26, 58, 35, 37, 33, 58, 50};
        auto cost = [&](int64_t k) {
            const int c = objectives_host[k].code;
            return c > APO_OBJ_CEC2022_BASE && c <= APO_OBJ_CEC2022_BASE + 12 ? kCecCost[c - APO_OBJ_CEC2022_BASE]
                                                                              : 20.0f;
        };
        std::vector<int> ord((size_t)nruns);
        for (int64_t k = 0; k < nruns; k++) ord[(size_t)k] = (int)k;
        std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return cost(a) > cost(b); });
        memcpy(stage.data() + desc_bytes, ord.data(), 4 * (size_t)nruns);
    }
    unsigned char* d_stage = nullptr;
    APO_CUDA(cudaMallocAsync((void**)&d_stage, stage.size(), st));
    APO_CUDA(cudaMemcpyAsync(d_stage, stage.data(), stage.size(), cudaMemcpyHostToDevice, st));
    ObjDesc* d_descs = reinterpret_cast<ObjDesc*>(d_stage);
    BatchArgs A;
    A.seeds = seeds;
    A.objs = d_descs;
    A.ps = (int)ps;
    A.dim = (int)dim;
    A.ld = (int)((dim + 1) & ~1LL);
    A.max_iterations = (int)max_iterations;
    A.n_iters = (int)n_iters;
    A.npairs = (int)npairs;
    A.pf_max = pf_max;
    A.lower = lower;
    A.upper = upper;
    A.span = upper - lower;
    A.eps = eps;
    A.sched = sched;
    A.p_dr = p_dr;
    A.best_fit = best_fit;
    A.best_pos = best_pos;
    A.trace = trace;
    A.final_pos = final_pos;
    A.final_fit = final_fit;
    A.warnings = (long long*)warnings;
    A.rng = rng;
    static const int env_lpp = getenv("APO_BATCH_LPP") ? atoi(getenv("APO_BATCH_LPP")) : 1;
    A.lpp = env_lpp && npairs == 1 ? 1 : 0;
    static const int env_lpp_g = getenv("APO_BATCH_LPP_G") ? atoi(getenv("APO_BATCH_LPP_G")) : 32;
    A.lpp_group = env_lpp_g;
    static const int env_g = getenv("APO_BATCH_G") ? atoi(getenv("APO_BATCH_G")) : 0;
    A.group = env_g;
    batch_smem_needs(objectives_host, nruns, dim, &A.cec_bufs, &A.tab_smem);
    BatchLayout L = batch_layout(A.ps, A.dim, A.ld, kWarps, A.cec_bufs, A.tab_smem);
    APO_CHECK((int64_t)L.total + 2048 <= smem_optin(), "population too large for the shared-memory batch kernel");
    // Launch shape (k_run_batch's comment): more runs than SMs -> one persistent kBatchPersistThreads CTA
    // per SM claiming runs costliest first (C2: 360 runs 1.8x faster than 3 x 256-thread CTAs per SM
    // with one run each, whose slowest SM holds three heavy runs); else one kBatchWideThreads CTA per
    // run (a run is latency-bound).  threads_per_run > 0 forces one CTA of that size per run (batches
    // sharing the GPU with others).  APO_BATCH_THREADS / APO_BATCH_WORKERS override (A/B runs).
    static const int env_threads = getenv("APO_BATCH_THREADS") ? atoi(getenv("APO_BATCH_THREADS")) : 0;
    static const int env_workers = getenv("APO_BATCH_WORKERS") ? atoi(getenv("APO_BATCH_WORKERS")) : 0;
    const int sms = num_sms();
    int threads = kThreads;
    long long workers = 0;  // 0: one CTA per run
    if (env_threads > 0 || env_workers > 0) {
        if (env_threads > 0) threads = env_threads & ~31;
        if (env_workers > 0 && env_workers < nruns) workers = env_workers;
    } else if (threads_per_run > 0) {
        threads = threads_per_run;
    } else if (nruns > sms) {
        threads = kBatchPersistThreads;
        workers = sms;
    } else if (ps > (int64_t)kWarps) {
        threads = kBatchWideThreads;
    }
    APO_CHECK(threads >= 32 && threads <= kBatchMaxThreads, "APO_BATCH_THREADS must be in [32, 640]");
    if (threads != kThreads) {
        const BatchLayout W = batch_layout(A.ps, A.dim, A.ld, threads / 32, A.cec_bufs, A.tab_smem);
        if ((int64_t)W.total + 2048 <= smem_optin()) {
            L = W;
        } else {  // the wide scratch does not fit: the default shape
            threads = kThreads;
            workers = 0;
        }
    }
    const void* fn = pick_run_batch((int)dim, rng, npairs > 1);
    if (int rc = set_smem(fn, L.total)) return rc;
    A.nruns = (int)nruns;
    A.run_order = nullptr;
    A.run_counter = nullptr;
    long long grid = nruns;
    if (workers > 0) {
        A.run_order = reinterpret_cast<const int*>(d_stage + desc_bytes);
        A.run_counter = reinterpret_cast<unsigned*>(d_stage + desc_bytes + order_bytes);
        grid = workers;
    }
    void* args[] = {(void*)&A};
    APO_CUDA(cudaLaunchKernel(fn, dim3((unsigned)grid), dim3((unsigned)threads), args, L.total, st));
    APO_CUDA(cudaGetLastError());
    cudaFreeAsync(d_stage, st);
    return APO_OK;
}

}  // extern "C"
