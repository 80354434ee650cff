// apo_cec_gemm.cu -- CEC2022 at large D (> 104): the rotation as a real DMMA GEMM.
//
// For D beyond the register-resident k_cec_eval tiles, one candidate's
// rotation is a GEMV with no reuse of M, so per-warp evaluation is bound by
// streaming M (8 MB at D = 1000) once per candidate.  Batching every
// candidate of the iteration turns it into the N x D x D contraction the
// north star asks for:
//   k_cec_prep    Y[r] = transform(candidate r)  ((x - o) * scale, the step
//                 rounding of F4; zero-padded to Kp)
//   k_dgemm_nn    Z = Y * R  (R = M^T zero-padded to Kp x Np, columns
//                 pre-permuted for the hybrids) -- mma.sync m8n8k4 f64, 64x64
//                 CTA tiles, 16-deep k slices double-buffered with cp.async
//   k_cec_finish  per candidate (one warp): offsets, segments / composition
//                 components, basic functions, greedy select, best-so-far
// Covers the CEC2022 functions with a single rotation (F1-F8, F10).
#include <cuda_runtime.h>

#include "apo_kernels.cuh"

namespace apo {
namespace {

constexpr int GBM = 64, GBN = 64, GBK = 16;
constexpr int GAS = GBK + 4;  // A smem row stride (doubles): bank-conflict-free fragment loads
constexpr int GBS = GBN + 4;  // B smem row stride

__device__ __forceinline__ void cp16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

// Y[r][i] = transform of candidate r (row pointer through the SEL selector or dense)
__global__ void __launch_bounds__(256) k_cec_prep(CecGemmArgs A) {
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    const CecSpec& S = kCecSpec[A.O.cec.fn - 1];
    const int k = A.comp;
    const int b = S.basic[k];
    const bool single = S.kind == 0, hybrid = S.kind == 1;
    const double sc = hybrid ? 1.0 : cec_scale(b);
    const double* o = A.O.cec.shift + (size_t)k * A.dim;
    for (int rr = warp; rr < A.n_rows; rr += nw) {
        const int r = A.row0 + rr;
        const double* x = A.sel ? ((A.sel[r] ? A.pos0 : A.pos1) + (size_t)r * A.ld) : A.out_pos + (size_t)r * A.ld;
        double* y = A.Y + (size_t)rr * A.kp;
        for (int i = lane; i < A.kp; i += 32) {
            double v = 0.0;
            if (i < A.dim) {
                double xi = x[i];
                const double oi = o[i];
                if (single && b == B_STEP_RASTRIGIN && fabs(xi - oi) > 0.5) xi = oi + floor(2.0 * (xi - oi) + 0.5) / 2.0;
                v = (xi - oi) * sc;
            }
            y[i] = v;
        }
    }
}

// Z[M x Np] = Y[M x Kp] * R[Kp x Np], all row-major, Kp % 16 == 0, Np % 64 == 0.
// 4 warps as 2 x 2, each a 32 x 32 sub-tile = 4 x 4 m8n8 tiles in registers.
__global__ void __launch_bounds__(128) k_dgemm_nn(const double* __restrict__ Y, const double* __restrict__ R,
                                                  double* __restrict__ Z, int M, int Kp, int Np) {
    __shared__ __align__(16) double As[2][GBM * GAS];
    __shared__ __align__(16) double Bs[2][GBK * GBS];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp >> 1, wn = warp & 1;
    const int g = lane >> 2, t = lane & 3;
    const int m0 = blockIdx.y * GBM, n0 = blockIdx.x * GBN;
    auto load = [&](int buf, int k0) {
        // A: 64 rows x 16 doubles = 512 x 16 B chunks; B: 16 rows x 64 doubles = 512 chunks
        for (int c = tid; c < GBM * GBK / 2; c += 128) {
            const int row = c >> 3, col = (c & 7) * 2;
            double* dst = &As[buf][row * GAS + col];
            if (m0 + row < M) cp16(dst, Y + (size_t)(m0 + row) * Kp + k0 + col);
            else dst[0] = dst[1] = 0.0;
        }
        for (int c = tid; c < GBK * GBN / 2; c += 128) {
            const int row = c >> 5, col = (c & 31) * 2;
            cp16(&Bs[buf][row * GBS + col], R + (size_t)(k0 + row) * Np + n0 + col);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    double acc[4][4][2];
#pragma unroll
    for (int a = 0; a < 4; a++)
#pragma unroll
        for (int c = 0; c < 4; c++) acc[a][c][0] = acc[a][c][1] = 0.0;
    const int nk = Kp / GBK;
    load(0, 0);
    for (int kt = 0; kt < nk; kt++) {
        const int buf = kt & 1;
        if (kt + 1 < nk) {
            load(buf ^ 1, (kt + 1) * GBK);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();
        const double* as = As[buf] + (wm * 32) * GAS;
        const double* bs = Bs[buf] + wn * 32;
#pragma unroll
        for (int k4 = 0; k4 < GBK; k4 += 4) {
            double af[4], bf[4];
#pragma unroll
            for (int a = 0; a < 4; a++) af[a] = as[(a * 8 + g) * GAS + k4 + t];
#pragma unroll
            for (int c = 0; c < 4; c++) bf[c] = bs[(k4 + t) * GBS + c * 8 + g];
#pragma unroll
            for (int a = 0; a < 4; a++)
#pragma unroll
                for (int c = 0; c < 4; c++) dmma_m8n8k4(acc[a][c][0], acc[a][c][1], af[a], bf[c]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int a = 0; a < 4; a++) {
        const int row = m0 + wm * 32 + a * 8 + g;
        if (row >= M) continue;
#pragma unroll
        for (int c = 0; c < 4; c++) {
            const int col = n0 + wn * 32 + c * 8 + 2 * t;
            *reinterpret_cast<double2*>(Z + (size_t)row * Np + col) = make_double2(acc[a][c][0], acc[a][c][1]);
        }
    }
}

// One warp per candidate: the rest of F_fn from the rotated row, then the greedy select.
__global__ void __launch_bounds__(256) k_cec_finish(CecGemmArgs A) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    double* z = reinterpret_cast<double*>(smem) + (size_t)wib * 2 * A.np;  // rotated row, then scratch
    double* y = z + A.np;
    const CecSpec& S = kCecSpec[A.O.cec.fn - 1];
    const int n = A.dim;
    unsigned long long my_min = ~0ull;
    unsigned my_warn = 0;
    for (int rr = warp; rr < A.n_rows; rr += nw) {
        const int r = A.row0 + rr;
        const uint8_t cur = A.sel ? A.sel[r] : 0;
        const double* x = A.sel ? ((cur ? A.pos0 : A.pos1) + (size_t)r * A.ld) : A.out_pos + (size_t)r * A.ld;
        const double* zr = A.Z + (size_t)rr * A.np;
        for (int i = lane; i < n; i += 32) z[i] = zr[i];
        __syncwarp();
        double f = 0.0;
        if (S.kind == 0) {
            const int b = S.basic[0];
            const double off = cec_offset(b);
            for (int i = lane; i < n; i += 32) z[i] = z[i] + off;
            __syncwarp();
            f = cec_basic_warp(b, z, n, lane);
        } else if (S.kind == 1) {  // z is already in segment order (R's columns are permuted)
            int sizes[6];
            int tot = 0;
            for (int k = 0; k < S.ncomp - 1; k++) {
                sizes[k] = (int)ceil(S.p[k] * n);
                if (sizes[k] > n - tot) sizes[k] = n - tot;  // oracle: or_cec_segments
                tot += sizes[k];
            }
            sizes[S.ncomp - 1] = n - tot;
            int start = 0;
            for (int k = 0; k < S.ncomp; k++) {
                const double sc = cec_scale(S.basic[k]), off = cec_offset(S.basic[k]);
                for (int i = lane; i < sizes[k]; i += 32) z[start + i] = z[start + i] * sc + off;
                start += sizes[k];
            }
            __syncwarp();
            start = 0;
            for (int k = 0; k < S.ncomp; k++) {
                if (sizes[k] > 0) f += cec_basic_warp(S.basic[k], z + start, sizes[k], lane);
                start += sizes[k];
            }
        } else {  // composition with exactly one rotated component (A.comp): its rotation came from the GEMM
            double fit[6], wk[6];
            int inf_at = -1;
            for (int k = 0; k < S.ncomp; k++) {
                const int b = S.basic[k];
                const double sc = cec_scale(b), off = cec_offset(b);
                const double* o = A.O.cec.shift + (size_t)k * n;
                double d2 = 0.0;
                for (int i = lane; i < n; i += 32) {
                    const double dv = x[i] - o[i];
                    d2 += dv * dv;
                    y[i] = k == A.comp ? z[i] + off : dv * sc + off;
                }
                d2 = wsum(d2);
                __syncwarp();
                fit[k] = S.lam[k] * cec_basic_warp(b, y, n, lane) + S.bias[k];
                __syncwarp();
                wk[k] = d2 != 0.0 ? sqrt(1.0 / d2) * exp(-d2 / 2.0 / n / (S.sigma[k] * S.sigma[k]))
                                  : __longlong_as_double(0x7ff0000000000000LL);
                if (d2 == 0.0 && inf_at < 0) inf_at = k;
            }
            double wmax = 0.0, wsum_ = 0.0;
            for (int k = 0; k < S.ncomp; k++)
                if (wk[k] > wmax) wmax = wk[k];
            if (inf_at >= 0) {
                f = fit[inf_at];
            } else if (wmax == 0.0) {
                for (int k = 0; k < S.ncomp; k++) f += fit[k] / S.ncomp;
            } else {
                for (int k = 0; k < S.ncomp; k++) wsum_ += wk[k];
                for (int k = 0; k < S.ncomp; k++) f += wk[k] / wsum_ * fit[k];
            }
        }
        f += S.fstar;
        bool acc = false;
        if (lane == 0) {
            const double fit_i = A.fit[A.order ? A.order[r] : r];
            double kept = fit_i;
            bool warned = false;
            if (A.cand_ok[r] && isfinite(f)) {
                acc = f < fit_i;
                if (acc) kept = f;
            } else {
                warned = true;
            }
            A.out_fit[r] = kept;
            if (A.sel) {
                A.sel_next[r] = acc ? (uint8_t)(cur ^ 1) : cur;
            } else {
                if (A.out_acc) A.out_acc[r] = acc ? 1 : 0;
                if (A.out_warn) A.out_warn[r] = warned ? 1 : 0;
            }
            const unsigned long long key = sort_key(kept);
            my_min = key < my_min ? key : my_min;
            my_warn += warned ? 1u : 0u;
        }
        acc = __shfl_sync(kFull, acc, 0);
        if (!A.sel && !acc) {  // dense: a rejected row keeps the old one
            const double* old = A.pos + (size_t)(A.order ? A.order[r] : r) * A.ld;
            double* dst = A.out_pos + (size_t)r * A.ld;
            for (int d = lane; d < n; d += 32) dst[d] = old[d];
        }
        __syncwarp();
    }
    block_finish(my_min, my_warn, A.warn_count, A.trace_key);
}

}  // namespace

int cec_gemm_finish(const CecGemmArgs& A0, cudaStream_t st, int num_sms) {
    CecGemmArgs A = A0;
    if (A.n_rows <= 0) return 0;
    static bool pool_kept = [] {  // keep freed scratch in the stream-ordered pool (no re-mapping per launch)
        int dev = 0;
        cudaGetDevice(&dev);
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t keep = ~0ull;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
        return true;
    }();
    (void)pool_kept;
    const size_t ybytes = 8 * (size_t)A.n_rows * A.kp, zbytes = 8 * (size_t)A.n_rows * A.np;
    if (cudaMallocAsync((void**)&A.Y, ybytes, st) != cudaSuccess) return 1;
    if (cudaMallocAsync((void**)&A.Z, zbytes, st) != cudaSuccess) {
        cudaFreeAsync(A.Y, st);
        return 1;
    }
    const int pw = (int)((A.n_rows + 7) / 8);
    k_cec_prep<<<pw < 16 * num_sms ? pw : 16 * num_sms, 256, 0, st>>>(A);
    dim3 grid(A.np / GBN, (A.n_rows + GBM - 1) / GBM);
    k_dgemm_nn<<<grid, 128, 0, st>>>(A.Y, A.O.cec.rot_gemm, A.Z, A.n_rows, A.kp, A.np);
    const size_t fsmem = 8 * 2 * (size_t)A.np * 8;
    // always set: the 48 KB default also has to hold the kernel's static shared memory
    cudaFuncSetAttribute((const void*)k_cec_finish, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsmem);
    k_cec_finish<<<pw < 8 * num_sms ? pw : 8 * num_sms, 256, fsmem, st>>>(A);
    cudaFreeAsync(A.Y, st);
    cudaFreeAsync(A.Z, st);
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

}  // namespace apo
