// Block-Jacobi generation and application (batched, one warp per block).
//
// Generation restates the reference's _JacobiGenerateKernel +
// gauss_jordan_inverse + _extract_block (src/precond.py:28-95, :200-208)
// operation for operation, so inverses, condition numbers and the adaptive
// storage decision are bit-identical to the reference:
//   * Gauss-Jordan on [B | I] with partial pivoting, pivot = first maximum of
//     |column| (np.argmax), row swap, pivot row divided by the pivot, then
//     aug -= outer(factor, pivot_row) as an IEEE multiply followed by a
//     subtraction (no FMA contraction: __dmul_rn / __dsub_rn);
//   * kappa_inf = max_i sum_j |B_ij| * max_i sum_j |inv_ij|, with each row sum
//     in NumPy's pairwise order (8 accumulators for 8 <= n <= 128);
//   * fp32 storage when adaptive and kappa < threshold.
#include "jacobi.cuh"

namespace b200sp {

constexpr int JG_WARPS = 2;  // warps (= blocks) per CTA
constexpr int JG_LD = 65;    // padded row length of [B | I] (2*32 + 1)

// NumPy pairwise_sum (n <= 128) of |a[0..n)| with element stride `st`
__device__ double np_abs_rowsum(const double* a, int n, int st) {
    if (n < 8) {
        double res = 0.0;
        for (int i = 0; i < n; ++i) res = __dadd_rn(res, fabs(a[i * st]));
        return res;
    }
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = fabs(a[j * st]);
    int i = 8;
    for (; i < n - (n % 8); i += 8)
        for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], fabs(a[(i + j) * st]));
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, fabs(a[i * st]));
    return res;
}

template <typename T>
__global__ void __launch_bounds__(32 * JG_WARPS)
jacobi_invert_kernel(int64_t nblocks, const int* __restrict__ starts, const int* __restrict__ rp,
                     const int* __restrict__ ci, const T* __restrict__ vals, const long long* __restrict__ off64,
                     double* __restrict__ inv64, double* __restrict__ cond, unsigned char* __restrict__ prec,
                     int* __restrict__ nbytes, int adaptive, double threshold, long long* __restrict__ singular) {
    __shared__ double s_aug[JG_WARPS][32 * JG_LD];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double* aug = s_aug[w];
    for (int64_t b = (int64_t)blockIdx.x * JG_WARPS + w; b < nblocks; b += (int64_t)gridDim.x * JG_WARPS) {
        const int r0 = starts[b];
        const int bs = starts[b + 1] - r0;
        // [B | I]
        for (int i = lane; i < 32 * JG_LD; i += 32) aug[i] = 0.0;
        __syncwarp();
        if (lane < bs) {
            const int row = r0 + lane;
            for (int k = rp[row]; k < rp[row + 1]; ++k) {
                const int c = ci[k] - r0;
                if (c >= 0 && c < bs) aug[lane * JG_LD + c] = (double)vals[k];
            }
            aug[lane * JG_LD + bs + lane] = 1.0;
        }
        __syncwarp();
        const double norm_b = lane < bs ? np_abs_rowsum(aug + lane * JG_LD, bs, 1) : 0.0;
        bool sing = false;
        for (int col = 0; col < bs; ++col) {
            double av = (lane >= col && lane < bs) ? fabs(aug[lane * JG_LD + col]) : -1.0;
            int idx = lane;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, av, o);
                const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
                if (ov > av || (ov == av && oi < idx)) {
                    av = ov;
                    idx = oi;
                }
            }
            const int piv = idx;
            if (aug[piv * JG_LD + col] == 0.0) {
                sing = true;
                break;
            }
            if (piv != col) {
                for (int c = lane; c < 2 * bs; c += 32) {
                    const double t = aug[col * JG_LD + c];
                    aug[col * JG_LD + c] = aug[piv * JG_LD + c];
                    aug[piv * JG_LD + c] = t;
                }
                __syncwarp();
            }
            const double pv = aug[col * JG_LD + col];
            __syncwarp();
            for (int c = lane; c < 2 * bs; c += 32) aug[col * JG_LD + c] = __ddiv_rn(aug[col * JG_LD + c], pv);
            __syncwarp();
            if (lane < bs && lane != col) {
                const double f = aug[lane * JG_LD + col];
                for (int c = 0; c < 2 * bs; ++c)
                    aug[lane * JG_LD + c] = __dsub_rn(aug[lane * JG_LD + c], __dmul_rn(f, aug[col * JG_LD + c]));
            }
            __syncwarp();
        }
        if (sing) {
            if (lane == 0) atomicMin(singular, (long long)b);
            __syncwarp();
            continue;
        }
        const double norm_inv = lane < bs ? np_abs_rowsum(aug + lane * JG_LD + bs, bs, 1) : 0.0;
        double mb = norm_b, mi = norm_inv;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            mb = fmax(mb, __shfl_xor_sync(0xffffffffu, mb, o));
            mi = fmax(mi, __shfl_xor_sync(0xffffffffu, mi, o));
        }
        const double kappa = __dmul_rn(mb, mi);
        const bool reduced = adaptive && kappa < threshold;
        double* dst = inv64 + off64[b];
        if (lane < bs)
            for (int c = 0; c < bs; ++c) dst[c * bs + lane] = aug[lane * JG_LD + bs + c];
        if (lane == 0) {
            cond[b] = kappa;
            prec[b] = reduced ? 1 : 0;
            nbytes[b] = bs * bs * (reduced ? 4 : 8);
        }
        __syncwarp();
    }
}

// pack fp64 inverses into the mixed-precision storage
__global__ void jacobi_pack_kernel(int64_t nblocks, const int* __restrict__ starts, const long long* __restrict__ off64,
                                   const double* __restrict__ inv64, const unsigned char* __restrict__ prec,
                                   const long long* __restrict__ offs, unsigned char* __restrict__ storage) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < nblocks; b += nw) {
        const int bs = starts[b + 1] - starts[b];
        const double* src = inv64 + off64[b];
        if (prec[b]) {
            float* d = reinterpret_cast<float*>(storage + offs[b]);
            for (int i = lane; i < bs * bs; i += 32) d[i] = (float)src[i];
        } else {
            double* d = reinterpret_cast<double*>(storage + offs[b]);
            for (int i = lane; i < bs * bs; i += 32) d[i] = src[i];
        }
    }
}

// z = M r for (n, m) blocks (column j by column), warp per block
template <typename T>
__global__ void jacobi_apply_kernel(JacobiView J, int m, const T* __restrict__ r, int64_t rs, T* __restrict__ z,
                                    int64_t zs, const int* guard) {
    if (guard && *(volatile const int*)guard) return;  // see b200sp_set_guard
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < J.nblocks; b += nw) {
        const int64_t r0 = J.starts[b];
        const int bs = J.starts[b + 1] - (int)r0;
        for (int j = 0; j < m; ++j) {
            const T rv = lane < bs ? r[(r0 + lane) * rs + j] : T(0);
            const T zv = jacobi_row<T>(J, b, bs, lane, rv);
            if (lane < bs) z[(r0 + lane) * zs + j] = zv;
        }
    }
}

// ---------------------------------------------------------------------------
// Blocks larger than a warp (reference: any block_size / block_boundaries,
// src/precond.py:155-197). One CTA per block; [B | I] lives in a global
// scratch slot (bs x 2bs fp64, row-major, L2-resident for moderate bs) and
// every Gauss-Jordan step is the reference's vectorised statement spread over
// the CTA: first-max pivot (np.argmax), row swap, pivot-row divide, then
// aug -= outer(factor, pivot_row) with the factors snapshotted first
// (factor = aug[:, col].copy(); factor[col] = 0). Same IEEE operations as the
// warp kernel above, so small and large blocks share one arithmetic contract.
// ---------------------------------------------------------------------------
constexpr int JL_THREADS = 256;
constexpr int JL_MAX_BS = 4096;

// NumPy pairwise_sum of |a[0..n)| with element stride st, any n
// (numpy/_core/src/umath/loops_utils.h.src: blocks of 128, 8 accumulators,
// recursive halving with n2 rounded down to a multiple of 8)
__device__ double np_abs_rowsum_any(const double* a, int n, int st) {
    if (n <= 128) return np_abs_rowsum(a, n, st);
    int n2 = n / 2;
    n2 -= n2 % 8;
    return __dadd_rn(np_abs_rowsum_any(a, n2, st), np_abs_rowsum_any(a + (int64_t)n2 * st, n - n2, st));
}

__device__ __forceinline__ double block_max(double v, double* sh) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    __syncthreads();
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    double r = sh[0];
    for (int w = 1; w < JL_THREADS / 32; ++w) r = fmax(r, sh[w]);
    return r;
}

template <typename T>
__global__ void __launch_bounds__(JL_THREADS)
jacobi_invert_large_kernel(int64_t nblocks, const int* __restrict__ starts, const int* __restrict__ rp,
                           const int* __restrict__ ci, const T* __restrict__ vals, const long long* __restrict__ off64,
                           double* __restrict__ inv64, double* __restrict__ cond, unsigned char* __restrict__ prec,
                           int* __restrict__ nbytes, int adaptive, double threshold, long long* __restrict__ singular,
                           int max_bs, double* __restrict__ scratch) {
    extern __shared__ double s_fac[];  // max_bs factors
    __shared__ double s_red[JL_THREADS / 32];
    __shared__ double s_rv[JL_THREADS / 32];
    __shared__ int s_ri[JL_THREADS / 32];
    __shared__ int s_piv;
    double* aug = scratch + (int64_t)blockIdx.x * max_bs * 2 * max_bs;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    for (int64_t b = blockIdx.x; b < nblocks; b += gridDim.x) {
        const int r0 = starts[b];
        const int bs = starts[b + 1] - r0;
        if (bs <= 0) continue;
        const int ld = 2 * bs;
        for (int64_t i = tid; i < (int64_t)bs * ld; i += JL_THREADS) aug[i] = 0.0;
        __syncthreads();
        for (int l = w; l < bs; l += JL_THREADS / 32) {  // _extract_block: a warp per row
            const int row = r0 + l;
            for (int k = rp[row] + lane; k < rp[row + 1]; k += 32) {
                const int c = ci[k] - r0;
                if (c >= 0 && c < bs) aug[(int64_t)l * ld + c] = (double)vals[k];
            }
            if (lane == 0) aug[(int64_t)l * ld + bs + l] = 1.0;
        }
        __syncthreads();
        double nb = 0.0;
        for (int l = tid; l < bs; l += JL_THREADS) nb = fmax(nb, np_abs_rowsum_any(aug + (int64_t)l * ld, bs, 1));
        const double norm_b = block_max(nb, s_red);
        bool sing = false;
        for (int col = 0; col < bs; ++col) {
            // pivot = col + argmax |aug[col:, col]| (first maximum)
            double av = -1.0;
            int ai = bs;
            for (int l = col + tid; l < bs; l += JL_THREADS) {
                const double v = fabs(aug[(int64_t)l * ld + col]);
                if (v > av) av = v, ai = l;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, av, o);
                const int oi = __shfl_xor_sync(0xffffffffu, ai, o);
                if (ov > av || (ov == av && oi < ai)) av = ov, ai = oi;
            }
            if (lane == 0) s_rv[w] = av, s_ri[w] = ai;
            __syncthreads();
            if (tid == 0) {
                double bv = s_rv[0];
                int bi = s_ri[0];
                for (int k = 1; k < JL_THREADS / 32; ++k)
                    if (s_rv[k] > bv || (s_rv[k] == bv && s_ri[k] < bi)) bv = s_rv[k], bi = s_ri[k];
                s_piv = bi;
            }
            __syncthreads();
            const int piv = s_piv;
            if (aug[(int64_t)piv * ld + col] == 0.0) {
                sing = true;
                break;
            }
            if (piv != col) {
                for (int c = tid; c < ld; c += JL_THREADS) {
                    const double t = aug[(int64_t)col * ld + c];
                    aug[(int64_t)col * ld + c] = aug[(int64_t)piv * ld + c];
                    aug[(int64_t)piv * ld + c] = t;
                }
                __syncthreads();
            }
            const double pv = aug[(int64_t)col * ld + col];
            __syncthreads();
            for (int c = tid; c < ld; c += JL_THREADS) aug[(int64_t)col * ld + c] = __ddiv_rn(aug[(int64_t)col * ld + c], pv);
            __syncthreads();
            for (int l = tid; l < bs; l += JL_THREADS) s_fac[l] = l == col ? 0.0 : aug[(int64_t)l * ld + col];
            __syncthreads();
            const double* prow = aug + (int64_t)col * ld;
            for (int l = w; l < bs; l += JL_THREADS / 32) {
                if (l == col) continue;  // factor 0: the reference leaves the pivot row as is
                const double f = s_fac[l];
                double* row = aug + (int64_t)l * ld;
                for (int c = lane; c < ld; c += 32) row[c] = __dsub_rn(row[c], __dmul_rn(f, prow[c]));
            }
            __syncthreads();
        }
        if (sing) {
            if (tid == 0) atomicMin(singular, (long long)b);
            __syncthreads();
            continue;
        }
        double ni = 0.0;
        for (int l = tid; l < bs; l += JL_THREADS) ni = fmax(ni, np_abs_rowsum_any(aug + (int64_t)l * ld + bs, bs, 1));
        const double norm_inv = block_max(ni, s_red);
        const double kappa = __dmul_rn(norm_b, norm_inv);
        const bool reduced = adaptive && kappa < threshold;
        double* dst = inv64 + off64[b];
        for (int64_t i = tid; i < (int64_t)bs * bs; i += JL_THREADS) {  // column-major: (l, c) at c*bs + l
            const int c = (int)(i / bs), l = (int)(i % bs);
            dst[i] = aug[(int64_t)l * ld + bs + c];
        }
        if (tid == 0) {
            cond[b] = kappa;
            prec[b] = reduced ? 1 : 0;
            nbytes[b] = bs * bs * (reduced ? 4 : 8);
        }
        __syncthreads();
    }
}

// z = M r for blocks of any size: a CTA per block, a warp per 32-row chunk of
// it; r[c] is loaded 32 entries at a time and broadcast with shuffles, the
// inverse's columns are read coalesced (column-major storage).
template <typename T, typename S>
__device__ __forceinline__ T jacobi_chunk_row(const S* inv, int bs, int l, const T* __restrict__ r, int64_t r0,
                                              int64_t rs, int j, int lane) {
    T acc = 0;
    for (int c0 = 0; c0 < bs; c0 += 32) {
        const T rv = c0 + lane < bs ? r[(r0 + c0 + lane) * rs + j] : T(0);
        const int cn = min(32, bs - c0);
        for (int cc = 0; cc < cn; ++cc) {
            const T rc = __shfl_sync(0xffffffffu, rv, cc);
            if (l < bs) acc += (T)(double)ld_stream(inv + (int64_t)(c0 + cc) * bs + l) * rc;
        }
    }
    return acc;
}

template <typename T>
__global__ void __launch_bounds__(JL_THREADS)
jacobi_apply_large_kernel(JacobiView J, int m, const T* __restrict__ r, int64_t rs, T* __restrict__ z, int64_t zs,
                          const int* guard) {
    if (guard && *(volatile const int*)guard) return;  // see b200sp_set_guard
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int64_t b = blockIdx.x; b < J.nblocks; b += gridDim.x) {
        const int64_t r0 = J.starts[b];
        const int bs = J.starts[b + 1] - (int)r0;
        const unsigned char* base = J.storage + J.offs[b];
        for (int ch = w * 32; ch < bs; ch += JL_THREADS) {
            const int l = ch + lane;
            for (int j = 0; j < m; ++j) {
                const T zv = J.prec[b] ? jacobi_chunk_row<T>(reinterpret_cast<const float*>(base), bs, l, r, r0, rs, j, lane)
                                       : jacobi_chunk_row<T>(reinterpret_cast<const double*>(base), bs, l, r, r0, rs, j, lane);
                if (l < bs) z[(r0 + l) * zs + j] = zv;
            }
        }
    }
}

__global__ void block_sizes_sq_kernel(int64_t nblocks, const int* __restrict__ starts, int* __restrict__ out) {
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nblocks; b += (int64_t)gridDim.x * blockDim.x) {
        const int bs = starts[b + 1] - starts[b];
        out[b] = bs * bs;
    }
}

}  // namespace b200sp

using namespace b200sp;

extern "C" {

int b200sp_jacobi_block_sizes_sq(int64_t nblocks, const int32_t* starts, int32_t* out, void* stream) {
    if (nblocks == 0) return B200SP_OK;
    block_sizes_sq_kernel<<<grid_for(nblocks, 256, 8), 256, 0, as_stream(stream)>>>(nblocks, starts, out);
    count_launch();
    return check_launch("jacobi_block_sizes_sq");
}

#define JACOBI_T(T, SUF)                                                                                         \
    int b200sp_jacobi_invert_##SUF(int64_t nblocks, const int32_t* starts, const int32_t* rp, const int32_t* ci,  \
                                   const T* vals, const int64_t* off64, double* inv64, double* cond,             \
                                   uint8_t* prec, int32_t* nbytes, int32_t adaptive, double threshold,            \
                                   int64_t* singular, void* stream) {                                             \
        if (nblocks == 0) return B200SP_OK;                                                                       \
        const int64_t want = ceil_div(nblocks, JG_WARPS), cap = (int64_t)kNumSMs * 16;                          \
        const unsigned grid = (unsigned)(want < cap ? want : cap);                                                \
        jacobi_invert_kernel<T><<<grid, 32 * JG_WARPS, 0, as_stream(stream)>>>(                                   \
            nblocks, starts, rp, ci, vals, (const long long*)off64, inv64, cond, prec, nbytes, adaptive, threshold, \
            (long long*)singular);                                                                                \
        count_launch();                                                                                           \
        return check_launch("jacobi_invert");                                                                     \
    }                                                                                                             \
    int b200sp_jacobi_apply_##SUF(int64_t nblocks, const int32_t* starts, const int64_t* offs, const uint8_t* prec, \
                                  const void* storage, int32_t m, const T* r, int64_t rs, T* z, int64_t zs,       \
                                  void* stream) {                                                                 \
        if (nblocks == 0) return B200SP_OK;                                                                       \
        JacobiView J{nblocks, starts, (const long long*)offs, prec, (const unsigned char*)storage};               \
        jacobi_apply_kernel<T><<<grid_for(nblocks * 32, 256, 8), 256, 0, as_stream(stream)>>>(J, m, r, rs, z, zs, current_guard()); \
        count_launch();                                                                                           \
        return check_launch("jacobi_apply");                                                                      \
    }

JACOBI_T(double, f64)
JACOBI_T(float, f32)

int64_t b200sp_jacobi_large_max_block(void) { return JL_MAX_BS; }

#define JACOBI_LARGE_T(T, SUF)                                                                                   \
    int b200sp_jacobi_invert_large_##SUF(int64_t nblocks, const int32_t* starts, const int32_t* rp,               \
                                         const int32_t* ci, const T* vals, const int64_t* off64, double* inv64,    \
                                         double* cond, uint8_t* prec, int32_t* nbytes, int32_t adaptive,           \
                                         double threshold, int64_t* singular, int32_t max_bs, double* scratch,     \
                                         int32_t slots, void* stream) {                                            \
        if (nblocks == 0) return B200SP_OK;                                                                       \
        B200SP_REQUIRE(max_bs >= 1 && max_bs <= JL_MAX_BS, B200SP_EINVAL,                                         \
                       "jacobi: blocks are limited to %d rows", JL_MAX_BS);                                        \
        B200SP_REQUIRE(slots >= 1, B200SP_EINVAL, "jacobi: need at least one scratch slot");                      \
        const unsigned grid = (unsigned)(nblocks < slots ? nblocks : slots);                                      \
        const size_t smem = (size_t)max_bs * sizeof(double);                                                      \
        if (smem > 48 * 1024)                                                                                     \
            B200SP_CHECK_CUDA(cudaFuncSetAttribute(jacobi_invert_large_kernel<T>,                                 \
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));      \
        jacobi_invert_large_kernel<T><<<grid, JL_THREADS, smem, as_stream(stream)>>>(                              \
            nblocks, starts, rp, ci, vals, (const long long*)off64, inv64, cond, prec, nbytes, adaptive, threshold, \
            (long long*)singular, max_bs, scratch);                                                               \
        count_launch();                                                                                           \
        return check_launch("jacobi_invert_large");                                                               \
    }                                                                                                             \
    int b200sp_jacobi_apply_large_##SUF(int64_t nblocks, const int32_t* starts, const int64_t* offs,              \
                                        const uint8_t* prec, const void* storage, int32_t m, const T* r, int64_t rs, \
                                        T* z, int64_t zs, void* stream) {                                         \
        if (nblocks == 0) return B200SP_OK;                                                                       \
        JacobiView J{nblocks, starts, (const long long*)offs, prec, (const unsigned char*)storage};               \
        const int64_t cap = (int64_t)kNumSMs * 8;                                                                 \
        jacobi_apply_large_kernel<T><<<(unsigned)(nblocks < cap ? nblocks : cap), JL_THREADS, 0, as_stream(stream)>>>( \
            J, m, r, rs, z, zs, current_guard());                                                                 \
        count_launch();                                                                                           \
        return check_launch("jacobi_apply_large");                                                                \
    }

JACOBI_LARGE_T(double, f64)
JACOBI_LARGE_T(float, f32)

int b200sp_jacobi_pack(int64_t nblocks, const int32_t* starts, const int64_t* off64, const double* inv64,
                       const uint8_t* prec, const int64_t* offs, void* storage, void* stream) {
    if (nblocks == 0) return B200SP_OK;
    jacobi_pack_kernel<<<grid_for(nblocks * 32, 256, 8), 256, 0, as_stream(stream)>>>(
        nblocks, starts, (const long long*)off64, inv64, prec, (const long long*)offs, (unsigned char*)storage);
    count_launch();
    return check_launch("jacobi_pack");
}

}  // extern "C"
