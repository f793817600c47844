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

int b200sp_jacobi_pack(int64_t nblocks, const int32_t* starts, const int64_t* off64, const double* inv64,
                       const uint8_t* prec, const int64_t* offs, void* storage, void* stream) {
    if (nblocks == 0) return B200SP_OK;
    jacobi_pack_kernel<<<grid_for(nblocks * 32, 256, 8), 256, 0, as_stream(stream)>>>(
        nblocks, starts, (const long long*)off64, inv64, prec, (const long long*)offs, (unsigned char*)storage);
    count_launch();
    return check_launch("jacobi_pack");
}

}  // extern "C"
