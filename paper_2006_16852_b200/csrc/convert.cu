// Device-side format conversions (two-phase: sizes, host-visible scan, fill).
//
// The reference converts every pair through canonical host MatrixData
// (src/formats.py:301-322, `convert`) and has no Ell/Sellp/Hybrid at all
// (SPEC.md:294). Here Csr is the hub: Csr <-> Coo/Ell/Sellp/Hybrid/Dense run
// on the device. Index arrays produced from a canonical Csr are bit-exact
// restatements of oracle/convert.py (the parity check for these layouts).
//
// Layouts (shared with oracle/convert.py):
//   Ell    : col-major, element (row, k) at k*stride + row; pad col=-1, val=0
//   Sellp  : slices of S rows; slice s has length L_s = round_up(max row nnz in
//            slice, stride_factor); element (row, k) at (sets[s]+k)*S + row%S
//   Hybrid : first `width` entries of each row in an Ell part, the remaining
//            entries, in row-major order, in a Coo part
#include "common.cuh"

namespace b200sp {

__global__ void csr_row_lengths_kernel(int64_t n, const int* __restrict__ rp, int* __restrict__ len) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        len[i] = rp[i + 1] - rp[i];
}

// sub-warp (32 lanes) per row, so long rows do not serialise one thread
__global__ void csr_to_coo_rows_kernel(int64_t n, const int* __restrict__ rp, int* __restrict__ rows) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n; r += nw) {
        const int s = rp[r], e = rp[r + 1];
        for (int k = s + lane; k < e; k += 32) rows[k] = (int)r;
    }
}

// rows sorted ascending -> row_ptrs[0..n]
__global__ void coo_to_csr_ptrs_kernel(int64_t nnz, int64_t n, const int* __restrict__ rows, int* __restrict__ rp) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k <= nnz; k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t prev = k > 0 ? rows[k - 1] : -1;
        const int64_t cur = k < nnz ? rows[k] : n;
        for (int64_t r = prev + 1; r <= cur; ++r) rp[r] = (int)k;
    }
}

template <typename T>
__global__ void csr_to_ell_kernel(int64_t n, const int* __restrict__ rp, const int* __restrict__ ci,
                                  const T* __restrict__ v, int64_t width, int64_t stride,
                                  int* __restrict__ eci, T* __restrict__ ev) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        const int s = rp[r];
        const int len = rp[r + 1] - s;
        for (int64_t k = 0; k < width; ++k) {
            const bool in = k < len;
            eci[k * stride + r] = in ? ci[s + k] : -1;
            ev[k * stride + r] = in ? v[s + k] : T(0);
        }
    }
}

// padding rows beyond n (stride > n) are also set to pad values
template <typename T>
__global__ void ell_pad_tail_kernel(int64_t n, int64_t width, int64_t stride, int* __restrict__ eci, T* __restrict__ ev) {
    const int64_t extra = stride - n;
    const int64_t tot = extra * width;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = t / extra, r = n + (t - k * extra);
        eci[k * stride + r] = -1;
        ev[k * stride + r] = T(0);
    }
}

__global__ void sellp_slice_lengths_kernel(int64_t n, const int* __restrict__ rp, int slice_size,
                                           int stride_factor, int64_t nslices, int* __restrict__ out) {
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < nslices; s += (int64_t)gridDim.x * blockDim.x) {
        int m = 0;
        const int64_t r0 = s * slice_size, r1 = min(r0 + slice_size, n);
        for (int64_t r = r0; r < r1; ++r) m = max(m, rp[r + 1] - rp[r]);
        out[s] = (m + stride_factor - 1) / stride_factor * stride_factor;
    }
}

template <typename T>
__global__ void csr_to_sellp_kernel(int64_t n, const int* __restrict__ rp, const int* __restrict__ ci,
                                    const T* __restrict__ v, int slice_size, int64_t nslices,
                                    const int* __restrict__ sl, const int* __restrict__ ss,
                                    int* __restrict__ sci, T* __restrict__ sv) {
    // one thread per slot row (covers the padded rows of the last slice too)
    const int64_t total_rows = nslices * slice_size;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < total_rows; r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = r / slice_size, local = r - s * slice_size;
        const int L = sl[s];
        const int64_t base = (int64_t)ss[s] * slice_size + local;
        int start = 0, len = 0;
        if (r < n) {
            start = rp[r];
            len = rp[r + 1] - start;
        }
        for (int k = 0; k < L; ++k) {
            const bool in = k < len;
            sci[base + (int64_t)k * slice_size] = in ? ci[start + k] : -1;
            sv[base + (int64_t)k * slice_size] = in ? v[start + k] : T(0);
        }
    }
}

__global__ void hybrid_overflow_kernel(int64_t n, const int* __restrict__ rp, int width, int* __restrict__ cnt) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
        cnt[r] = max(0, rp[r + 1] - rp[r] - width);
}

template <typename T>
__global__ void csr_to_hybrid_coo_kernel(int64_t n, const int* __restrict__ rp, const int* __restrict__ ci,
                                         const T* __restrict__ v, int width, const int* __restrict__ offs,
                                         int* __restrict__ crow, int* __restrict__ cci, T* __restrict__ cv) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n; r += nw) {
        const int s = rp[r] + width, e = rp[r + 1];
        const int o = offs[r] - s;
        for (int k = s + lane; k < e; k += 32) {
            crow[o + k] = (int)r;
            cci[o + k] = ci[k];
            cv[o + k] = v[k];
        }
    }
}

// count of stored (col >= 0) entries per row of an Ell block
__global__ void ell_row_lengths_kernel(int64_t n, int64_t width, int64_t stride, const int* __restrict__ eci,
                                       int* __restrict__ len) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        int c = 0;
        for (int64_t k = 0; k < width; ++k) c += eci[k * stride + r] >= 0;
        len[r] = c;
    }
}

// Ell entries of each row appended at rp[r] (+ optional extra offset array),
// padding skipped
template <typename T>
__global__ void ell_to_csr_fill_kernel(int64_t n, int64_t width, int64_t stride, const int* __restrict__ eci,
                                       const T* __restrict__ ev, const int* __restrict__ rp,
                                       int* __restrict__ ci, T* __restrict__ v) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        int o = rp[r];
        for (int64_t k = 0; k < width; ++k) {
            const int c = eci[k * stride + r];
            if (c >= 0) {
                ci[o] = c;
                v[o] = ev[k * stride + r];
                ++o;
            }
        }
    }
}

__global__ void sellp_row_lengths_kernel(int64_t n, int slice_size, const int* __restrict__ sl,
                                         const int* __restrict__ ss, const int* __restrict__ sci,
                                         int* __restrict__ len) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = r / slice_size, local = r - s * slice_size;
        const int64_t base = (int64_t)ss[s] * slice_size + local;
        int c = 0;
        for (int k = 0; k < sl[s]; ++k) c += sci[base + (int64_t)k * slice_size] >= 0;
        len[r] = c;
    }
}

template <typename T>
__global__ void sellp_to_csr_fill_kernel(int64_t n, int slice_size, const int* __restrict__ sl,
                                         const int* __restrict__ ss, const int* __restrict__ sci,
                                         const T* __restrict__ sv, const int* __restrict__ rp,
                                         int* __restrict__ ci, T* __restrict__ v) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = r / slice_size, local = r - s * slice_size;
        const int64_t base = (int64_t)ss[s] * slice_size + local;
        int o = rp[r];
        for (int k = 0; k < sl[s]; ++k) {
            const int c = sci[base + (int64_t)k * slice_size];
            if (c >= 0) {
                ci[o] = c;
                v[o] = sv[base + (int64_t)k * slice_size];
                ++o;
            }
        }
    }
}

// Hybrid -> Csr: row length = ell stored + coo entries of the row
__global__ void add_csr_lengths_kernel(int64_t n, const int* __restrict__ rp2, int* __restrict__ len) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
        len[r] += rp2[r + 1] - rp2[r];
}

// append the Coo part of each row after its Ell entries (rp = combined ptrs,
// ell_len = stored Ell entries per row, crp = Coo row ptrs)
template <typename T>
__global__ void hybrid_coo_append_kernel(int64_t n, const int* __restrict__ rp, const int* __restrict__ ell_len,
                                         const int* __restrict__ crp, const int* __restrict__ cci,
                                         const T* __restrict__ cv, int* __restrict__ ci, T* __restrict__ v) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        int o = rp[r] + ell_len[r];
        for (int k = crp[r]; k < crp[r + 1]; ++k, ++o) {
            ci[o] = cci[k];
            v[o] = cv[k];
        }
    }
}

// histogram of row lengths (bins >= nbins - 1 collapse into the last bin)
__global__ void length_histogram_kernel(int64_t n, const int* __restrict__ rp, int nbins,
                                        unsigned long long* __restrict__ hist) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        int l = rp[r + 1] - rp[r];
        if (l >= nbins) l = nbins - 1;
        atomicAdd(hist + l, 1ull);
    }
}

// Dense (n, k) row-major <-> Csr
template <typename T>
__global__ void dense_row_nnz_kernel(int64_t n, int64_t k, const T* __restrict__ a, int64_t as, int* __restrict__ len) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        int c = 0;
        for (int64_t j = 0; j < k; ++j) c += a[r * as + j] != T(0);
        len[r] = c;
    }
}

template <typename T>
__global__ void dense_to_csr_fill_kernel(int64_t n, int64_t k, const T* __restrict__ a, int64_t as,
                                         const int* __restrict__ rp, int* __restrict__ ci, T* __restrict__ v) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        int o = rp[r];
        for (int64_t j = 0; j < k; ++j) {
            const T x = a[r * as + j];
            if (x != T(0)) {
                ci[o] = (int)j;
                v[o] = x;
                ++o;
            }
        }
    }
}

template <typename T>
__global__ void csr_to_dense_kernel(int64_t n, const int* __restrict__ rp, const int* __restrict__ ci,
                                    const T* __restrict__ v, T* __restrict__ a, int64_t as) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
        for (int k = rp[r]; k < rp[r + 1]; ++k) a[r * as + ci[k]] += v[k];
}

// rows with no stored entry (Coo prefill list): flag then compact by scan
__global__ void empty_row_flags_kernel(int64_t n, const int* __restrict__ rp, int* __restrict__ flag) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
        flag[r] = rp[r + 1] == rp[r];
}

__global__ void compact_flags_kernel(int64_t n, const int* __restrict__ flag, const int* __restrict__ pos,
                                     int* __restrict__ out) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
        if (flag[r]) out[pos[r]] = (int)r;
}

}  // namespace b200sp

using namespace b200sp;

#define LAUNCH1D(kernel, work, ...)                                                        \
    do {                                                                                   \
        kernel<<<grid_for((work) > 0 ? (work) : 1, 256, 8), 256, 0, as_stream(stream)>>>(__VA_ARGS__); \
        count_launch();                                                                    \
        return check_launch(#kernel);                                                      \
    } while (0)

extern "C" {

int b200sp_csr_row_lengths(int64_t n, const int32_t* rp, int32_t* len, void* stream) {
    if (n == 0) return B200SP_OK;
    LAUNCH1D(csr_row_lengths_kernel, n, n, rp, len);
}

int b200sp_csr_to_coo_rows(int64_t n, const int32_t* rp, int32_t* rows, void* stream) {
    if (n == 0) return B200SP_OK;
    LAUNCH1D(csr_to_coo_rows_kernel, n * 32, n, rp, rows);
}

int b200sp_coo_to_csr_ptrs(int64_t nnz, int64_t n, const int32_t* rows, int32_t* rp, void* stream) {
    LAUNCH1D(coo_to_csr_ptrs_kernel, nnz + 1, nnz, n, rows, rp);
}

int b200sp_sellp_slice_lengths(int64_t n, const int32_t* rp, int32_t slice_size, int32_t stride_factor,
                               int32_t* out, void* stream) {
    const int64_t ns = ceil_div(n, slice_size);
    if (ns == 0) return B200SP_OK;
    B200SP_REQUIRE(slice_size > 0 && stride_factor > 0, B200SP_EINVAL, "sellp: bad slice_size/stride_factor");
    LAUNCH1D(sellp_slice_lengths_kernel, ns, n, rp, slice_size, stride_factor, ns, out);
}

int b200sp_hybrid_overflow_counts(int64_t n, const int32_t* rp, int32_t width, int32_t* cnt, void* stream) {
    if (n == 0) return B200SP_OK;
    LAUNCH1D(hybrid_overflow_kernel, n, n, rp, width, cnt);
}

int b200sp_ell_row_lengths(int64_t n, int64_t width, int64_t stride, const int32_t* eci, int32_t* len, void* stream) {
    if (n == 0) return B200SP_OK;
    LAUNCH1D(ell_row_lengths_kernel, n, n, width, stride, eci, len);
}

int b200sp_sellp_row_lengths(int64_t n, int32_t slice_size, const int32_t* sl, const int32_t* ss,
                             const int32_t* sci, int32_t* len, void* stream) {
    if (n == 0) return B200SP_OK;
    LAUNCH1D(sellp_row_lengths_kernel, n, n, slice_size, sl, ss, sci, len);
}

int b200sp_add_csr_lengths(int64_t n, const int32_t* rp2, int32_t* len, void* stream) {
    if (n == 0) return B200SP_OK;
    LAUNCH1D(add_csr_lengths_kernel, n, n, rp2, len);
}

int b200sp_length_histogram(int64_t n, const int32_t* rp, int32_t nbins, unsigned long long* hist, void* stream) {
    B200SP_CHECK_CUDA(cudaMemsetAsync(hist, 0, sizeof(unsigned long long) * nbins, as_stream(stream)));
    if (n == 0) return B200SP_OK;
    LAUNCH1D(length_histogram_kernel, n, n, rp, nbins, hist);
}

int b200sp_empty_row_flags(int64_t n, const int32_t* rp, int32_t* flag, void* stream) {
    if (n == 0) return B200SP_OK;
    LAUNCH1D(empty_row_flags_kernel, n, n, rp, flag);
}

int b200sp_compact_flags(int64_t n, const int32_t* flag, const int32_t* pos, int32_t* out, void* stream) {
    if (n == 0) return B200SP_OK;
    LAUNCH1D(compact_flags_kernel, n, n, flag, pos, out);
}

#define CONVERT_T(T, SUF)                                                                                     \
    int b200sp_csr_to_ell_##SUF(int64_t n, const int32_t* rp, const int32_t* ci, const T* v, int64_t width,   \
                                int64_t stride, int32_t* eci, T* ev, void* stream) {                          \
        B200SP_REQUIRE(stride >= n, B200SP_EINVAL, "ell: stride < rows");                                    \
        if (stride > n && width > 0) {                                                                        \
            ell_pad_tail_kernel<T><<<grid_for((stride - n) * width, 256, 8), 256, 0, as_stream(stream)>>>(    \
                n, width, stride, eci, ev);                                                                   \
            count_launch();                                                                                   \
        }                                                                                                     \
        if (n == 0 || width == 0) return check_launch("ell_pad");                                             \
        LAUNCH1D(csr_to_ell_kernel<T>, n, n, rp, ci, v, width, stride, eci, ev);                              \
    }                                                                                                         \
    int b200sp_csr_to_sellp_##SUF(int64_t n, const int32_t* rp, const int32_t* ci, const T* v,               \
                                  int32_t slice_size, const int32_t* sl, const int32_t* ss, int32_t* sci,     \
                                  T* sv, void* stream) {                                                      \
        const int64_t ns = ceil_div(n, slice_size);                                                           \
        if (ns == 0) return B200SP_OK;                                                                        \
        LAUNCH1D(csr_to_sellp_kernel<T>, ns* slice_size, n, rp, ci, v, slice_size, ns, sl, ss, sci, sv);      \
    }                                                                                                         \
    int b200sp_csr_to_hybrid_coo_##SUF(int64_t n, const int32_t* rp, const int32_t* ci, const T* v,         \
                                       int32_t width, const int32_t* offs, int32_t* crow, int32_t* cci,       \
                                       T* cv, void* stream) {                                                 \
        if (n == 0) return B200SP_OK;                                                                         \
        LAUNCH1D(csr_to_hybrid_coo_kernel<T>, n * 32, n, rp, ci, v, width, offs, crow, cci, cv);              \
    }                                                                                                         \
    int b200sp_ell_to_csr_fill_##SUF(int64_t n, int64_t width, int64_t stride, const int32_t* eci,           \
                                     const T* ev, const int32_t* rp, int32_t* ci, T* v, void* stream) {       \
        if (n == 0) return B200SP_OK;                                                                         \
        LAUNCH1D(ell_to_csr_fill_kernel<T>, n, n, width, stride, eci, ev, rp, ci, v);                         \
    }                                                                                                         \
    int b200sp_sellp_to_csr_fill_##SUF(int64_t n, int32_t slice_size, const int32_t* sl, const int32_t* ss,  \
                                       const int32_t* sci, const T* sv, const int32_t* rp, int32_t* ci, T* v, \
                                       void* stream) {                                                        \
        if (n == 0) return B200SP_OK;                                                                         \
        LAUNCH1D(sellp_to_csr_fill_kernel<T>, n, n, slice_size, sl, ss, sci, sv, rp, ci, v);                  \
    }                                                                                                         \
    int b200sp_hybrid_coo_append_##SUF(int64_t n, const int32_t* rp, const int32_t* ell_len,                 \
                                       const int32_t* crp, const int32_t* cci, const T* cv, int32_t* ci,     \
                                       T* v, void* stream) {                                                  \
        if (n == 0) return B200SP_OK;                                                                         \
        LAUNCH1D(hybrid_coo_append_kernel<T>, n, n, rp, ell_len, crp, cci, cv, ci, v);                        \
    }                                                                                                         \
    int b200sp_dense_row_nnz_##SUF(int64_t n, int64_t k, const T* a, int64_t as, int32_t* len,               \
                                   void* stream) {                                                            \
        if (n == 0) return B200SP_OK;                                                                         \
        LAUNCH1D(dense_row_nnz_kernel<T>, n, n, k, a, as, len);                                               \
    }                                                                                                         \
    int b200sp_dense_to_csr_fill_##SUF(int64_t n, int64_t k, const T* a, int64_t as, const int32_t* rp,      \
                                       int32_t* ci, T* v, void* stream) {                                     \
        if (n == 0) return B200SP_OK;                                                                         \
        LAUNCH1D(dense_to_csr_fill_kernel<T>, n, n, k, a, as, rp, ci, v);                                     \
    }                                                                                                         \
    int b200sp_csr_to_dense_##SUF(int64_t n, const int32_t* rp, const int32_t* ci, const T* v, T* a,         \
                                  int64_t as, void* stream) {                                                 \
        if (n == 0) return B200SP_OK;                                                                         \
        LAUNCH1D(csr_to_dense_kernel<T>, n, n, rp, ci, v, a, as);                                             \
    }

CONVERT_T(double, f64)
CONVERT_T(float, f32)

}  // extern "C"
