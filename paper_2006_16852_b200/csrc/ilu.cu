// ParILU(0) generation and sparse triangular solves.
//
// ParILU (reference src/precond.py:211-331, the Chow-Patel fixed-point
// iteration): L = unit-lower with the pattern of tril(A), U = upper with the
// pattern of triu(A); initial L = tril(A) scaled by the diagonal, U = triu(A);
// every sweep recomputes ALL entries from the previous sweep's values
// (Jacobi style):
//     l_ij = (a_ij - sum_{k<j} l_ik u_kj) / u_jj      (i > j)
//     u_ij =  a_ij - sum_{k<i} l_ik u_kj               (i <= j)
// summed over k ascending where (i,k) is in L and (k,j) in U. One thread per
// stored entry walks row i of L and finds (k, j) in row k of U by binary
// search (columns sorted), so no transposed pattern is needed.
//
// Triangular solves (reference src/solvers/triangular.py:18-155): a
// synchronisation-free substitution. Warps claim rows in dependency order
// through an atomic ticket (forward order for L, backward for U), wait on
// the per-row "solved" flags of the row's dependencies (acquire loads), and
// publish x_i with a release store of the flag -- no level sets, no host
// round trips, and deadlock-free because a row only waits on rows claimed
// before it. Flags carry an epoch so they never need clearing.
#include <cstdint>

#include "common.cuh"

namespace b200sp {

// ---- pattern split ----------------------------------------------------------
// per row: entries with col <= i (L, diagonal included) / col >= i (U)
__global__ void ilu_counts_kernel(int64_t n, const int* __restrict__ rp, const int* __restrict__ ci,
                                  int* __restrict__ lcnt, int* __restrict__ ucnt, int* __restrict__ nodiag) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int l = 0, u = 0, d = 0;
        for (int p = rp[i]; p < rp[i + 1]; ++p) {
            const int c = ci[p];
            l += c <= i;
            u += c >= i;
            d |= c == i;
        }
        lcnt[i] = l;
        ucnt[i] = u;
        if (!d) atomicMin(nodiag, (int)i);
    }
}

template <typename T>
__global__ void ilu_diag_kernel(int64_t n, const int* __restrict__ rp, const int* __restrict__ ci,
                                const T* __restrict__ v, T* __restrict__ diag, int* __restrict__ zero) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        T d = 0;
        for (int p = rp[i]; p < rp[i + 1]; ++p)
            if (ci[p] == i) {
                d = v[p];  // first stored diagonal (canonical matrices have one)
                break;
            }
        diag[i] = d;
        if (d == T(0)) atomicMin(zero, (int)i);
    }
}

// fill the L / U patterns, the original values (a_lower / a_upper) and the
// initial iterate: l_ij = a_ij / a_jj (l_ii = 1), u_ij = a_ij
template <typename T>
__global__ void ilu_fill_kernel(int64_t n, const int* __restrict__ rp, const int* __restrict__ ci,
                                const T* __restrict__ v, const T* __restrict__ diag, const int* __restrict__ lrp,
                                const int* __restrict__ urp, int* __restrict__ lci, T* __restrict__ al,
                                T* __restrict__ lv, int* __restrict__ uci, T* __restrict__ au, T* __restrict__ uv) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int lp = lrp[i], up = urp[i];
        for (int p = rp[i]; p < rp[i + 1]; ++p) {
            const int c = ci[p];
            const T a = v[p];
            if (c <= i) {
                lci[lp] = c;
                al[lp] = a;
                lv[lp] = c == i ? T(1) : a / diag[c];
                ++lp;
            }
            if (c >= i) {
                uci[up] = c;
                au[up] = a;
                uv[up] = a;
                ++up;
            }
        }
    }
}

// position of column j in row k of U (cols sorted), or -1
__device__ __forceinline__ int u_find(const int* __restrict__ urp, const int* __restrict__ uci, int k, int j) {
    int lo = urp[k], hi = urp[k + 1];
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        const int c = uci[mid];
        if (c == j) return mid;
        if (c < j) lo = mid + 1;
        else hi = mid;
    }
    return -1;
}

// one Jacobi sweep: entries e < nl are L entries, the rest U entries
template <typename T>
__global__ void parilu_sweep_kernel(int64_t n, int64_t nl, int64_t nu, const int* __restrict__ lrow,
                                    const int* __restrict__ lrp, const int* __restrict__ lci,
                                    const T* __restrict__ al, const T* __restrict__ lold, T* __restrict__ lnew,
                                    const int* __restrict__ urow, const int* __restrict__ urp,
                                    const int* __restrict__ uci, const T* __restrict__ au,
                                    const T* __restrict__ uold, T* __restrict__ unew) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nl + nu; t += (int64_t)gridDim.x * blockDim.x) {
        const bool lower = t < nl;
        const int64_t e = lower ? t : t - nl;
        const int i = lower ? lrow[e] : urow[e];
        const int j = lower ? lci[e] : uci[e];
        if (lower && i == j) {
            lnew[e] = T(1);
            continue;
        }
        const int kmax = min(i, j);
        T s = 0;
        bool any = false;
        for (int p = lrp[i]; p < lrp[i + 1]; ++p) {
            const int k = lci[p];
            if (k >= kmax) break;
            const int q = u_find(urp, uci, k, j);
            if (q >= 0) {
                const T prod = mul_rn(lold[p], uold[q]);
                s = any ? s + prod : prod;
                any = true;
            }
        }
        if (lower) lnew[e] = (al[e] - s) / uold[urp[j]];  // U's diagonal leads row j
        else unew[e] = au[e] - s;
    }
}

// row index of every entry of a CSR pattern
__global__ void ilu_rows_kernel(int64_t n, const int* __restrict__ rp, int* __restrict__ row) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        for (int p = rp[i]; p < rp[i + 1]; ++p) row[p] = (int)i;
}

// ---- sync-free triangular solve ------------------------------------------------
__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <typename T>
__global__ void __launch_bounds__(256)
trs_kernel(int64_t n, const int* __restrict__ rp, const int* __restrict__ ci, const T* __restrict__ v,
           const T* __restrict__ diag, int lower, const T* __restrict__ b, int64_t bs, T* x, int64_t xs,
           int* ready, int epoch, int* ticket) {
    const int lane = threadIdx.x & 31;
    while (true) {
        int t = 0;
        if (lane == 0) t = atomicAdd(ticket, 1);
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= n) return;
        const int i = lower ? t : (int)(n - 1 - t);
        T s = 0;
        for (int p = rp[i] + lane; p < rp[i + 1]; p += 32) {
            const int c = ci[p];
            if (c == i) continue;
            while (ld_acquire(ready + c) != epoch) {
            }
            s += v[p] * __ldcg(x + (int64_t)c * xs);
        }
        s = warp_sum(s);
        if (lane == 0) {
            T xi = b[(int64_t)i * bs] - s;
            if (diag) xi = xi / diag[i];
            x[(int64_t)i * xs] = xi;
            st_release(ready + i, epoch);
        }
    }
}

}  // namespace b200sp

using namespace b200sp;

#define ILU_GRID(n) grid_for((n), 256, 8)

extern "C" {

/* per-row L / U entry counts of A's pattern; *nodiag = first row without a
 * stored diagonal (INT_MAX if none; initialise it to INT_MAX) */
int b200sp_ilu_counts(int64_t n, const int32_t* rp, const int32_t* ci, int32_t* lcnt, int32_t* ucnt,
                      int32_t* nodiag, void* stream) {
    if (n == 0) return B200SP_OK;
    ilu_counts_kernel<<<ILU_GRID(n), 256, 0, as_stream(stream)>>>(n, rp, ci, lcnt, ucnt, nodiag);
    count_launch();
    return check_launch("ilu_counts");
}

int b200sp_csr_rows(int64_t n, const int32_t* rp, int32_t* row, void* stream) {
    if (n == 0) return B200SP_OK;
    ilu_rows_kernel<<<ILU_GRID(n), 256, 0, as_stream(stream)>>>(n, rp, row);
    count_launch();
    return check_launch("csr_rows");
}

#define ILU_T(T, SUF)                                                                                              \
    int b200sp_diag_##SUF(int64_t n, const int32_t* rp, const int32_t* ci, const T* v, T* diag, int32_t* zero,      \
                          void* stream) {                                                                          \
        if (n == 0) return B200SP_OK;                                                                              \
        ilu_diag_kernel<T><<<ILU_GRID(n), 256, 0, as_stream(stream)>>>(n, rp, ci, v, diag, zero);                  \
        count_launch();                                                                                            \
        return check_launch("diag");                                                                               \
    }                                                                                                              \
    int b200sp_ilu_fill_##SUF(int64_t n, const int32_t* rp, const int32_t* ci, const T* v, const T* diag,          \
                              const int32_t* lrp, const int32_t* urp, int32_t* lci, T* al, T* lv, int32_t* uci,    \
                              T* au, T* uv, void* stream) {                                                        \
        if (n == 0) return B200SP_OK;                                                                              \
        ilu_fill_kernel<T><<<ILU_GRID(n), 256, 0, as_stream(stream)>>>(n, rp, ci, v, diag, lrp, urp, lci, al, lv,  \
                                                                       uci, au, uv);                               \
        count_launch();                                                                                            \
        return check_launch("ilu_fill");                                                                           \
    }                                                                                                              \
    int b200sp_parilu_sweep_##SUF(int64_t n, int64_t nl, int64_t nu, const int32_t* lrow, const int32_t* lrp,       \
                                  const int32_t* lci, const T* al, const T* lold, T* lnew, const int32_t* urow,    \
                                  const int32_t* urp, const int32_t* uci, const T* au, const T* uold, T* unew,     \
                                  void* stream) {                                                                  \
        if (nl + nu == 0) return B200SP_OK;                                                                        \
        parilu_sweep_kernel<T><<<ILU_GRID(nl + nu), 256, 0, as_stream(stream)>>>(                                  \
            n, nl, nu, lrow, lrp, lci, al, lold, lnew, urow, urp, uci, au, uold, unew);                            \
        count_launch();                                                                                            \
        return check_launch("parilu_sweep");                                                                       \
    }                                                                                                              \
    int b200sp_trs_##SUF(int64_t n, const int32_t* rp, const int32_t* ci, const T* v, const T* diag,               \
                         int32_t lower, const T* b, int64_t bs, T* x, int64_t xs, int32_t* ready, int32_t epoch,   \
                         int32_t* ticket, void* stream) {                                                          \
        if (n == 0) return B200SP_OK;                                                                              \
        cudaStream_t st = as_stream(stream);                                                                       \
        B200SP_CHECK_CUDA(cudaMemsetAsync(ticket, 0, sizeof(int32_t), st));                                        \
        trs_kernel<T><<<grid_for(n * 32, 256, 8), 256, 0, st>>>(n, rp, ci, v, diag, lower, b, bs, x, xs, ready,    \
                                                               epoch, ticket);                                     \
        count_launch();                                                                                            \
        return check_launch("trs");                                                                                \
    }

ILU_T(double, f64)
ILU_T(float, f32)

}  // extern "C"
