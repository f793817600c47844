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
#include <cooperative_groups.h>

#include <algorithm>
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

// Rows are claimed in `order` (rows grouped by dependency level, from
// b200sp_trs_levels / b200sp_trs_order) when given: consecutive tickets then
// hold independent rows, so the waits are short and warps solve a whole level
// in parallel. Claiming in plain row order (order = NULL) serialises along
// the x-neighbour chain of a stencil (measured: 143 ms per ILU apply at 128^3).
template <typename T>
__global__ void __launch_bounds__(256)
trs_kernel(int64_t n, const int* __restrict__ rp, const int* __restrict__ ci, const T* __restrict__ v,
           const T* __restrict__ diag, int lower, const T* __restrict__ b, int64_t bs, T* x, int64_t xs,
           int* ready, int epoch, int* ticket, const int* __restrict__ order, int per_claim) {
    const int lane = threadIdx.x & 31;
    while (true) {
        // one atomic claims `per_claim` consecutive order positions (a single
        // global counter bumped per row serialises ~1 ns per row), solved by
        // the warp in order
        int t0 = 0;
        if (lane == 0) t0 = atomicAdd(ticket, per_claim);
        t0 = __shfl_sync(0xffffffffu, t0, 0);
        if (t0 >= n) return;
        const int t1 = (int)min((int64_t)t0 + per_claim, n);
        for (int t = t0; t < t1; ++t) {
            const int i = order ? order[t] : (lower ? t : (int)(n - 1 - t));
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
}

// Thread-per-row variant for short rows (triangular stencil factors): a warp
// claims 32 consecutive order positions with one atomic (a single global
// ticket per row was itself the bottleneck: 2M serialised atomics) and every
// lane solves its own row; lanes may wait on rows of the same warp (level
// boundaries), which independent thread scheduling lets progress.
template <typename T>
__global__ void __launch_bounds__(256)
trs_rows_kernel(int64_t n, const int* __restrict__ rp, const int* __restrict__ ci, const T* __restrict__ v,
                const T* __restrict__ diag, int lower, const T* __restrict__ b, int64_t bs, T* x, int64_t xs,
                int* ready, int epoch, int* ticket, const int* __restrict__ order) {
    const int lane = threadIdx.x & 31;
    while (true) {
        int t0 = 0;
        if (lane == 0) t0 = atomicAdd(ticket, 32);
        t0 = __shfl_sync(0xffffffffu, t0, 0);
        if (t0 >= n) return;
        const int64_t t = (int64_t)t0 + lane;
        if (t < n) {
            const int i = order ? order[t] : (lower ? (int)t : (int)(n - 1 - t));
            T s = 0;
            for (int p = rp[i]; p < rp[i + 1]; ++p) {
                const int c = ci[p];
                if (c == i) continue;
                while (ld_acquire(ready + c) != epoch) {
                }
                s += v[p] * __ldcg(x + (int64_t)c * xs);
            }
            T xi = b[(int64_t)i * bs] - s;
            if (diag) xi = xi / diag[i];
            x[(int64_t)i * xs] = xi;
            st_release(ready + i, epoch);
        }
    }
}

// Level-synchronous substitution as ONE cooperative launch: the rows of a
// level are independent, so each thread solves rows of the current level
// (thread per row, no flags, no spinning) and a grid barrier separates the
// levels. Replaces ~5.6 us of flag-polling latency per level of the
// sync-free kernel by one barrier.
template <typename T>
__global__ void __launch_bounds__(512)
trs_coop_kernel(const int* __restrict__ rp, const int* __restrict__ ci, const T* __restrict__ v,
                const T* __restrict__ diag, const T* __restrict__ b, int64_t bs, T* x, int64_t xs,
                const int* __restrict__ order, const int* __restrict__ offs, int nlevels) {
    cooperative_groups::grid_group grid = cooperative_groups::this_grid();
    const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t gs = (int64_t)gridDim.x * blockDim.x;
    for (int lv = 0; lv < nlevels; ++lv) {
        const int64_t s0 = offs[lv], s1 = offs[lv + 1];
        for (int64_t t = s0 + gt; t < s1; t += gs) {
            const int i = order[t];
            T s = 0;
            for (int p = rp[i]; p < rp[i + 1]; ++p) {
                const int c = ci[p];
                if (c != i) s += v[p] * __ldcg(x + (int64_t)c * xs);
            }
            T xi = b[(int64_t)i * bs] - s;
            if (diag) xi = xi / diag[i];
            x[(int64_t)i * xs] = xi;
        }
        if (lv + 1 < nlevels) grid.sync();
    }
}

// one relaxation sweep of the dependency levels: level[i] = 1 + max over
// the row's off-diagonal columns c (c < i for lower, c > i for upper)
__global__ void trs_levels_kernel(int64_t n, const int* __restrict__ rp, const int* __restrict__ ci, int lower,
                                  int* level, int* changed) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int lv = 0;
        for (int p = rp[i]; p < rp[i + 1]; ++p) {
            const int c = ci[p];
            if (lower ? c < i : c > i) lv = max(lv, 1 + ((volatile int*)level)[c]);
        }
        if (lv != level[i]) {
            level[i] = lv;
            *changed = 1;
        }
    }
}

__global__ void trs_level_hist_kernel(int64_t n, const int* __restrict__ level, int* count) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(count + level[i], 1);
}

__global__ void trs_order_kernel(int64_t n, const int* __restrict__ level, const int* __restrict__ offs,
                                 int* cursor, int* order) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int lv = level[i];
        order[offs[lv] + atomicAdd(cursor + lv, 1)] = (int)i;
    }
}

}  // namespace b200sp

using namespace b200sp;

#define ILU_GRID(n) grid_for((n), 256, 8)

template <typename T>
static int trs_coop(int64_t n, const int32_t* rp, const int32_t* ci, const T* v, const T* diag, const T* b, int64_t bs,
                    T* x, int64_t xs, const int32_t* order, const int32_t* offs, int32_t nlevels, void* stream) {
    if (n == 0) return B200SP_OK;
    int dev = 0, sms = 0, per_sm = 0;
    B200SP_CHECK_CUDA(cudaGetDevice(&dev));
    B200SP_CHECK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    B200SP_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, trs_coop_kernel<T>, 512, 0));
    int64_t grid = (int64_t)sms * std::min(per_sm, tuning("trs_coop_per_sm", 1));
    grid = std::max<int64_t>(1, std::min<int64_t>(grid, ceil_div(n, 512)));
    void* args[] = {(void*)&rp, (void*)&ci, (void*)&v, (void*)&diag, (void*)&b, &bs, &x, &xs, (void*)&order,
                    (void*)&offs, &nlevels};
    B200SP_CHECK_CUDA(cudaLaunchCooperativeKernel((const void*)trs_coop_kernel<T>, dim3((unsigned)grid), dim3(512),
                                                  args, 0, as_stream(stream)));
    count_launch();
    return B200SP_OK;
}


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

/* One relaxation sweep of the triangular solve's dependency levels (level
 * zero-initialised by the caller); *changed set when any level moved. The
 * caller repeats until a sweep changes nothing (at most depth + 1 sweeps). */
int b200sp_trs_levels(int64_t n, const int32_t* rp, const int32_t* ci, int32_t lower, int32_t* level,
                      int32_t* changed, void* stream) {
    if (n == 0) return B200SP_OK;
    trs_levels_kernel<<<ILU_GRID(n), 256, 0, as_stream(stream)>>>(n, rp, ci, lower, level, changed);
    count_launch();
    return check_launch("trs_levels");
}

/* rows grouped by level: count (nlevels, zeroed) -> exclusive scan offs ->
 * order (cursor: nlevels, zeroed) */
int b200sp_trs_level_hist(int64_t n, const int32_t* level, int32_t* count, void* stream) {
    if (n == 0) return B200SP_OK;
    trs_level_hist_kernel<<<ILU_GRID(n), 256, 0, as_stream(stream)>>>(n, level, count);
    count_launch();
    return check_launch("trs_level_hist");
}

int b200sp_trs_order(int64_t n, const int32_t* level, const int32_t* offs, int32_t* cursor, int32_t* order,
                     void* stream) {
    if (n == 0) return B200SP_OK;
    trs_order_kernel<<<ILU_GRID(n), 256, 0, as_stream(stream)>>>(n, level, offs, cursor, order);
    count_launch();
    return check_launch("trs_order");
}

int b200sp_trs_coop_f64(int64_t n, const int32_t* rp, const int32_t* ci, const double* v, const double* diag,
                        const double* b, int64_t bs, double* x, int64_t xs, const int32_t* order, const int32_t* offs,
                        int32_t nlevels, void* stream) {
    return trs_coop<double>(n, rp, ci, v, diag, b, bs, x, xs, order, offs, nlevels, stream);
}
int b200sp_trs_coop_f32(int64_t n, const int32_t* rp, const int32_t* ci, const float* v, const float* diag,
                        const float* b, int64_t bs, float* x, int64_t xs, const int32_t* order, const int32_t* offs,
                        int32_t nlevels, void* stream) {
    return trs_coop<float>(n, rp, ci, v, diag, b, bs, x, xs, order, offs, nlevels, stream);
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
                         int32_t* ticket, const int32_t* order, void* stream) {                                    \
        if (n == 0) return B200SP_OK;                                                                              \
        cudaStream_t st = as_stream(stream);                                                                       \
        B200SP_CHECK_CUDA(cudaMemsetAsync(ticket, 0, sizeof(int32_t), st));                                        \
        if (tuning("trs_thread_rows", 0))                                                                          \
            trs_rows_kernel<T><<<grid_for(n, 256, 8), 256, 0, st>>>(n, rp, ci, v, diag, lower, b, bs, x, xs, ready, \
                                                                    epoch, ticket, order);                         \
        else                                                                                                       \
            trs_kernel<T><<<grid_for(n * 32, 256, 8), 256, 0, st>>>(n, rp, ci, v, diag, lower, b, bs, x, xs, ready, \
                                                                   epoch, ticket, order, tuning("trs_per_claim", 1)); \
        count_launch();                                                                                            \
        return check_launch("trs");                                                                                \
    }

ILU_T(double, f64)
ILU_T(float, f32)

}  // extern "C"
