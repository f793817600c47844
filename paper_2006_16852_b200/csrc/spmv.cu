// SpMV kernels for every storage format on the path (sm_100a, HBM-bound).
//
// Semantics shared by all kernels (one right-hand-side column per launch):
//     x[i] = alpha * (A b)[i] + beta * x_in[i]        (x_in may be NULL -> 0)
// which covers LinOp.apply (alpha=1, x_in=NULL; reference src/base.py:60-70),
// apply_advanced (x_in == x; src/base.py:72-82) and the fused residual
// r = b - A x (alpha=-1, beta=1, x_in=b; src/kernels.py:243-275).
//
// Reference kernels these replace (all host NumPy in the reference):
//   Csr  -> CsrSpmvKernel + csr_row_sums     src/kernels.py:278-316
//   Coo  -> CooSpmvKernel / CooAdvSpmvKernel src/kernels.py:163-240
//   Ell / Sellp / Hybrid have no reference kernel; their results
//   are pinned through the format-independent SpMV result.
#include <algorithm>
#include <climits>
#include <cstdint>

#include "common.cuh"

namespace b200sp {

// ===========================================================================
// Csr, classical strategy: one sub-warp of SW lanes per row (SW = 1..32).
// ===========================================================================
// Each sub-warp owns U consecutive rows per step and issues the loads of all
// U rows before any FMA: U x SW independent gathers in flight per sub-warp
// (one row per warp leaves HBM latency exposed: the first B200 measurement of
// the one-row variant reached 32% of peak on C2).
// rows in flight per sub-warp (2 rows per thread at sub-warp 1 strides the
// row accesses of a warp by 2 and measured slower: 0.745 vs 0.748 / CG
// 0.81 vs 0.51 ms; profiles/r02_classical_sweep.txt)
// (ClassicalRows<SW> in common.cuh: shared with the host-stream kernel)

// L1: matrix reads allocate in L1 (a sub-warp touches only part of each
// sector per step; the next steps re-read the rest of it from L1, not L2)
template <typename T> struct Vec2;
template <> struct Vec2<double> { using type = double2; };
template <> struct Vec2<float> { using type = float2; };

// KB > 0 (U = 1): the row's entries in predicated blocks of KB per lane --
// every load of a block is issued before its gathers and no remainder loop
// adds dependent (index -> gather) round trips after the unrolled body (a
// 27-entry row at sub-warp 4 is 7 entries per lane: one block of 4 and one
// of 3 instead of the compiler's pairs plus 2- and 1-entry tails). Same
// single accumulator and entry order as the loop: the same sums.
template <typename T, int SW, bool XIN, bool L1, int U, int KB = 0>
__global__ void __launch_bounds__(256)
csr_classical_kernel(int64_t n, const int* __restrict__ rp, const int* __restrict__ ci,
                     const T* __restrict__ v, const T* __restrict__ b, int64_t bs,
                     T* __restrict__ x, int64_t xs, Coef<T> alpha, Coef<T> beta,
                     const T* __restrict__ xin, int64_t xins) {
    if (alpha.skip()) return;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & (SW - 1);
    const int64_t nsw = (int64_t)gridDim.x * blockDim.x / SW;
    const T a = alpha.get();
    const T bt = XIN ? beta.get() : T(0);
    // loop while the warp's first sub-warp has rows (uniform trip count: the
    // sub-warp shuffles below use the full mask); later sub-warps are masked
    const int64_t wfirst = (tid / 32) * (32 / SW) * U;
    for (int64_t row0 = (tid / SW) * U, w0 = wfirst; w0 < n; row0 += nsw * U, w0 += nsw * U) {
        int s[U], len[U];
        int ptr_next = row0 < n ? ld_stream(rp + row0) : 0;
        int maxlen = 0;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            s[u] = ptr_next;
            ptr_next = (row0 + u < n) ? ld_stream(rp + row0 + u + 1) : ptr_next;
            len[u] = ptr_next - s[u];
            maxlen = max(maxlen, len[u]);
        }
        T acc[U];
#pragma unroll
        for (int u = 0; u < U; ++u) acc[u] = 0;
        if (KB < 0 && U == 1) {
            // entry pairs: lane l reads the 8-byte-aligned pairs (index, value)
            // starting at (s & ~1) + 2 l; entries outside [s, e) are masked
            // (a row's first / last pair may straddle its neighbours)
            constexpr int K = KB < 0 ? -KB : 1;  // pairs per lane per block
            const int s0 = s[0], e0 = s[0] + len[0];
            const int a0 = s0 & ~1;
#pragma unroll 1
            for (int k0 = a0 + 2 * lane; k0 < e0; k0 += 2 * K * SW) {
                int2 c[K];
                typename Vec2<T>::type vv[K];
#pragma unroll
                for (int j = 0; j < K; ++j) {
                    const int k = k0 + j * 2 * SW;
                    if (k < e0) {
                        c[j] = __ldg(reinterpret_cast<const int2*>(ci + k));
                        vv[j] = __ldg(reinterpret_cast<const typename Vec2<T>::type*>(v + k));
                    } else {
                        c[j] = make_int2(-1, -1);
                    }
                }
#pragma unroll
                for (int j = 0; j < K; ++j) {
                    const int k = k0 + j * 2 * SW;
                    if (k >= s0 && c[j].x >= 0) acc[0] += vv[j].x * ld_gather(b + (int64_t)c[j].x * bs);
                    if (k + 1 < e0 && c[j].y >= 0) acc[0] += vv[j].y * ld_gather(b + (int64_t)c[j].y * bs);
                }
            }
        } else if (KB > 0 && U == 1) {
            constexpr int K = KB > 0 ? KB : 1;
#pragma unroll 1
            for (int k0 = lane; k0 < maxlen; k0 += K * SW) {
                int c[K];
                T vv[K];
#pragma unroll
                for (int j = 0; j < K; ++j) {
                    const int k = k0 + j * SW;
                    const bool ok = k < len[0];
                    c[j] = ok ? (L1 ? __ldg(ci + s[0] + k) : ld_stream(ci + s[0] + k)) : -1;
                    vv[j] = ok ? (L1 ? __ldg(v + s[0] + k) : ld_stream(v + s[0] + k)) : T(0);
                }
#pragma unroll
                for (int j = 0; j < K; ++j)
                    if (c[j] >= 0) acc[0] += vv[j] * ld_gather(b + (int64_t)c[j] * bs);
            }
        } else
        for (int k = lane; k < maxlen; k += SW) {
            int c[U];
            T vv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const bool ok = k < len[u];
                c[u] = ok ? (L1 ? __ldg(ci + s[u] + k) : ld_stream(ci + s[u] + k)) : -1;
                vv[u] = ok ? (L1 ? __ldg(v + s[u] + k) : ld_stream(v + s[u] + k)) : T(0);
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (c[u] >= 0) acc[u] += vv[u] * ld_gather(b + (int64_t)c[u] * bs);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc[u] = subwarp_sum<SW>(acc[u]);
        // every lane holds every row's total (xor reduction); row u is
        // written by lane u % SW (U may exceed SW: thread-per-row takes 2)
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t row = row0 + u;
            if (u % SW == lane && row < n) {
                T r = a * acc[u];
                if (XIN) r += bt * xin[row * xins];
                x[row * xs] = r;
            }
        }
    }
}

template <typename T, int SW>
static void launch_classical(int64_t n, const int* rp, const int* ci, const T* v, const T* b,
                             int64_t bs, T* x, int64_t xs, Coef<T> al, Coef<T> be,
                             const T* xin, int64_t xins, bool even_nnz, cudaStream_t st) {
    const int block = 256;
    // measured on B200 (profiles/r02_classical_sweep.txt): L1-allocating
    // matrix loads lift C2 fp64 (sub-warp 4) from 0.43 to 0.85 of the HBM
    // roofline and 7-point (sub-warp 1) from 0.27 to 0.85; two waves of CTAs
    // (the no_allocate build of this kernel is gone; its numbers stay in the
    // sweep file). U = rows in flight per sub-warp: knob "classical_rows" 2
    // doubles it for the narrow sub-warps
    constexpr int U0 = ClassicalRows<SW>::v;
    constexpr int U2 = U0 < 2 ? 2 : U0;
    const bool two = tuning("classical_rows", 0) == 2;
    const int grid = grid_for(ceil_div(n, two ? U2 : U0) * SW, block, tuning("classical_per_sm", 32));
    auto kern = two ? (xin ? csr_classical_kernel<T, SW, true, true, U2> : csr_classical_kernel<T, SW, false, true, U2>)
                    : (xin ? csr_classical_kernel<T, SW, true, true, U0> : csr_classical_kernel<T, SW, false, true, U0>);
    // pair loads need 16-byte aligned arrays and an even entry count (a pair
    // starts at an even entry, so it never reaches past entry nnz - 1)
    const bool pairs_ok = even_nnz && ((reinterpret_cast<uintptr_t>(ci) | reinterpret_cast<uintptr_t>(v)) & 15) == 0;
    if (!two && U0 == 1) {
        // predicated entry blocks (knob "classical_kb": 0 = the loop, 2 / 3 / 4
        // entries per lane per block, -1 / -2 / -4 aligned (index, value) pairs
        // per lane per block). Measured (profiles/r03_classical_kb.txt): pairs
        // in blocks of 2 win for fp32 (27-point 0.715 -> 0.808, 7-point 0.767
        // -> 0.886, 5-point 0.720 -> 0.789) and fp64 thread-per-row (7-point
        // 0.816 -> 0.876); fp64 sub-warp 4 (27-point) keeps 4-entry blocks
        // (0.826, pairs 0.735)
        const int kb = tuning("classical_kb", (sizeof(T) == 4 || SW == 1) ? -2 : 4);
        if (kb == -1 && pairs_ok) kern = xin ? csr_classical_kernel<T, SW, true, true, 1, -1> : csr_classical_kernel<T, SW, false, true, 1, -1>;
        if (kb == -2 && pairs_ok) kern = xin ? csr_classical_kernel<T, SW, true, true, 1, -2> : csr_classical_kernel<T, SW, false, true, 1, -2>;
        if (kb == -4 && pairs_ok) kern = xin ? csr_classical_kernel<T, SW, true, true, 1, -4> : csr_classical_kernel<T, SW, false, true, 1, -4>;
        if (kb == 2) kern = xin ? csr_classical_kernel<T, SW, true, true, 1, 2> : csr_classical_kernel<T, SW, false, true, 1, 2>;
        if (kb == 3) kern = xin ? csr_classical_kernel<T, SW, true, true, 1, 3> : csr_classical_kernel<T, SW, false, true, 1, 3>;
        if (kb == 4) kern = xin ? csr_classical_kernel<T, SW, true, true, 1, 4> : csr_classical_kernel<T, SW, false, true, 1, 4>;
    }
    kern<<<grid, block, 0, st>>>(n, rp, ci, v, b, bs, x, xs, al, be, xin, xins);
}

template <typename T>
static int csr_classical(int64_t n, const int* rp, const int* ci, const T* v, const T* b, int64_t bs,
                         T* x, int64_t xs, T alpha, const T* alpha_dev, T beta, const T* beta_dev,
                         const T* xin, int64_t xins, int subwarp, void* stream) {
    if (n == 0) return B200SP_OK;
    cudaStream_t st = as_stream(stream);
    Coef<T> al = coef(alpha, alpha_dev), be = coef(beta, beta_dev);
    const bool ev = (subwarp & B200SP_SUBWARP_EVEN_NNZ) != 0;  // caller: the matrix has an even entry count
    subwarp &= ~B200SP_SUBWARP_EVEN_NNZ;
    switch (subwarp) {
        case 1: launch_classical<T, 1>(n, rp, ci, v, b, bs, x, xs, al, be, xin, xins, ev, st); break;
        case 2: launch_classical<T, 2>(n, rp, ci, v, b, bs, x, xs, al, be, xin, xins, ev, st); break;
        case 4: launch_classical<T, 4>(n, rp, ci, v, b, bs, x, xs, al, be, xin, xins, ev, st); break;
        case 8: launch_classical<T, 8>(n, rp, ci, v, b, bs, x, xs, al, be, xin, xins, ev, st); break;
        case 16: launch_classical<T, 16>(n, rp, ci, v, b, bs, x, xs, al, be, xin, xins, ev, st); break;
        case 32: launch_classical<T, 32>(n, rp, ci, v, b, bs, x, xs, al, be, xin, xins, ev, st); break;
        default: set_error("csr classical: subwarp must be a power of two <= 32 (got %d)", subwarp);
                 return B200SP_EINVAL;
    }
    count_launch();
    return check_launch("csr_classical");
}

// ===========================================================================
// Csr, stream strategy (row blocks staged through shared memory).
// A CTA of R threads owns R consecutive rows. Their nonzeros are one
// contiguous range; it is streamed in chunks of STREAM_CAP entries with
// 128-bit loads (4 entries per thread per step, all independent), the
// products v*b[c] go to shared memory, and thread t then sums row t from
// shared memory. Every global load is coalesced and vectorised and no warp
// reduction is needed -- the instruction count per nonzero is close to Ell's
// while keeping the Csr layout. Rows longer than a chunk are handled by
// accumulating across chunks (correct, but serial: skewed matrices use the
// load-balanced strategy).
// ===========================================================================
template <typename T> struct StreamCap { static constexpr int v = 8192; };  // 64 KB / 32 KB of smem

template <typename T> struct Quad;
template <> struct Quad<double> {
    __device__ static void load(const double* p, double (&o)[4]) {
        double2 a = ld_stream_v2(p), b = ld_stream_v2(p + 2);
        o[0] = a.x; o[1] = a.y; o[2] = b.x; o[3] = b.y;
    }
    __device__ static void store(double* s, const double (&o)[4]) {
        reinterpret_cast<double2*>(s)[0] = make_double2(o[0], o[1]);
        reinterpret_cast<double2*>(s)[1] = make_double2(o[2], o[3]);
    }
};
template <> struct Quad<float> {
    __device__ static void load(const float* p, float (&o)[4]) {
        float4 a = ld_stream_v4(p);
        o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w;
    }
    __device__ static void store(float* s, const float (&o)[4]) {
        reinterpret_cast<float4*>(s)[0] = make_float4(o[0], o[1], o[2], o[3]);
    }
};

// Shape of a CTA (256 threads): TPR threads share a row in the reduction and
// each thread group reduces RPT rows, so a CTA owns (256 / TPR) * RPT rows.
// Long rows (27-point) use TPR = 2; short rows (5/7-point) use RPT > 1 so a
// CTA still streams thousands of nonzeros per staging chunk.
constexpr int STREAM_NT = 256;

// GR ("gather in reduce"): stage (col, val) instead of products and gather x
// in the thread-per-row reduction, where the lanes of a warp walk consecutive
// rows -- for banded matrices those gathers are coalesced, while gathers in
// the staging phase touch ~10 lines per warp instruction and saturate the
// L1TEX LSU pipe (ncu: 85-94% busy at 47% DRAM, profiles/r01_ncu_c2_stream.txt).
template <typename T, int TPR, int RPT, bool XIN, bool GR>
__global__ void __launch_bounds__(STREAM_NT)
csr_stream_kernel(int64_t n, int64_t nnz, const int* __restrict__ rp, const int* __restrict__ ci,
                  const T* __restrict__ v, const T* __restrict__ b, int64_t bs, T* __restrict__ x,
                  int64_t xs, Coef<T> alpha, Coef<T> beta, const T* __restrict__ xin, int64_t xins,
                  int CAP) {
    if (alpha.skip()) return;
    constexpr int NT = STREAM_NT;
    constexpr int G = NT / TPR;  // thread groups (rows reduced concurrently)
    constexpr int R = G * RPT;
    // quads per thread in flight per step; 4 measured worse (79 registers ->
    // lower occupancy; profiles/r01_stream_sweep.txt)
    constexpr int UQ = 2;
    extern __shared__ __align__(16) unsigned char s_raw[];
    T* s_prod = reinterpret_cast<T*>(s_raw);
    int* s_ci = reinterpret_cast<int*>(s_raw);                             // GR only
    T* s_v = reinterpret_cast<T*>(s_raw + (size_t)CAP * sizeof(int));      // GR only
    const int t = threadIdx.x;
    const int grp = t / TPR, sub = t % TPR;
    const int64_t r0 = (int64_t)blockIdx.x * R;
    const int rows = (int)min((int64_t)R, n - r0);
    int row_s[RPT], row_e[RPT];
#pragma unroll
    for (int k = 0; k < RPT; ++k) {
        const int lr = grp + k * G;
        row_s[k] = lr < rows ? ld_stream(rp + r0 + lr) : 0;
        row_e[k] = lr < rows ? ld_stream(rp + r0 + lr + 1) : 0;
    }
    const int seg_s = ld_stream(rp + r0);
    const int seg_e = ld_stream(rp + r0 + rows);
    T acc[RPT];
#pragma unroll
    for (int k = 0; k < RPT; ++k) acc[k] = 0;
    for (int64_t lo = seg_s & ~3; lo < seg_e; lo += CAP) {
        const int64_t hi = min(lo + (int64_t)CAP, (int64_t)seg_e);
        const int nq = (int)((hi - lo + 3) >> 2);
        for (int q0 = t; q0 < nq; q0 += NT * UQ) {
            int cc[UQ][4];
            T vv[UQ][4];
#pragma unroll
            for (int u = 0; u < UQ; ++u) {
                const int q = q0 + u * NT;
                const int64_t e = lo + 4 * (int64_t)q;
                if (q < nq && e + 4 <= hi) {
                    int4 c4 = ld_stream_v4(ci + e);
                    cc[u][0] = c4.x; cc[u][1] = c4.y; cc[u][2] = c4.z; cc[u][3] = c4.w;
                    Quad<T>::load(v + e, vv[u]);
                } else {
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const bool ok = q < nq && e + i < hi;
                        cc[u][i] = ok ? ld_stream(ci + e + i) : 0;
                        vv[u][i] = ok ? ld_stream(v + e + i) : T(0);
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < UQ; ++u) {
                const int q = q0 + u * NT;
                if (q < nq) {
                    if (GR) {
                        reinterpret_cast<int4*>(s_ci)[q] = make_int4(cc[u][0], cc[u][1], cc[u][2], cc[u][3]);
                        Quad<T>::store(s_v + 4 * q, vv[u]);
                    } else {
                        T p[4];
#pragma unroll
                        for (int i = 0; i < 4; ++i) p[i] = vv[u][i] * ld_gather(b + (int64_t)cc[u][i] * bs);
                        Quad<T>::store(s_prod + 4 * q, p);
                    }
                }
            }
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
            const int a0 = (int)(max((int64_t)row_s[r], lo) - lo), a1 = (int)(min((int64_t)row_e[r], hi) - lo);
            T s0 = 0, s1 = 0;
            int k = a0 + sub;
            if (GR) {
                T s2 = 0, s3 = 0;
                for (; k + 3 * TPR < a1; k += 4 * TPR) {
                    const int c0 = s_ci[k], c1 = s_ci[k + TPR], c2 = s_ci[k + 2 * TPR], c3 = s_ci[k + 3 * TPR];
                    s0 += s_v[k] * ld_gather(b + (int64_t)c0 * bs);
                    s1 += s_v[k + TPR] * ld_gather(b + (int64_t)c1 * bs);
                    s2 += s_v[k + 2 * TPR] * ld_gather(b + (int64_t)c2 * bs);
                    s3 += s_v[k + 3 * TPR] * ld_gather(b + (int64_t)c3 * bs);
                }
                if (k < a1) {  // the rest (< 4) as one predicated block, gathers in flight together
                    T t[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int ki = k + i * TPR;
                        t[i] = ki < a1 ? s_v[ki] * ld_gather(b + (int64_t)s_ci[ki] * bs) : T(0);
                    }
                    s0 += t[0];
                    s1 += t[1];
                    s2 += t[2];
                    s3 += t[3];
                }
                s0 += s2;
                s1 += s3;
            } else {
                for (; k + TPR < a1; k += 2 * TPR) {
                    s0 += s_prod[k];
                    s1 += s_prod[k + TPR];
                }
                if (k < a1) s0 += s_prod[k];
            }
            acc[r] += s0 + s1;
        }
        __syncthreads();
    }
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
        const T sum = subwarp_sum<TPR>(acc[r]);
        const int lr = grp + r * G;
        if (sub == 0 && lr < rows) {
            const int64_t row = r0 + lr;
            T out = alpha.get() * sum;
            if (XIN) out += beta.get() * xin[row * xins];
            x[row * xs] = out;
        }
    }
}

template <typename T, int TPR, int RPT, bool GR>
static void launch_stream(int64_t n, int64_t nnz, const int* rp, const int* ci, const T* v, const T* b,
                          int64_t bs, T* x, int64_t xs, Coef<T> al, Coef<T> be, const T* xin, int64_t xins,
                          int cap, cudaStream_t st) {
    const unsigned grid = (unsigned)ceil_div(n, (STREAM_NT / TPR) * RPT);
    const size_t per = GR ? sizeof(int) + sizeof(T) : sizeof(T);
    const size_t smem = (size_t)cap * per;
    static bool attr_set = false;  // > 48 KB dynamic shared memory needs an opt-in
    if (!attr_set) {
        const int maxb = StreamCap<T>::v * (int)per;
        cudaFuncSetAttribute(csr_stream_kernel<T, TPR, RPT, true, GR>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxb);
        cudaFuncSetAttribute(csr_stream_kernel<T, TPR, RPT, false, GR>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxb);
        attr_set = true;
    }
    if (xin)
        csr_stream_kernel<T, TPR, RPT, true, GR><<<grid, STREAM_NT, smem, st>>>(n, nnz, rp, ci, v, b, bs, x, xs, al, be, xin, xins, cap);
    else
        csr_stream_kernel<T, TPR, RPT, false, GR><<<grid, STREAM_NT, smem, st>>>(n, nnz, rp, ci, v, b, bs, x, xs, al, be, xin, xins, cap);
}

template <typename T>
static int csr_stream(int64_t n, int64_t nnz, const int* rp, const int* ci, const T* v, const T* b,
                      int64_t bs, T* x, int64_t xs, T alpha, const T* alpha_dev, T beta,
                      const T* beta_dev, const T* xin, int64_t xins, int chunk_cap, int tpr, int rpt, int gr,
                      void* stream) {
    if (n == 0) return B200SP_OK;
    B200SP_REQUIRE(aligned16(ci) && aligned16(v), B200SP_EINVAL, "csr stream: col_idxs/vals must be 16-byte aligned");
    B200SP_REQUIRE(chunk_cap >= 4 && chunk_cap % 4 == 0 && chunk_cap <= StreamCap<T>::v, B200SP_EINVAL,
                   "csr stream: chunk_cap must be a multiple of 4 in [4, %d]", StreamCap<T>::v);
    cudaStream_t st = as_stream(stream);
    Coef<T> al = coef(alpha, alpha_dev), be = coef(beta, beta_dev);
#define STREAM_CASE(TP, RP)                                                                                   \
    if (tpr == TP && rpt == RP) {                                                                             \
        if (gr)                                                                                               \
            launch_stream<T, TP, RP, true>(n, nnz, rp, ci, v, b, bs, x, xs, al, be, xin, xins, chunk_cap, st); \
        else                                                                                                  \
            launch_stream<T, TP, RP, false>(n, nnz, rp, ci, v, b, bs, x, xs, al, be, xin, xins, chunk_cap, st); \
        count_launch();                                                                                       \
        return check_launch("csr_stream");                                                                    \
    }
    STREAM_CASE(1, 1) STREAM_CASE(2, 1) STREAM_CASE(4, 1) STREAM_CASE(1, 2) STREAM_CASE(1, 4) STREAM_CASE(1, 8)
#undef STREAM_CASE
    set_error("csr stream: unsupported (threads per row, rows per thread) = (%d, %d)", tpr, rpt);
    return B200SP_EINVAL;
}

// ===========================================================================
// Csr, stream strategy as a persistent TMA pipeline ("pipe").
// One CTA per SM = 8 consumer warps + 1 producer warp. The matrix is cut into
// tiles of TR = 256 * RPT consecutive rows; CTA c takes tiles c, c + grid, ...
// (neighbouring tiles run concurrently on different SMs, so the x window they
// gather from stays L2-resident). The producer lane bulk-copies each tile's
// row_ptrs slice and its contiguous col_idxs / vals range into a STAGES-deep
// ring of shared-memory stages (cp.async.bulk, completion on a `full`
// mbarrier); consumers sum thread-per-row straight out of shared memory (lanes
// = consecutive rows, so the x gathers of one warp instruction are coalesced
// for banded matrices) and hand the stage back through an `empty` mbarrier.
// No load/store instruction is spent staging the matrix -- the previous
// register-staged kernel was L1TEX-LSU bound (ncu 85-94% busy) -- and the next
// tiles stream in while the current one is reduced. A tile whose nonzeros
// exceed one stage (long rows) is consumed in several chunks, rows
// accumulating across them.
// ===========================================================================
constexpr int PIPE_BAR_BYTES = 256;          // mbarriers at the front of smem

__host__ __device__ constexpr int pipe_rp_slots(int tr) { return (tr + 1 + 3) / 4 * 4; }

template <typename T>
__host__ __device__ inline int64_t pipe_stage_bytes(int tr, int cap) {
    return (int64_t)pipe_rp_slots(tr) * 4 + (int64_t)cap * (4 + (int64_t)sizeof(T));
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <typename T, int NT, int TPR, int RPT, bool XIN>
__global__ void __launch_bounds__(NT + 32, 1)
csr_pipe_kernel(int64_t n, const int* __restrict__ rp, const int* __restrict__ ci, const T* __restrict__ v,
                const T* __restrict__ b, int64_t bs, T* __restrict__ x, int64_t xs, Coef<T> alpha, Coef<T> beta,
                const T* __restrict__ xin, int64_t xins, int CAP, int STAGES) {
    if (alpha.skip()) return;
    constexpr int G = NT / TPR;  // rows reduced concurrently (TPR threads each)
    constexpr int TR = G * RPT;  // rows per tile
    constexpr int RPS = pipe_rp_slots(TR);
    extern __shared__ __align__(16) unsigned char s_raw[];
    uint64_t* full = reinterpret_cast<uint64_t*>(s_raw);
    uint64_t* empty = full + STAGES;
    unsigned char* stages = s_raw + PIPE_BAR_BYTES;
    const int64_t SB = pipe_stage_bytes<T>(TR, CAP);
    const int t = threadIdx.x;
    const int64_t ntiles = (n + TR - 1) / TR;
    if (t == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NT / 32);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (t >= NT) {  // ---- producer warp
        // The segment bounds of the next 32 tiles are fetched by the 32 lanes
        // at once (one exposed row_ptrs latency per 32 tiles instead of one per
        // tile); lane 0 then issues every copy.
        const int lane = t - NT;
        const int64_t stride = gridDim.x;
        int it = 0;
        for (int64_t base = blockIdx.x; base < ntiles; base += 32 * stride) {
            const int64_t mine = base + lane * stride;
            int my_s = 0, my_e = 0;
            if (mine < ntiles) {
                my_s = __ldg(rp + mine * TR);
                my_e = __ldg(rp + min(mine * TR + TR, n));
            }
            const int batch = (int)min((int64_t)32, (ntiles - base + stride - 1) / stride);
            for (int j = 0; j < batch; ++j) {
                const int64_t seg_s = __shfl_sync(0xffffffffu, my_s, j);
                const int64_t seg_e = __shfl_sync(0xffffffffu, my_e, j);
                if (lane == 0) {
                    const int64_t r0 = (base + j * stride) * TR;
                    const int64_t lo0 = seg_s & ~(int64_t)3;
                    const int nch = max(1, (int)((seg_e - lo0 + CAP - 1) / CAP));
                    const int rpc = (int)min((int64_t)RPS, (n + 1 - r0) & ~(int64_t)3);
                    for (int c = 0; c < nch; ++c, ++it) {
                        const int s = it % STAGES;
                        if (it >= STAGES) mbar_wait(&empty[s], (uint32_t)(((it / STAGES) - 1) & 1));
                        const int64_t lo = lo0 + (int64_t)c * CAP;
                        const int64_t hi = min(lo + (int64_t)CAP, seg_e);
                        const uint32_t cnt = (uint32_t)(max(hi - lo, (int64_t)0) & ~(int64_t)3);
                        unsigned char* st = stages + s * SB;
                        mbar_arrive_expect_tx(&full[s], (uint32_t)rpc * 4u + cnt * (uint32_t)(4 + sizeof(T)));
                        tma_load_1d(st, rp + r0, (uint32_t)rpc * 4u, &full[s]);
                        if (cnt) {
                            tma_load_1d(st + RPS * 4, ci + lo, cnt * 4u, &full[s]);
                            tma_load_1d(st + RPS * 4 + (int64_t)CAP * 4, v + lo, cnt * (uint32_t)sizeof(T), &full[s]);
                        }
                    }
                }
                __syncwarp();
            }
        }
        return;
    }

    // ---- consumers: the TPR threads of group g reduce rows g, g + G, ... of
    // each tile (entries interleaved across the group)
    const int lane = t & 31;
    const int grp = t / TPR, sub = t % TPR;
    int it = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t r0 = tile * TR;
        const int rows = (int)min((int64_t)TR, n - r0);
        const int rpc = (int)min((int64_t)RPS, (n + 1 - r0) & ~(int64_t)3);
        T acc[RPT];
        int rs[RPT], re[RPT];
#pragma unroll
        for (int k = 0; k < RPT; ++k) acc[k] = 0;
        int nch = 1;
        int64_t lo0 = 0, seg_e = 0;
        for (int c = 0; c < nch; ++c, ++it) {
            const int s = it % STAGES;
            mbar_wait(&full[s], (uint32_t)((it / STAGES) & 1));
            const unsigned char* st = stages + s * SB;
            const int* srp = reinterpret_cast<const int*>(st);
            const int* sci = reinterpret_cast<const int*>(st + RPS * 4);
            const T* sv = reinterpret_cast<const T*>(st + RPS * 4 + (int64_t)CAP * 4);
            if (c == 0) {
                const int64_t seg_s = srp[0];
                seg_e = rows < rpc ? srp[rows] : __ldg(rp + r0 + rows);
                lo0 = seg_s & ~(int64_t)3;
                nch = max(1, (int)((seg_e - lo0 + CAP - 1) / CAP));
#pragma unroll
                for (int k = 0; k < RPT; ++k) {
                    const int lr = grp + k * G;
                    rs[k] = lr < rows ? (lr < rpc ? srp[lr] : __ldg(rp + r0 + lr)) : 0;
                    re[k] = lr < rows ? (lr + 1 < rpc ? srp[lr + 1] : __ldg(rp + r0 + lr + 1)) : 0;
                }
            }
            const int64_t lo = lo0 + (int64_t)c * CAP;
            const int64_t hi = min(lo + (int64_t)CAP, seg_e);
            const int64_t hia = lo + (max(hi - lo, (int64_t)0) & ~(int64_t)3);
            int e[RPT], ee[RPT];
#pragma unroll
            for (int k = 0; k < RPT; ++k) {
                e[k] = (int)(max((int64_t)rs[k], lo) - lo) + sub;
                ee[k] = (int)(max(min((int64_t)re[k], hia), lo) - lo);
            }
            // 8 independent smem reads + x gathers in flight per row step
#pragma unroll
            for (int k = 0; k < RPT; ++k) {
                int q = e[k];
                const int qe = ee[k];
                T s0 = 0, s1 = 0, s2 = 0, s3 = 0;
                for (; q + 7 * TPR < qe; q += 8 * TPR) {
                    int cc[8];
                    T vv[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) cc[i] = sci[q + i * TPR];
#pragma unroll
                    for (int i = 0; i < 8; ++i) vv[i] = sv[q + i * TPR] * ld_gather(b + (int64_t)cc[i] * bs);
                    s0 += vv[0] + vv[4];
                    s1 += vv[1] + vv[5];
                    s2 += vv[2] + vv[6];
                    s3 += vv[3] + vv[7];
                }
                // the rest (< 8 per thread) as one predicated block: all its
                // gathers in flight together, no dependent remainder loop
                // (27-point fp64 0.725 -> 0.767, 7-point 0.30 -> 0.46;
                // profiles/r03_pipe_sweep.txt)
                if (q < qe) {
                    T vv[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const int qi = q + i * TPR;
                        vv[i] = qi < qe ? sv[qi] * ld_gather(b + (int64_t)sci[qi] * bs) : T(0);
                    }
                    s0 += vv[0] + vv[4];
                    s1 += vv[1] + vv[5];
                    s2 += vv[2] + vv[6];
                    s3 += vv[3] + vv[7];
                }
                acc[k] += (s0 + s1) + (s2 + s3);
            }
            if (sub == 0) {
#pragma unroll
                for (int k = 0; k < RPT; ++k)  // the <= 3 entries past the last bulk-copied quad of the segment
                    for (int64_t g = max((int64_t)rs[k], hia); g < min((int64_t)re[k], hi); ++g)
                        acc[k] += ld_stream(v + g) * ld_gather(b + (int64_t)ld_stream(ci + g) * bs);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
#pragma unroll
        for (int k = 0; k < RPT; ++k) {
            const T sum = subwarp_sum<TPR>(acc[k]);
            const int lr = grp + k * G;
            if (sub == 0 && lr < rows) {
                const int64_t row = r0 + lr;
                T out = alpha.get() * sum;
                if (XIN) out += beta.get() * xin[row * xins];
                x[row * xs] = out;
            }
        }
    }
}

template <typename T, int NT, int TPR, int RPT>
static int launch_pipe(int64_t n, const int* rp, const int* ci, const T* v, const T* b, int64_t bs, T* x,
                       int64_t xs, Coef<T> al, Coef<T> be, const T* xin, int64_t xins, int cap, int stages,
                       cudaStream_t st) {
    constexpr int TR = NT / TPR * RPT;
    const int64_t smem = PIPE_BAR_BYTES + (int64_t)stages * pipe_stage_bytes<T>(TR, cap);
    B200SP_REQUIRE(smem <= 226 * 1024, B200SP_EINVAL,
                   "csr pipe: %d stages x %d entries need %lld bytes of shared memory (> 226 KB)", stages, cap,
                   (long long)smem);
    auto kern = xin ? csr_pipe_kernel<T, NT, TPR, RPT, true> : csr_pipe_kernel<T, NT, TPR, RPT, false>;
    B200SP_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int64_t ntiles = ceil_div(n, TR);
    // CTAs per SM: 2 when two stage rings fit (more consumer warps to hide
    // the gather latency), knob "pipe_ctas" to force
    const int per_sm = tuning("pipe_ctas", smem * 2 <= 226 * 1024 ? 2 : 1);
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)kNumSMs * per_sm));
    kern<<<grid, NT + 32, (size_t)smem, st>>>(n, rp, ci, v, b, bs, x, xs, al, be, xin, xins, cap, stages);
    return B200SP_OK;
}

template <typename T>
static int csr_pipe(int64_t n, const int* rp, const int* ci, const T* v, const T* b, int64_t bs, T* x, int64_t xs,
                    T alpha, const T* alpha_dev, T beta, const T* beta_dev, const T* xin, int64_t xins, int cap,
                    int rpt, int stages, int consumers, int tpr, void* stream) {
    if (n == 0) return B200SP_OK;
    B200SP_REQUIRE(aligned16(rp) && aligned16(ci) && aligned16(v), B200SP_EINVAL,
                   "csr pipe: row_ptrs/col_idxs/vals must be 16-byte aligned");
    B200SP_REQUIRE(cap >= 16 && cap % 4 == 0, B200SP_EINVAL, "csr pipe: stage capacity must be a multiple of 4, >= 16");
    B200SP_REQUIRE(stages >= 2 && stages <= 16, B200SP_EINVAL, "csr pipe: stages must be in [2, 16]");
    cudaStream_t st = as_stream(stream);
    Coef<T> al = coef(alpha, alpha_dev), be = coef(beta, beta_dev);
    int rc;
#define PIPE_CASE(NT, TP, RP)                                                                                     \
    if (consumers == NT && tpr == TP && rpt == RP)                                                                \
        rc = launch_pipe<T, NT, TP, RP>(n, rp, ci, v, b, bs, x, xs, al, be, xin, xins, cap, stages, st); \
    else
    PIPE_CASE(256, 1, 1) PIPE_CASE(256, 1, 2) PIPE_CASE(256, 1, 4) PIPE_CASE(256, 2, 1) PIPE_CASE(256, 2, 2)
    PIPE_CASE(512, 2, 1) PIPE_CASE(512, 2, 2)
    PIPE_CASE(512, 4, 1) PIPE_CASE(512, 4, 2) {
        set_error("csr pipe: unsupported (consumer threads, threads per row, rows per thread) = (%d, %d, %d)",
                  consumers, tpr, rpt);
        return B200SP_EINVAL;
    }
#undef PIPE_CASE
    if (rc != B200SP_OK) return rc;
    count_launch();
    return check_launch("csr_pipe");
}

// ===========================================================================
// Csr, load-balanced strategy: merge-path decomposition (Merrill & Garland).
// The merge of the row-end offsets rp[1..n] with the nonzero indices 0..nnz-1
// is cut into equal tiles of merge items; a CTA reduces its tile's rows
// (mode 2, below), and the partial row straddling each tile end is carried
// out and added by a deterministic fix-up pass. Work per CTA is bounded
// regardless of row-length skew. (Round 1's item-level merge through shared
// memory, "mode 1", measured slower on every matrix -- C2 0.43, C3 497 us --
// and was removed: profiles/r02_lb_coo_sweep.txt.)
// ===========================================================================
constexpr int LB_BLOCK = 256;

// merge items (rows + nonzeros) per tile of mode 2: 16384 (measured best of
// 2K/8K/16K on the stencils; knob "lb_tile")
inline int lb_tile() { return tuning("lb_tile", 16384); }

// merge-path search: returns number of row-end items (rows) consumed at `diag`
__device__ __forceinline__ int64_t merge_search_global(int64_t diag, const int* rp, int64_t n,
                                                       int64_t nnz) {
    int64_t lo = diag > nnz ? diag - nnz : 0;
    int64_t hi = diag < n ? diag : n;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        // row-end of row `mid` is rp[mid+1]; compare with nonzero index diag-mid-1
        if ((int64_t)rp[mid + 1] <= diag - mid - 1) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__global__ void csr_lb_plan_kernel(int64_t n, int64_t nnz, const int* __restrict__ rp,
                                   int64_t ntiles, int tile, int* __restrict__ coords) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t > ntiles) return;
    int64_t diag = t * (int64_t)tile;
    if (diag > n + nnz) diag = n + nnz;
    int64_t r = merge_search_global(diag, rp, n, nnz);
    coords[2 * t] = (int)r;
    coords[2 * t + 1] = (int)(diag - r);
}

// deterministic fix-up: the first tile of each run of equal carry rows adds the
// whole run (tiles are in row order, so equal rows are adjacent)
template <typename T>
__global__ void csr_lb_fixup_kernel(int64_t n, int64_t ntiles, const int* __restrict__ carry_row,
                                    const T* __restrict__ carry_val, T* __restrict__ x, int64_t xs,
                                    Coef<T> alpha) {
    if (alpha.skip()) return;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= ntiles) return;
    const int row = carry_row[t];
    if (row >= n) return;
    if (t > 0 && carry_row[t - 1] == row) return;
    T sum = carry_val[t];
    for (int64_t u = t + 1; u < ntiles && carry_row[u] == row; ++u) sum += carry_val[u];
    x[(int64_t)row * xs] += alpha.get() * sum;
}

// ---------------------------------------------------------------------------
// Load-balanced strategy, row-parallel tile processing ("lb2"). Same
// merge-path tiles and carry fix-up as above, but a CTA processes its tile's
// rows directly from global memory like the classical kernel (sub-warp per
// row with L1-allocating loads; the sub-warp width follows the tile's mean
// row length), instead of staging products and merging item by item. Rows of
// the tile longer than LB2_LONG entries and the carried-out last row are
// reduced by the whole CTA. Rows whose start precedes the tile are clipped
// to the tile's first nonzero (the fix-up adds the earlier tiles' carries).
// ---------------------------------------------------------------------------
constexpr int LB2_LONG = 16;  // x sub-warp width: longer rows take the CTA-wide pass

// rows [r0, r_end) of a tile; row rc (the tile's carried-out last row, or
// -1) ends at the tile's last entry kc and its partial sum goes to *s_carry
// for the fix-up instead of x -- it is just one more row of the loop, so no
// warp-0 epilogue holds the CTA's slot after the other warps are done
template <typename T, int SW, bool XIN, bool UNR4>
__device__ __forceinline__ void lb2_rows(int r0, int r_end, int k0, int rc, int kc, const int* __restrict__ rp,
                                         const int* __restrict__ ci, const T* __restrict__ v,
                                         const T* __restrict__ b, int64_t bs, T* __restrict__ x, int64_t xs,
                                         T a, T bt, const T* __restrict__ xin, int64_t xins, int* s_long,
                                         int* s_nlong, T* s_carry) {
    const int lane = threadIdx.x & (SW - 1);
    constexpr int SPW = 32 / SW;  // sub-warps per warp
    // the trip count is uniform across a warp (the sub-warp shuffles use the
    // full mask); rows past r_end are masked
#pragma unroll 1
    for (int rb = r0 + (threadIdx.x >> 5) * SPW; rb < r_end; rb += LB_BLOCK / SW) {
        const int row = rb + (threadIdx.x & 31) / SW;
        const bool active = row < r_end;
        int s = 0, e = 0;
        if (active) {
            s = max(__ldg(rp + row), k0);
            e = row == rc ? kc : __ldg(rp + row + 1);
        }
        const bool lng = e - s > LB2_LONG * SW;
        if (lng) {  // deferred to the CTA-wide pass
            if (lane == 0) s_long[atomicAdd(s_nlong, 1)] = row;
            e = s;
        }
        T a0 = 0, a1 = 0, a2 = 0, a3 = 0;
        if (UNR4) {
            // predicated blocks of 4 entries per lane: every load of a block
            // in flight together, no dependent remainder loop
#pragma unroll 1
            for (int k = s + lane; k < e; k += 4 * SW) {
                int c[4];
                T vv[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const bool ok = k + j * SW < e;
                    c[j] = ok ? __ldg(ci + k + j * SW) : -1;
                    vv[j] = ok ? __ldg(v + k + j * SW) : T(0);
                }
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (c[j] >= 0) a0 += vv[j] * ld_gather(b + (int64_t)c[j] * bs);
            }
        } else {
            for (int k = s + lane; k < e; k += SW) {
                int c0 = __ldg(ci + k);
                a0 += __ldg(v + k) * ld_gather(b + (int64_t)c0 * bs);
            }
        }
        const T sum = subwarp_sum<SW>((a0 + a1) + (a2 + a3));
        if (active && !lng && lane == 0) {
            if (row == rc) {
                *s_carry = sum;
            } else {
                T out = a * sum;
                if (XIN) out += bt * xin[(int64_t)row * xins];
                x[(int64_t)row * xs] = out;
            }
        }
    }
}

// CTA-wide sum of entries [s, e) (result valid in thread 0)
template <typename T>
__device__ __forceinline__ T lb2_block_dot(int s, int e, const int* __restrict__ ci, const T* __restrict__ v,
                                           const T* __restrict__ b, int64_t bs, T* sh) {
    T a0 = 0, a1 = 0;
    int k = s + threadIdx.x;
    for (; k + LB_BLOCK < e; k += 2 * LB_BLOCK) {
        const int c0 = __ldg(ci + k), c1 = __ldg(ci + k + LB_BLOCK);
        a0 += __ldg(v + k) * ld_gather(b + (int64_t)c0 * bs);
        a1 += __ldg(v + k + LB_BLOCK) * ld_gather(b + (int64_t)c1 * bs);
    }
    if (k < e) a0 += __ldg(v + k) * ld_gather(b + (int64_t)__ldg(ci + k) * bs);
    return block_sum(a0 + a1, sh);
}

template <typename T, bool XIN, bool UNR4>
__global__ void __launch_bounds__(LB_BLOCK)
csr_lb2_kernel(int64_t n, int64_t ntiles, const int* __restrict__ rp, const int* __restrict__ ci, const T* __restrict__ v,
               const T* __restrict__ b, int64_t bs, T* __restrict__ x, int64_t xs, Coef<T> alpha, Coef<T> beta,
               const T* __restrict__ xin, int64_t xins, const int* __restrict__ coords, int* __restrict__ carry_row,
               T* __restrict__ carry_val) {
    if (alpha.skip()) return;
    __shared__ int s_long[LB_BLOCK];
    __shared__ int s_nlong;
    __shared__ T s_red[LB_BLOCK / 32];
    __shared__ T s_carry;
    const T a = alpha.get();
    const T bt = XIN ? beta.get() : T(0);
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int r0 = coords[2 * tile], k0 = coords[2 * tile + 1];
        const int r1 = coords[2 * tile + 2], k1 = coords[2 * tile + 3];
        if (threadIdx.x == 0) {
            s_nlong = 0;
            s_carry = T(0);
        }
        __syncthreads();
        // rows r0 .. r1 - 1, plus the carried-out row r1 (its entries before k1)
        const int rc = r1 < n ? r1 : -1;
        const int r_end = rc >= 0 ? r1 + 1 : r1;
        const int nrows = r_end - r0;
        if (nrows > 0) {
            // sub-warp width from the tile's mean row length (classical rule)
            const int mean = (k1 - k0 + nrows - 1) / nrows;
            const int per_lane = (mean + 7) / 8;
#define LB2_ROWS(SW) lb2_rows<T, SW, XIN, UNR4>(r0, r_end, k0, rc, k1, rp, ci, v, b, bs, x, xs, a, bt, xin, xins, \
                                                  s_long, &s_nlong, &s_carry)
            if (per_lane <= 1) { LB2_ROWS(1); }
            else if (per_lane <= 2) { LB2_ROWS(2); }
            else if (per_lane <= 4) { LB2_ROWS(4); }
            else if (per_lane <= 8) { LB2_ROWS(8); }
            else if (per_lane <= 16) { LB2_ROWS(16); }
            else { LB2_ROWS(32); }
#undef LB2_ROWS
        }
        __syncthreads();
        const int nlong = s_nlong;
        for (int i = 0; i < nlong; ++i) {
            const int row = s_long[i];
            const int e = row == rc ? k1 : __ldg(rp + row + 1);
            const T sum = lb2_block_dot(max(__ldg(rp + row), k0), e, ci, v, b, bs, s_red);
            if (threadIdx.x == 0) {
                if (row == rc) {
                    s_carry = sum;
                } else {
                    T out = a * sum;
                    if (XIN) out += bt * xin[(int64_t)row * xins];
                    x[(int64_t)row * xs] = out;
                }
            }
        }
        if (threadIdx.x == 0) {
            carry_row[tile] = r1;
            carry_val[tile] = s_carry;
        }
        if (gridDim.x < ntiles) __syncthreads();  // persistent: s_carry / s_nlong are reused
    }
}

template <typename T>
static int csr_lb(int64_t n, int64_t nnz, const int* rp, const int* ci, const T* v, const T* b,
                  int64_t bs, T* x, int64_t xs, T alpha, const T* alpha_dev, T beta,
                  const T* beta_dev, const T* xin, int64_t xins, const int* coords,
                  int* carry_row, T* carry_val, int tile, int mode, void* stream) {
    if (n == 0) return B200SP_OK;
    B200SP_REQUIRE(mode == 2, B200SP_EINVAL, "csr lb: mode must be 2 (row tiles) or 3 (nnz split), got %d", mode);
    B200SP_REQUIRE(tile > 0, B200SP_EINVAL, "csr lb: tile must be positive (plan with b200sp_csr_lb_tile)");
    cudaStream_t st = as_stream(stream);
    Coef<T> al = coef(alpha, alpha_dev), be = coef(beta, beta_dev);
    const int64_t ntiles = ceil_div(n + nnz, tile);
    {
        // predicated blocks of 4 entries per lane (lb2_unroll 4) vs the plain loop (1):
        // 27-point fp64 0.711 vs 0.667, fp32 0.629 vs 0.558 (profiles/r03_lb_blocks.txt)
        auto k2 = tuning("lb2_unroll", 4) == 4 ? (xin ? csr_lb2_kernel<T, true, true> : csr_lb2_kernel<T, false, true>)
                                                : (xin ? csr_lb2_kernel<T, true, false> : csr_lb2_kernel<T, false, false>);
        // (aligned pair loads, as the classical kernel's fp32 default, measured
        // 0.49 / 0.42 vs 0.71 / 0.62 here: profiles/r03_lb_blocks.txt)
        const unsigned g2 = (unsigned)std::min<int64_t>(ntiles, (int64_t)kNumSMs * tuning("lb2_per_sm", 1 << 20));  // one CTA per tile measured best (0.66 vs 0.51 persistent)
        k2<<<g2, LB_BLOCK, 0, st>>>(n, ntiles, rp, ci, v, b, bs, x, xs, al, be, xin, xins, coords, carry_row,
                                    carry_val);
    }
    csr_lb_fixup_kernel<T><<<(unsigned)ceil_div(ntiles, 256), 256, 0, st>>>(n, ntiles, carry_row, carry_val, x, xs, al);
    count_launch(2);
    return check_launch("csr_lb");
}

// ===========================================================================
// Coo: warp-chunked segmented reduction over the (row, col)-sorted entries.
// Each warp owns a contiguous chunk of 32*COO_E entries; every lane loads
// COO_E consecutive entries with 128-bit streaming loads (the warp's loads
// are fully coalesced and all independent), reduces its equal-row runs in
// registers, and one shuffle segmented scan per chunk joins runs that cross
// lanes. Rows owned by the chunk are written directly; rows that straddle a
// chunk boundary leave per-chunk partials that a fix-up pass sums in chunk
// order, so the result is deterministic (no floating-point atomics) and needs
// no pre-zero pass over x.
// ===========================================================================
constexpr int COO_BLOCK = 256;

// The segmented reduction of one warp chunk (shared by Coo and the Csr
// nnz-split strategy): r[i] / p[i] = row and product of the lane's entries
// (r = INT_MAX past the chunk end), head/tail = rows of the chunk's first /
// last entry and whether they continue into the previous / next chunk.
template <typename T, bool XIN, int E>
__device__ __forceinline__ void coo_segments(int64_t c, int64_t e0, int64_t e1, int cnt, const int (&r)[E],
                                             const T (&p)[E], int head_row, int tail_row, bool head_shared,
                                             bool tail_shared, T a, T bt, T* __restrict__ x, int64_t xs,
                                             const T* __restrict__ xin, int64_t xins, T* __restrict__ carry_head,
                                             T* __restrict__ carry_tail) {
    const int lane = threadIdx.x & 31;
    // lane-local runs: the first completed run may continue from earlier
    // lanes (needs the scan), later completed runs are final
    int cur = r[0], first_row = INT_MIN;
    T acc = 0, first_val = 0;
#pragma unroll
    for (int i = 0; i < E; ++i) {
        if (i < cnt) {
            if (r[i] != cur) {
                if (first_row == INT_MIN) {
                    first_row = cur;
                    first_val = acc;
                } else {
                    T out = a * acc;
                    if (XIN) out += bt * xin[(int64_t)cur * xins];
                    x[(int64_t)cur * xs] = out;
                }
                cur = r[i];
                acc = 0;
            }
            acc += p[i];
        }
    }
    // a lane's first run continues the previous lane's last run only if the
    // rows match (a new row may start exactly at a lane boundary)
    int prev_last = __shfl_up_sync(0xffffffffu, cur, 1);
    const int next_first = __shfl_down_sync(0xffffffffu, r[0], 1);
    const bool continues = lane > 0 && cnt > 0 && r[0] == prev_last;
    // warp segmented inclusive scan of carry-outs; a segment starts at every
    // lane that closed a run or does not continue its predecessor
    T sv = acc;
    int sf = (first_row != INT_MIN) || !continues;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T vn = __shfl_up_sync(0xffffffffu, sv, o);
        int fn = __shfl_up_sync(0xffffffffu, sf, o);
        if (lane >= o) {
            if (!sf) sv += vn;
            sf |= fn;
        }
    }
    T excl = __shfl_up_sync(0xffffffffu, sv, 1);
    if (!continues) excl = 0;
    const int last_lane = (int)((e1 - 1 - e0) / E);  // lane holding the chunk's last entry
    if (first_row != INT_MIN) {
        const T val = first_val + excl;
        if (first_row == head_row && head_shared) {
            carry_head[c] = val;
        } else {
            T out = a * val;
            if (XIN) out += bt * xin[(int64_t)first_row * xins];
            x[(int64_t)first_row * xs] = out;
        }
    }
    // last run ends exactly at this lane's boundary: complete here
    if (cnt > 0 && lane < last_lane && next_first != cur) {
        if (cur == head_row && head_shared) {
            carry_head[c] = sv;
        } else {
            T out = a * sv;
            if (XIN) out += bt * xin[(int64_t)cur * xins];
            x[(int64_t)cur * xs] = out;
        }
    }
    if (lane == last_lane) {
        const bool single = head_row == tail_row;
        if (!(tail_shared || (single && head_shared))) {
            T out = a * sv;
            if (XIN) out += bt * xin[(int64_t)tail_row * xins];
            x[(int64_t)tail_row * xs] = out;
        } else if (single) {
            carry_head[c] = sv;
        } else {
            carry_tail[c] = sv;
        }
    }
}

// MINB: 6 CTAs per SM (<= 40 registers) measured best for fp32 (0.70 vs
// 0.63 of the roofline), unbounded (62 registers) for fp64 (0.645 vs 0.55).
template <typename T, bool XIN, bool VEC, int E>
__device__ __forceinline__ void coo_body(int64_t nnz, const int* __restrict__ rows, const int* __restrict__ cols,
           const T* __restrict__ vals, const T* __restrict__ b, int64_t bs, T* __restrict__ x,
           int64_t xs, Coef<T> alpha, Coef<T> beta, const T* __restrict__ xin, int64_t xins,
           T* __restrict__ carry_head, T* __restrict__ carry_tail, int2* __restrict__ chunk_rows) {
    constexpr int CHUNK = 32 * E;
    const int lane = threadIdx.x & 31;
    const int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t e0 = c * CHUNK;
    if (e0 >= nnz) return;
    const int64_t e1 = min(e0 + (int64_t)CHUNK, nnz);
    const int head_row = rows[e0], tail_row = rows[e1 - 1];
    if (chunk_rows && lane == 0) chunk_rows[c] = make_int2(head_row, tail_row);  // for the fix-up
    const bool head_shared = e0 > 0 && rows[e0 - 1] == head_row;
    const bool tail_shared = e1 < nnz && rows[e1] == tail_row;
    const T a = alpha.get();
    const T bt = XIN ? beta.get() : T(0);

    const int64_t l0 = e0 + (int64_t)lane * E;
    const int cnt = (int)max((int64_t)0, min((int64_t)E, e1 - l0));
    int r[E], cc[E];
    T vv[E];
    if (VEC && cnt == E) {
        // streaming loads measured best on C2 (0.646 vs 0.623 with
        // L1-allocating ones; the power law prefers L1: 0.39 vs 0.36)
        ld_stream_vec<E>(rows + l0, r);
        ld_stream_vec<E>(cols + l0, cc);
        ld_stream_vec<E>(vals + l0, vv);
    } else {
#pragma unroll
        for (int i = 0; i < E; ++i) {
            const bool ok = i < cnt;
            r[i] = ok ? ld_stream(rows + l0 + i) : INT_MAX;
            cc[i] = ok ? ld_stream(cols + l0 + i) : 0;
            vv[i] = ok ? ld_stream(vals + l0 + i) : T(0);
        }
    }
    T p[E];
#pragma unroll
    for (int i = 0; i < E; ++i) p[i] = i < cnt ? vv[i] * ld_gather(b + (int64_t)cc[i] * bs) : T(0);
    coo_segments<T, XIN, E>(c, e0, e1, cnt, r, p, head_row, tail_row, head_shared, tail_shared, a, bt, x, xs,
                            xin, xins, carry_head, carry_tail);
}

#define COO_ARGS                                                                                         \
    int64_t nnz, const int* __restrict__ rows, const int* __restrict__ cols, const T* __restrict__ vals,   \
        const T* __restrict__ b, int64_t bs, T* __restrict__ x, int64_t xs, Coef<T> alpha, Coef<T> beta,   \
        const T* __restrict__ xin, int64_t xins, T* __restrict__ carry_head, T* __restrict__ carry_tail,        \
        int2* __restrict__ chunk_rows
#define COO_PASS nnz, rows, cols, vals, b, bs, x, xs, alpha, beta, xin, xins, carry_head, carry_tail, chunk_rows
template <typename T, bool XIN, bool VEC, int E>
__global__ void __launch_bounds__(COO_BLOCK) coo_kernel(COO_ARGS) {
    if (alpha.skip()) return;
    coo_body<T, XIN, VEC, E>(COO_PASS);
}
template <typename T, bool XIN, bool VEC, int E>
__global__ void __launch_bounds__(COO_BLOCK, 6) coo_kernel_b6(COO_ARGS) {
    if (alpha.skip()) return;
    coo_body<T, XIN, VEC, E>(COO_PASS);
}
#undef COO_ARGS
#undef COO_PASS


// Carry fix-up: the owner of a row shared by several chunks (the chunk holding
// the row's first entries) adds the head partials of the chunks that follow
// it in chunk order. Chains of up to COO_FIX_SERIAL chunks are summed by the
// owner thread; a longer chain (a row of thousands of entries: the power
// law's 50k rows span ~200 chunks and serialised this pass for ~110 us) is
// summed by the owner's whole warp, lanes striding over the chain and a
// shuffle tree combining them (deterministic: the order depends only on the
// chain length).
constexpr int COO_FIX_SERIAL = 32;

// rows of a chunk's first / last entry: read from the Coo row indices, or
// (Csr nnz-split) from the plan's chunk start rows and the kernel's tail rows
struct CooChunkRows {
    const int* rows;
    int chunk;
    int64_t nnz;
    __device__ int head(int64_t c) const { return rows[c * chunk]; }
    __device__ int tail(int64_t c) const { return rows[min((c + 1) * chunk, nnz) - 1]; }
};
struct PairChunkRows {  // (head, tail) per chunk, recorded by the Coo kernel
    const int2* cr;
    __device__ int head(int64_t c) const { return cr[c].x; }
    __device__ int tail(int64_t c) const { return cr[c].y; }
};
struct CsrChunkRows {
    const int* srow;
    const int* ctail;
    __device__ int head(int64_t c) const { return srow[c]; }
    __device__ int tail(int64_t c) const { return ctail[c]; }
};

template <typename T, bool XIN, class Rows>
__global__ void __launch_bounds__(256)
coo_fixup_kernel(int64_t nchunks, Rows R, const T* __restrict__ carry_head, const T* __restrict__ carry_tail,
                 T* __restrict__ x, int64_t xs, Coef<T> alpha, Coef<T> beta,
                 const T* __restrict__ xin, int64_t xins) {
    if (alpha.skip()) return;
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    bool is_long = false, single = false;
    int tail_row = 0;
    if (c < nchunks) {
        const int head_row = R.head(c);
        tail_row = R.tail(c);
        const bool head_shared = c > 0 && R.tail(c - 1) == head_row;
        const bool tail_shared = c + 1 < nchunks && R.head(c + 1) == tail_row;
        single = head_row == tail_row;
        if (tail_shared && !(single && head_shared)) {  // owner of a shared row
            const int64_t probe = c + COO_FIX_SERIAL + 1;
            is_long = probe < nchunks && R.head(probe) == tail_row;
            if (!is_long) {
                T sum = single ? carry_head[c] : carry_tail[c];
                for (int64_t u = c + 1; u < nchunks; ++u) {
                    sum += carry_head[u];
                    const int u_tail = R.tail(u);
                    const bool u_single = R.head(u) == u_tail;
                    const bool u_tail_shared = u + 1 < nchunks && R.head(u + 1) == u_tail;
                    if (!(u_single && u_tail_shared)) break;
                }
                T out = alpha.get() * sum;
                if (XIN) out += beta.get() * xin[(int64_t)tail_row * xins];
                x[(int64_t)tail_row * xs] = out;
            }
        }
    }
    // long chains: the owner's warp sums them (every lane is still here)
    unsigned longs = __ballot_sync(0xffffffffu, is_long);
    while (longs) {
        const int src = __ffs(longs) - 1;
        longs &= longs - 1;
        const int64_t oc = __shfl_sync(0xffffffffu, c, src);
        const int row = __shfl_sync(0xffffffffu, tail_row, src);
        T acc = 0;
        // the chain: every later chunk whose first entry is still in `row`
        for (int64_t u = oc + 1 + lane;; u += 32) {
            const bool in = u < nchunks && R.head(u) == row;
            if (in) acc += carry_head[u];
            if (__ballot_sync(0xffffffffu, in) != 0xffffffffu) break;
        }
        acc = warp_sum(acc);
        if (lane == src) {
            T out = alpha.get() * ((single ? carry_head[oc] : carry_tail[oc]) + acc);
            if (XIN) out += beta.get() * xin[(int64_t)row * xins];
            x[(int64_t)row * xs] = out;
        }
    }
}

// ===========================================================================
// Csr, load-balanced strategy mode 3 ("nnz split"): the Coo kernel's warp
// chunks of 32 x SEG_E consecutive nonzeros, with each entry's row derived
// from the row pointers instead of read from a row-index array. The plan
// holds the row of every chunk's first entry (srow[c]); a lane binary-
// searches its first entry's row inside [srow[c], srow[c+1]] and walks
// row_ptrs from there. Empty rows are written by the lane whose entry starts
// the next non-empty row
// (trailing ones by the last lane). Chunk carries and the fix-up are the
// Coo ones (the kernel records each chunk's tail row for the fix-up). For
// skewed row lengths (the C3 power law): every warp gets the same number
// of nonzeros and all of a lane's gathers are independent.
// ===========================================================================
constexpr int SEG_E = 8;  // entries per lane (round 1: 4 -> 464 us, 8 -> 433 us, 16 -> 679 us on C3)
constexpr int SEG_CHUNK = 32 * SEG_E;

// srow[c] = row of chunk c's first entry; srow[nchunks] = n
__global__ void csr_seg_plan_kernel(int64_t n, int64_t nnz, const int* __restrict__ rp, int64_t nchunks,
                                    int* __restrict__ srow) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t > nchunks) return;
    if (t == nchunks) {
        srow[t] = (int)n;
        return;
    }
    const int64_t e = t * SEG_CHUNK;
    int64_t lo = 0, hi = n - 1;  // largest row r with rp[r] <= e
    while (lo < hi) {
        const int64_t mid = (lo + hi + 1) >> 1;
        if (rp[mid] <= e) lo = mid;
        else hi = mid - 1;
    }
    srow[t] = (int)lo;
}

template <typename T, bool XIN, bool VEC, int MINB>
__global__ void __launch_bounds__(COO_BLOCK, MINB)
csr_seg_kernel(int64_t n, int64_t nnz, const int* __restrict__ rp, const int* __restrict__ ci,
               const T* __restrict__ v, const T* __restrict__ b, int64_t bs, T* __restrict__ x, int64_t xs,
               Coef<T> alpha, Coef<T> beta, const T* __restrict__ xin, int64_t xins, const int* __restrict__ srow,
               int* __restrict__ ctail, T* __restrict__ carry_head, T* __restrict__ carry_tail) {
    if (alpha.skip()) return;
    constexpr int E = SEG_E;
    const int lane = threadIdx.x & 31;
    const int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t e0 = c * SEG_CHUNK;
    if (e0 >= nnz) return;
    const int64_t e1 = min(e0 + (int64_t)SEG_CHUNK, nnz);
    const T a = alpha.get();
    const T bt = XIN ? beta.get() : T(0);
    auto write_empty = [&](int64_t q) {
        T out = a * T(0);
        if (XIN) out += bt * xin[q * xins];
        x[q * xs] = out;
    };
    const int64_t l0 = e0 + (int64_t)lane * E;
    const int cnt = (int)max((int64_t)0, min((int64_t)E, e1 - l0));
    int cc[E];
    T vv[E];
    if (VEC && cnt == E) {
        ld_cached_vec<E>(ci + l0, cc);  // L1-allocating: 433 vs 452 us streaming on C3
        ld_cached_vec<E>(v + l0, vv);
    } else {
#pragma unroll
        for (int i = 0; i < E; ++i) {
            const bool ok = i < cnt;
            cc[i] = ok ? __ldg(ci + l0 + i) : 0;
            vv[i] = ok ? __ldg(v + l0 + i) : T(0);
        }
    }
    T p[E];
#pragma unroll
    for (int i = 0; i < E; ++i) p[i] = i < cnt ? vv[i] * ld_gather(b + (int64_t)cc[i] * bs) : T(0);

    // rows of the lane's entries: binary search for the first one inside the
    // chunk's row range, then a walk over row_ptrs (L1 hits, issued while the
    // gathers are in flight). Measured alternatives (profiles/r02_c3_lb3.txt):
    // a per-lane start-row plan (0.5 B per nonzero) 444 vs 433 us on C3, a
    // shuffle search over a 32-row window 521 us
    const int head_row = srow[c];
    int r[E];
    int cur = head_row;
    // Fast path: the chunk's row starts as a 256-bit mask. Row starts inside
    // (e0, e1) are rp[head_row + 1 .. srow[c + 1]] -- loaded once per chunk,
    // coalesced, one per lane -- and bit q marks a row starting at entry
    // e0 + q; an entry's row is head_row + the set bits at or before it. No
    // per-lane search, no load chain. Taken when the chunk holds no empty row
    // (set bits == starts) and at most 256 row starts; else the search below.
    __shared__ unsigned s_mask[COO_BLOCK / 32][SEG_CHUNK / 32];
    unsigned* mask = s_mask[threadIdx.x >> 5];
    const int nstart = min(srow[c + 1], (int)n) - head_row;
    const int clen = (int)(e1 - e0);
    bool fast = nstart <= SEG_CHUNK;
    int mine_starts = 0;
    if (fast) {
#pragma unroll
        for (int w = lane; w < SEG_CHUNK / 32; w += 32) mask[w] = 0u;
        __syncwarp();
        int& mine = mine_starts;
        for (int j = lane; j < nstart; j += 32) {
            const int q = __ldg(rp + head_row + 1 + j) - (int)e0;
            if (q > 0 && q < clen) {
                atomicOr(&mask[q >> 5], 1u << (q & 31));
                ++mine;
            }
        }
        __syncwarp();
    }
    // lane w < 8 holds mask word w and the count of set bits in words < w
    const unsigned mw = fast && lane < SEG_CHUNK / 32 ? mask[lane] : 0u;
    int incl = __popc(mw);
#pragma unroll
    for (int o = 1; o < SEG_CHUNK / 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (fast) fast = __all_sync(0xffffffffu, warp_sum(mine_starts) == __shfl_sync(0xffffffffu, incl, SEG_CHUNK / 32 - 1));
    if (fast) {
        // rows started at or before the lane's first entry (positions <= E lane)
        const int p0 = lane * E;
        const int wl = p0 >> 5;  // E | 32: the lane's bits stay in one word
        const unsigned myw = __shfl_sync(0xffffffffu, mw, wl);
        int d = __shfl_sync(0xffffffffu, incl - __popc(mw), wl) + __popc(myw & (0xffffffffu >> (31 - (p0 & 31))));
        const unsigned word = myw >> (p0 & 31);
#pragma unroll
        for (int i = 0; i < E; ++i) {
            if (i > 0) d += (word >> i) & 1u;
            r[i] = i < cnt ? head_row + d : INT_MAX;
            if (i < cnt) cur = head_row + d;
        }
        if (lane == 0 && __ldg(rp + head_row) == e0)  // empty rows ending right before the chunk
            for (int q = head_row - 1; q >= 0 && __ldg(rp + q) == e0; --q) write_empty(q);
    } else if (cnt > 0) {
        int lo = head_row, hi = min(srow[c + 1], (int)n - 1);
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (__ldg(rp + mid) <= l0) lo = mid;
            else hi = mid - 1;
        }
        cur = lo;
        if (__ldg(rp + cur) == l0)  // the empty rows just before a row starting here
            for (int q = cur - 1; q >= 0 && __ldg(rp + q) == l0; --q) write_empty(q);
        // the ends of rows cur .. cur+E-1: independent loads, then every
        // entry's row is a count of ends at or before it (no load chain)
        int ends[E];
#pragma unroll
        for (int k = 0; k < E; ++k) ends[k] = cur + 1 + k <= n ? __ldg(rp + cur + 1 + k) : INT_MAX;
        const int last = (int)(l0 + cnt - 1);
        if (ends[E - 1] > last) {
            const int row0 = cur;
#pragma unroll
            for (int i = 0; i < E; ++i) {
                const int e = (int)(l0 + i);
                int d = 0;
#pragma unroll
                for (int k = 0; k < E; ++k) d += ends[k] <= e;
                r[i] = i < cnt ? row0 + d : INT_MAX;
                if (i < cnt) cur = row0 + d;
            }
#pragma unroll
            for (int k = 1; k < E; ++k)  // empty rows starting inside the lane's range
                if (ends[k - 1] == ends[k] && ends[k - 1] <= last) write_empty(row0 + k);
        } else {  // the lane's entries reach past E rows (runs of empty rows)
            int nend = ends[0];
#pragma unroll
            for (int i = 0; i < E; ++i) {
                if (i < cnt) {
                    const int e = (int)(l0 + i);
                    while (e >= nend) {
                        ++cur;
                        nend = __ldg(rp + cur + 1);
                        if (nend <= e) write_empty(cur);
                    }
                    r[i] = cur;
                } else {
                    r[i] = INT_MAX;
                }
            }
        }
    } else {
#pragma unroll
        for (int i = 0; i < E; ++i) r[i] = INT_MAX;
    }
    if (fast && cnt == 0) cur = head_row;
    const int last_lane = (int)((e1 - 1 - e0) / E);
    const int tail_row = __shfl_sync(0xffffffffu, cur, last_lane);
    const bool head_shared = e0 > 0 && __ldg(rp + head_row) < e0;
    const bool tail_shared = e1 < nnz && __ldg(rp + tail_row + 1) > e1;
    if (lane == last_lane) {
        ctail[c] = tail_row;
        if (e1 == nnz)
            for (int64_t q = (int64_t)tail_row + 1; q < n; ++q) write_empty(q);  // trailing empty rows
    }
    coo_segments<T, XIN, E>(c, e0, e1, cnt, r, p, head_row, tail_row, head_shared, tail_shared, a, bt, x, xs,
                            xin, xins, carry_head, carry_tail);
}

template <typename T>
static int csr_seg(int64_t n, int64_t nnz, const int* rp, const int* ci, const T* v, const T* b, int64_t bs, T* x,
                   int64_t xs, T alpha, const T* alpha_dev, T beta, const T* beta_dev, const T* xin, int64_t xins,
                   const int* srow, int* ctail, T* carry, int tile, void* stream) {
    if (n == 0) return B200SP_OK;
    B200SP_REQUIRE(tile == SEG_CHUNK, B200SP_EINVAL, "csr lb mode 3: tile must be %d (got %d)", SEG_CHUNK, tile);
    B200SP_REQUIRE(nnz < INT_MAX - SEG_CHUNK, B200SP_EINVAL, "csr lb mode 3: nnz must fit int32 entry indices");
    if (nnz == 0)  // every row empty: the classical kernel writes alpha * 0 + beta * x_in
        return csr_classical<T>(n, rp, ci, v, b, bs, x, xs, alpha, alpha_dev, beta, beta_dev, xin, xins, 1, stream);
    cudaStream_t st = as_stream(stream);
    Coef<T> al = coef(alpha, alpha_dev), be = coef(beta, beta_dev);
    const int64_t nchunks = ceil_div(nnz, SEG_CHUNK);
    T* carry_head = carry;
    T* carry_tail = carry + nchunks;
    const unsigned grid = (unsigned)ceil_div(nchunks * 32, COO_BLOCK);
    const unsigned fgrid = (unsigned)ceil_div(nchunks, 256);
    const bool vec = aligned16(ci) && aligned16(v);
    const CsrChunkRows R{srow, ctail};
    // 5 CTAs per SM (48 registers): C3 404.5 us vs 447.7 unbounded (70 registers, 3 CTAs), 420.9 at 4, 451.7 at 6 (spills)
    const int minb = tuning("seg_minb", 5);
#define SEG_LAUNCH(XI, VE)                                                                                   \
    do {                                                                                                     \
        if (minb >= 6)                                                                                       \
            csr_seg_kernel<T, XI, VE, 6><<<grid, COO_BLOCK, 0, st>>>(n, nnz, rp, ci, v, b, bs, x, xs, al, be,  \
                                                                     xin, xins, srow, ctail, carry_head, carry_tail); \
        else if (minb == 4)                                                                                  \
            csr_seg_kernel<T, XI, VE, 4><<<grid, COO_BLOCK, 0, st>>>(n, nnz, rp, ci, v, b, bs, x, xs, al, be,  \
                                                                     xin, xins, srow, ctail, carry_head, carry_tail); \
        else if (minb == 5)                                                                                  \
            csr_seg_kernel<T, XI, VE, 5><<<grid, COO_BLOCK, 0, st>>>(n, nnz, rp, ci, v, b, bs, x, xs, al, be,  \
                                                                     xin, xins, srow, ctail, carry_head, carry_tail); \
        else                                                                                                 \
            csr_seg_kernel<T, XI, VE, 1><<<grid, COO_BLOCK, 0, st>>>(n, nnz, rp, ci, v, b, bs, x, xs, al, be,  \
                                                                     xin, xins, srow, ctail, carry_head, carry_tail); \
    } while (0)
    if (xin) {
        if (vec) SEG_LAUNCH(true, true); else SEG_LAUNCH(true, false);
        coo_fixup_kernel<T, true><<<fgrid, 256, 0, st>>>(nchunks, R, carry_head, carry_tail, x, xs, al, be, xin, xins);
    } else {
        if (vec) SEG_LAUNCH(false, true); else SEG_LAUNCH(false, false);
        coo_fixup_kernel<T, false><<<fgrid, 256, 0, st>>>(nchunks, R, carry_head, carry_tail, x, xs, al, be, xin, xins);
    }
#undef SEG_LAUNCH
    count_launch(2);
    return check_launch("csr_seg");
}

template <typename T>
static int coo_spmv(int64_t nnz, int chunk, const int* rows, const int* cols, const T* vals,
                    const T* b, int64_t bs, T* x, int64_t xs, T alpha, const T* alpha_dev, T beta,
                    const T* beta_dev, const T* xin, int64_t xins, T* carry_head, T* carry_tail,
                    int32_t* chunk_rows_ws, void* stream) {
    if (nnz == 0) return B200SP_OK;
    B200SP_REQUIRE(chunk == 128 || chunk == 256, B200SP_EINVAL, "coo: chunk must be 128 or 256 (got %d)", chunk);
    cudaStream_t st = as_stream(stream);
    Coef<T> al = coef(alpha, alpha_dev), be = coef(beta, beta_dev);
    const int64_t nchunks = ceil_div(nnz, chunk);
    const int64_t threads = nchunks * 32;
    const unsigned grid = (unsigned)ceil_div(threads, COO_BLOCK);
    const unsigned fgrid = (unsigned)ceil_div(nchunks, 256);
    const bool vec = aligned16(rows) && aligned16(cols) && aligned16(vals);
    const int minb = tuning("coo_minb", sizeof(T) == 4 ? 6 : 1);
    int2* crows = reinterpret_cast<int2*>(chunk_rows_ws);
    B200SP_REQUIRE(!crows || (reinterpret_cast<uintptr_t>(crows) & 7) == 0, B200SP_EINVAL,
                   "coo: chunk_rows must be 8-byte aligned");
#define COO_LAUNCH(XI, VE)                                                                                  \
    do {                                                                                                    \
        if (chunk == 128)                                                                                   \
            coo_kernel<T, XI, VE, 4><<<grid, COO_BLOCK, 0, st>>>(nnz, rows, cols, vals, b, bs, x, xs, al,  \
                                                                    be, xin, xins, carry_head, carry_tail, crows); \
        else if (minb == 6)                                                                                 \
            coo_kernel_b6<T, XI, VE, 8><<<grid, COO_BLOCK, 0, st>>>(nnz, rows, cols, vals, b, bs, x, xs, al,  \
                                                                    be, xin, xins, carry_head, carry_tail, crows); \
        else                                                                                                \
            coo_kernel<T, XI, VE, 8><<<grid, COO_BLOCK, 0, st>>>(nnz, rows, cols, vals, b, bs, x, xs, al,  \
                                                                    be, xin, xins, carry_head, carry_tail, crows); \
    } while (0)
    // the fix-up reads each chunk's (head, tail) rows from the kernel's record
    // when given the workspace (2 ints per chunk, contiguous) instead of
    // strided row-index loads (C3: 76 MB of scattered sectors, 32 us)
#define COO_FIXUP(XI)                                                                                       \
    do {                                                                                                    \
        if (crows)                                                                                          \
            coo_fixup_kernel<T, XI><<<fgrid, 256, 0, st>>>(nchunks, PairChunkRows{crows}, carry_head, carry_tail, \
                                                           x, xs, al, be, xin, xins);                       \
        else                                                                                                \
            coo_fixup_kernel<T, XI><<<fgrid, 256, 0, st>>>(nchunks, CooChunkRows{rows, chunk, nnz}, carry_head, \
                                                           carry_tail, x, xs, al, be, xin, xins);           \
    } while (0)
    if (xin) {
        if (vec) COO_LAUNCH(true, true); else COO_LAUNCH(true, false);
        COO_FIXUP(true);
    } else {
        if (vec) COO_LAUNCH(false, true); else COO_LAUNCH(false, false);
        COO_FIXUP(false);
    }
#undef COO_FIXUP
#undef COO_LAUNCH
    count_launch(2);
    return check_launch("coo_spmv");
}

// x[rows[i]] = beta * x_in[rows[i]] (or 0): rows that hold no entry
template <typename T>
__global__ void rows_scale_kernel(int64_t count, const int* __restrict__ rows, T* __restrict__ x,
                                  int64_t xs, Coef<T> beta, const T* __restrict__ xin, int64_t xins) {
    if (beta.skip()) return;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const int64_t r = rows[i];
    x[r * xs] = xin ? beta.get() * xin[r * xins] : T(0);
}

template <typename T>
static int rows_scale(int64_t count, const int* rows, T* x, int64_t xs, T beta, const T* beta_dev,
                      const T* xin, int64_t xins, void* stream) {
    if (count == 0) return B200SP_OK;
    rows_scale_kernel<T><<<(unsigned)ceil_div(count, 256), 256, 0, as_stream(stream)>>>(
        count, rows, x, xs, coef(beta, beta_dev), xin, xins);
    count_launch();
    return check_launch("rows_scale");
}

// Dot product of one row stored at base, base+step, ... (len slots, padding
// col = -1) with b: UNR independent loads in flight per thread.
template <typename T, int UNR, bool L1 = false>
__device__ __forceinline__ T strided_dot(const int* __restrict__ ci, const T* __restrict__ v, int64_t base,
                                         int64_t step, int len, const T* __restrict__ b, int64_t bs) {
    T acc[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) acc[u] = 0;
    int k = 0;
#pragma unroll 1
    for (; k + UNR <= len; k += UNR) {
        int c[UNR];
        T vv[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            c[u] = L1 ? __ldg(ci + base + (int64_t)(k + u) * step) : ld_stream(ci + base + (int64_t)(k + u) * step);
            vv[u] = L1 ? __ldg(v + base + (int64_t)(k + u) * step) : ld_stream(v + base + (int64_t)(k + u) * step);
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u)
            if (c[u] >= 0) acc[u] += vv[u] * ld_gather(b + (int64_t)c[u] * bs);
    }
    if (k < len) {  // the tail as one more predicated block: its loads in flight together
        int c[UNR];
        T vv[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const bool ok = k + u < len;
            c[u] = ok ? ld_stream(ci + base + (int64_t)(k + u) * step) : -1;
            vv[u] = ok ? ld_stream(v + base + (int64_t)(k + u) * step) : T(0);
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u)
            if (c[u] >= 0) acc[u] += vv[u] * ld_gather(b + (int64_t)c[u] * bs);
    }
    T sum = acc[0];
#pragma unroll
    for (int u = 1; u < UNR; ++u) sum += acc[u];
    return sum;
}

// ===========================================================================
// Ell: column-major (stride >= n), one thread per row, padding col = -1.
// Consecutive threads read consecutive addresses of every stored column.
// ===========================================================================
template <typename T, bool XIN, int UNR, bool L1>
__global__ void __launch_bounds__(256)
ell_kernel(int64_t n, int64_t width, int64_t stride, const int* __restrict__ ci,
           const T* __restrict__ v, const T* __restrict__ b, int64_t bs, T* __restrict__ x,
           int64_t xs, Coef<T> alpha, Coef<T> beta, const T* __restrict__ xin, int64_t xins) {
    if (alpha.skip()) return;
    const T a = alpha.get();
    const T bt = XIN ? beta.get() : T(0);
    for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < n;
         row += (int64_t)gridDim.x * blockDim.x) {
        const T sum = strided_dot<T, UNR, L1>(ci, v, row, stride, (int)width, b, bs);
        T out = a * sum;
        if (XIN) out += bt * xin[row * xins];
        x[row * xs] = out;
    }
}

template <typename T>
static int ell_spmv(int64_t n, int64_t width, int64_t stride, const int* ci, const T* v, const T* b,
                    int64_t bs, T* x, int64_t xs, T alpha, const T* alpha_dev, T beta,
                    const T* beta_dev, const T* xin, int64_t xins, void* stream) {
    if (n == 0) return B200SP_OK;
    B200SP_REQUIRE(stride >= n, B200SP_EINVAL, "ell: stride %lld < rows %lld", (long long)stride, (long long)n);
    cudaStream_t st = as_stream(stream);
    Coef<T> al = coef(alpha, alpha_dev), be = coef(beta, beta_dev);
    const int per_sm = tuning("ell_per_sm", 16);
    const int grid = per_sm > 0 ? grid_for(n, 256, per_sm) : (int)ceil_div(n, 256);
    // 4 entries in flight per thread, the tail as one predicated block (ell_unr
    // 3 / 4 / 6 / 8 measured 0.897 / 0.928 / 0.816 / 0.816 on C2 fp64,
    // profiles/r03_ell_tail.txt)
    auto kern = xin ? ell_kernel<T, true, 4, false> : ell_kernel<T, false, 4, false>;
    kern<<<grid, 256, 0, st>>>(n, width, stride, ci, v, b, bs, x, xs, al, be, xin, xins);
    count_launch();
    return check_launch("ell_spmv");
}

// ===========================================================================
// Sellp: slices of `slice_size` rows, each stored column-major with its own
// length (slice_sets = exclusive prefix of slice lengths). Thread per row.
// ===========================================================================
// One thread per row, no grid-stride loop (every CTA covers 256 / slice
// rows of whole slices): fewer live registers than the grid-stride form
// (ncu: 40 registers capped warps active at 66% vs Ell's 96%).
// S > 0: compile-time slice size (the default 64: shifts instead of a 64-bit
// division per row). GS: grid-stride rows (fp32) or one row per thread (fp64).
// MINB = 8 caps registers at 32 (8 CTAs per SM): the unbounded build used
// 56-66 registers and held warps active at 46-66% (ncu), 0.52 / 0.65 of the
// roofline; bounded: 0.64 / 0.79 (profiles/r02_format_sweep.txt).
template <typename T, bool XIN, int UNR, int MINB, bool GS, int S>
__global__ void __launch_bounds__(256, MINB)
sellp_kernel(int64_t n, int slice_size, const int* __restrict__ slice_lengths,
             const int* __restrict__ slice_sets, const int* __restrict__ ci, const T* __restrict__ v,
             const T* __restrict__ b, int64_t bs, T* __restrict__ x, int64_t xs, Coef<T> alpha,
             Coef<T> beta, const T* __restrict__ xin, int64_t xins) {
    if (alpha.skip()) return;
    const int ss = S > 0 ? S : slice_size;
#pragma unroll 1
    for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < n;
         row += GS ? (int64_t)gridDim.x * blockDim.x : n) {
        const int64_t slice = row / ss;
        const int local = (int)(row - slice * ss);
        const int len = __ldg(slice_lengths + slice);
        const int64_t base = (int64_t)__ldg(slice_sets + slice) * ss + local;
        const T sum = strided_dot<T, UNR>(ci, v, base, ss, len, b, bs);
        T out = alpha.get() * sum;
        if (XIN) out += beta.get() * xin[row * xins];
        x[row * xs] = out;
    }
}

template <typename T, bool XIN, int S>
static void launch_sellp(int64_t n, int slice_size, const int* sl, const int* ss, const int* ci, const T* v,
                         const T* b, int64_t bs, T* x, int64_t xs, Coef<T> al, Coef<T> be, const T* xin,
                         int64_t xins, cudaStream_t st) {
    const bool gs = tuning("sellp_grid_stride", 1);  // fp64 0.876 vs 0.860 one row per thread (r03_ell_tail)
    if (gs)
        sellp_kernel<T, XIN, 4, 8, true, S><<<grid_for(n, 256, 16), 256, 0, st>>>(n, slice_size, sl, ss, ci, v, b, bs,
                                                                                 x, xs, al, be, xin, xins);
    else
        sellp_kernel<T, XIN, 4, 8, false, S><<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(
            n, slice_size, sl, ss, ci, v, b, bs, x, xs, al, be, xin, xins);
}

template <typename T>
static int sellp_spmv(int64_t n, int slice_size, const int* sl, const int* ss, const int* ci,
                      const T* v, const T* b, int64_t bs, T* x, int64_t xs, T alpha,
                      const T* alpha_dev, T beta, const T* beta_dev, const T* xin, int64_t xins,
                      void* stream) {
    if (n == 0) return B200SP_OK;
    B200SP_REQUIRE(slice_size > 0, B200SP_EINVAL, "sellp: slice_size must be positive");
    cudaStream_t st = as_stream(stream);
    Coef<T> al = coef(alpha, alpha_dev), be = coef(beta, beta_dev);
    if (slice_size == 64) {
        if (xin) launch_sellp<T, true, 64>(n, slice_size, sl, ss, ci, v, b, bs, x, xs, al, be, xin, xins, st);
        else launch_sellp<T, false, 64>(n, slice_size, sl, ss, ci, v, b, bs, x, xs, al, be, xin, xins, st);
    } else {
        if (xin) launch_sellp<T, true, 0>(n, slice_size, sl, ss, ci, v, b, bs, x, xs, al, be, xin, xins, st);
        else launch_sellp<T, false, 0>(n, slice_size, sl, ss, ci, v, b, bs, x, xs, al, be, xin, xins, st);
    }
    count_launch();
    return check_launch("sellp_spmv");
}

// ===========================================================================
// Matrix-free tridiagonal stencil (StencilMatrix; StencilApplyKernel,
// src/kernels.py:335-363): x_i = c b_i, then += l b_{i-1}, then += r b_{i+1},
// each product rounded before its add as in the reference's NumPy passes.
// ===========================================================================
template <typename T>
__global__ void stencil3_kernel(int64_t n, int m, T l, T c, T r, const T* __restrict__ b, int64_t bs,
                                T* __restrict__ x, int64_t xs) {
    const int64_t tot = n * m;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / m, j = t - i * m;
        T v = mul_rn(c, b[i * bs + j]);
        if (i > 0) v = v + mul_rn(l, b[(i - 1) * bs + j]);
        if (i < n - 1) v = v + mul_rn(r, b[(i + 1) * bs + j]);
        x[i * xs + j] = v;
    }
}

// ===========================================================================
// Dense (n, k) row-major times b: warp per row (DenseSpmvKernel,
// src/kernels.py:319-332; small operators only, not a performance target)
// ===========================================================================
template <typename T>
__global__ void dense_spmv_kernel(int64_t n, int64_t k, const T* __restrict__ a, int64_t as,
                                  const T* __restrict__ b, int64_t bs, T* __restrict__ x, int64_t xs) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n; r += nw) {
        T s = 0;
        for (int64_t j = lane; j < k; j += 32) s += a[r * as + j] * b[j * bs];
        s = warp_sum(s);
        if (lane == 0) x[r * xs] = s;
    }
}

template <typename T>
static int dense_spmv(int64_t n, int64_t k, const T* a, int64_t as, const T* b, int64_t bs, T* x,
                      int64_t xs, void* stream) {
    if (n == 0) return B200SP_OK;
    dense_spmv_kernel<T><<<grid_for(n * 32, 256, 8), 256, 0, as_stream(stream)>>>(n, k, a, as, b, bs, x, xs);
    count_launch();
    return check_launch("dense_spmv");
}

}  // namespace b200sp

// ===========================================================================
// C ABI
// ===========================================================================
using namespace b200sp;

#define SPMV_TAIL_ARGS(T) T alpha, const T *alpha_dev, T beta, const T *beta_dev, const T *x_in, int64_t x_in_stride, void *stream

extern "C" {

int b200sp_csr_spmv_classical_f64(int64_t n, const int32_t* rp, const int32_t* ci, const double* v,
                                  const double* b, int64_t bs, double* x, int64_t xs, double alpha,
                                  const double* alpha_dev, double beta, const double* beta_dev,
                                  const double* xin, int64_t xins, int32_t subwarp, void* stream) {
    return csr_classical<double>(n, rp, ci, v, b, bs, x, xs, alpha, alpha_dev, beta, beta_dev, xin, xins, subwarp, stream);
}
int b200sp_csr_spmv_classical_f32(int64_t n, const int32_t* rp, const int32_t* ci, const float* v,
                                  const float* b, int64_t bs, float* x, int64_t xs, float alpha,
                                  const float* alpha_dev, float beta, const float* beta_dev,
                                  const float* xin, int64_t xins, int32_t subwarp, void* stream) {
    return csr_classical<float>(n, rp, ci, v, b, bs, x, xs, alpha, alpha_dev, beta, beta_dev, xin, xins, subwarp, stream);
}

int b200sp_csr_spmv_stream_f64(int64_t n, int64_t nnz, const int32_t* rp, const int32_t* ci, const double* v,
                               const double* b, int64_t bs, double* x, int64_t xs, double alpha,
                               const double* alpha_dev, double beta, const double* beta_dev,
                               const double* xin, int64_t xins, int32_t chunk_cap, int32_t tpr, int32_t rpt,
                               int32_t gather_in_reduce, void* stream) {
    return csr_stream<double>(n, nnz, rp, ci, v, b, bs, x, xs, alpha, alpha_dev, beta, beta_dev, xin, xins, chunk_cap,
                              tpr, rpt, gather_in_reduce, stream);
}
int b200sp_csr_spmv_stream_f32(int64_t n, int64_t nnz, const int32_t* rp, const int32_t* ci, const float* v,
                               const float* b, int64_t bs, float* x, int64_t xs, float alpha,
                               const float* alpha_dev, float beta, const float* beta_dev,
                               const float* xin, int64_t xins, int32_t chunk_cap, int32_t tpr, int32_t rpt,
                               int32_t gather_in_reduce, void* stream) {
    return csr_stream<float>(n, nnz, rp, ci, v, b, bs, x, xs, alpha, alpha_dev, beta, beta_dev, xin, xins, chunk_cap,
                             tpr, rpt, gather_in_reduce, stream);
}
int b200sp_csr_spmv_tma_f64(int64_t n, int64_t nnz, const int32_t* rp, const int32_t* ci, const double* v,
                            const double* b, int64_t bs, double* x, int64_t xs, double alpha, const double* alpha_dev,
                            double beta, const double* beta_dev, const double* xin, int64_t xins, int32_t cap,
                            int32_t rpt, int32_t stages, int32_t consumers, int32_t tpr, void* stream) {
    (void)nnz;
    return csr_pipe<double>(n, rp, ci, v, b, bs, x, xs, alpha, alpha_dev, beta, beta_dev, xin, xins, cap, rpt, stages,
                            consumers, tpr, stream);
}
int b200sp_csr_spmv_tma_f32(int64_t n, int64_t nnz, const int32_t* rp, const int32_t* ci, const float* v,
                            const float* b, int64_t bs, float* x, int64_t xs, float alpha, const float* alpha_dev,
                            float beta, const float* beta_dev, const float* xin, int64_t xins, int32_t cap,
                            int32_t rpt, int32_t stages, int32_t consumers, int32_t tpr, void* stream) {
    (void)nnz;
    return csr_pipe<float>(n, rp, ci, v, b, bs, x, xs, alpha, alpha_dev, beta, beta_dev, xin, xins, cap, rpt, stages,
                           consumers, tpr, stream);
}
int64_t b200sp_csr_tma_stage_bytes(int32_t value_bytes, int32_t rows_per_tile, int32_t cap) {
    const int tr = rows_per_tile;
    return value_bytes == 4 ? pipe_stage_bytes<float>(tr, cap) : pipe_stage_bytes<double>(tr, cap);
}
int32_t b200sp_csr_stream_capacity(int32_t value_bytes) {
    return value_bytes == 4 ? StreamCap<float>::v : StreamCap<double>::v;
}

int32_t b200sp_csr_lb_tile(int32_t value_bytes, int32_t mode) {
    (void)value_bytes;
    return mode == 3 ? SEG_CHUNK : lb_tile();
}

int b200sp_csr_seg_plan(int64_t n, int64_t nnz, const int32_t* rp, int32_t* chunk_rows, void* stream) {
    if (n == 0) return B200SP_OK;
    const int64_t nchunks = ceil_div(nnz, SEG_CHUNK);
    csr_seg_plan_kernel<<<(unsigned)ceil_div(nchunks + 1, 256), 256, 0, as_stream(stream)>>>(n, nnz, rp, nchunks,
                                                                                           chunk_rows);
    count_launch();
    return check_launch("csr_seg_plan");
}

int64_t b200sp_csr_lb_num_tiles(int64_t n, int64_t nnz, int32_t tile) { return ceil_div(n + nnz, tile); }

int b200sp_csr_lb_plan(int64_t n, int64_t nnz, const int32_t* rp, int32_t tile, int32_t* coords, void* stream) {
    B200SP_REQUIRE(tile > 0, B200SP_EINVAL, "csr lb plan: tile must be positive");
    const int64_t ntiles = ceil_div(n + nnz, tile);
    csr_lb_plan_kernel<<<(unsigned)ceil_div(ntiles + 1, 256), 256, 0, as_stream(stream)>>>(
        n, nnz, rp, ntiles, tile, coords);
    count_launch();
    return check_launch("csr_lb_plan");
}

int b200sp_csr_spmv_lb_f64(int64_t n, int64_t nnz, const int32_t* rp, const int32_t* ci,
                           const double* v, const double* b, int64_t bs, double* x, int64_t xs,
                           double alpha, const double* alpha_dev, double beta,
                           const double* beta_dev, const double* xin, int64_t xins,
                           const int32_t* coords, int32_t* carry_row, double* carry_val, int32_t tile,
                           int32_t mode, void* stream) {
    if (mode == 3)
        return csr_seg<double>(n, nnz, rp, ci, v, b, bs, x, xs, alpha, alpha_dev, beta, beta_dev, xin, xins, coords,
                               carry_row, carry_val, tile, stream);
    return csr_lb<double>(n, nnz, rp, ci, v, b, bs, x, xs, alpha, alpha_dev, beta, beta_dev, xin, xins, coords,
                          carry_row, carry_val, tile, mode, stream);
}
int b200sp_csr_spmv_lb_f32(int64_t n, int64_t nnz, const int32_t* rp, const int32_t* ci,
                           const float* v, const float* b, int64_t bs, float* x, int64_t xs,
                           float alpha, const float* alpha_dev, float beta, const float* beta_dev,
                           const float* xin, int64_t xins, const int32_t* coords,
                           int32_t* carry_row, float* carry_val, int32_t tile, int32_t mode, void* stream) {
    if (mode == 3)
        return csr_seg<float>(n, nnz, rp, ci, v, b, bs, x, xs, alpha, alpha_dev, beta, beta_dev, xin, xins, coords,
                              carry_row, carry_val, tile, stream);
    return csr_lb<float>(n, nnz, rp, ci, v, b, bs, x, xs, alpha, alpha_dev, beta, beta_dev, xin, xins, coords,
                         carry_row, carry_val, tile, mode, stream);
}

int b200sp_coo_spmv_f64(int64_t nnz, int32_t chunk, const int32_t* rows, const int32_t* cols,
                        const double* vals, const double* b, int64_t bs, double* x, int64_t xs,
                        double alpha, const double* alpha_dev, double beta, const double* beta_dev,
                        const double* xin, int64_t xins, double* carry_head, double* carry_tail,
                        int32_t* chunk_rows, void* stream) {
    return coo_spmv<double>(nnz, chunk, rows, cols, vals, b, bs, x, xs, alpha, alpha_dev, beta, beta_dev, xin, xins, carry_head, carry_tail, chunk_rows, stream);
}
int b200sp_coo_spmv_f32(int64_t nnz, int32_t chunk, const int32_t* rows, const int32_t* cols,
                        const float* vals, const float* b, int64_t bs, float* x, int64_t xs,
                        float alpha, const float* alpha_dev, float beta, const float* beta_dev,
                        const float* xin, int64_t xins, float* carry_head, float* carry_tail,
                        int32_t* chunk_rows, void* stream) {
    return coo_spmv<float>(nnz, chunk, rows, cols, vals, b, bs, x, xs, alpha, alpha_dev, beta, beta_dev, xin, xins, carry_head, carry_tail, chunk_rows, stream);
}

int b200sp_rows_scale_f64(int64_t count, const int32_t* rows, double* x, int64_t xs, double beta,
                          const double* beta_dev, const double* xin, int64_t xins, void* stream) {
    return rows_scale<double>(count, rows, x, xs, beta, beta_dev, xin, xins, stream);
}
int b200sp_rows_scale_f32(int64_t count, const int32_t* rows, float* x, int64_t xs, float beta,
                          const float* beta_dev, const float* xin, int64_t xins, void* stream) {
    return rows_scale<float>(count, rows, x, xs, beta, beta_dev, xin, xins, stream);
}

int b200sp_ell_spmv_f64(int64_t n, int64_t width, int64_t stride, const int32_t* ci, const double* v,
                        const double* b, int64_t bs, double* x, int64_t xs, double alpha,
                        const double* alpha_dev, double beta, const double* beta_dev,
                        const double* xin, int64_t xins, void* stream) {
    return ell_spmv<double>(n, width, stride, ci, v, b, bs, x, xs, alpha, alpha_dev, beta, beta_dev, xin, xins, stream);
}
int b200sp_ell_spmv_f32(int64_t n, int64_t width, int64_t stride, const int32_t* ci, const float* v,
                        const float* b, int64_t bs, float* x, int64_t xs, float alpha,
                        const float* alpha_dev, float beta, const float* beta_dev, const float* xin,
                        int64_t xins, void* stream) {
    return ell_spmv<float>(n, width, stride, ci, v, b, bs, x, xs, alpha, alpha_dev, beta, beta_dev, xin, xins, stream);
}

int b200sp_sellp_spmv_f64(int64_t n, int32_t slice_size, const int32_t* slice_lengths,
                          const int32_t* slice_sets, const int32_t* ci, const double* v,
                          const double* b, int64_t bs, double* x, int64_t xs, double alpha,
                          const double* alpha_dev, double beta, const double* beta_dev,
                          const double* xin, int64_t xins, void* stream) {
    return sellp_spmv<double>(n, slice_size, slice_lengths, slice_sets, ci, v, b, bs, x, xs, alpha, alpha_dev, beta, beta_dev, xin, xins, stream);
}
int b200sp_sellp_spmv_f32(int64_t n, int32_t slice_size, const int32_t* slice_lengths,
                          const int32_t* slice_sets, const int32_t* ci, const float* v,
                          const float* b, int64_t bs, float* x, int64_t xs, float alpha,
                          const float* alpha_dev, float beta, const float* beta_dev,
                          const float* xin, int64_t xins, void* stream) {
    return sellp_spmv<float>(n, slice_size, slice_lengths, slice_sets, ci, v, b, bs, x, xs, alpha, alpha_dev, beta, beta_dev, xin, xins, stream);
}

int b200sp_stencil3_apply_f64(int64_t n, int32_t m, double l, double c, double r, const double* b, int64_t bs,
                              double* x, int64_t xs, void* stream) {
    if (n == 0) return B200SP_OK;
    stencil3_kernel<double><<<grid_for(n * m, 256, 8), 256, 0, as_stream(stream)>>>(n, m, l, c, r, b, bs, x, xs);
    count_launch();
    return check_launch("stencil3_apply");
}
int b200sp_stencil3_apply_f32(int64_t n, int32_t m, float l, float c, float r, const float* b, int64_t bs,
                              float* x, int64_t xs, void* stream) {
    if (n == 0) return B200SP_OK;
    stencil3_kernel<float><<<grid_for(n * m, 256, 8), 256, 0, as_stream(stream)>>>(n, m, l, c, r, b, bs, x, xs);
    count_launch();
    return check_launch("stencil3_apply");
}
int b200sp_dense_spmv_f64(int64_t n, int64_t k, const double* a, int64_t as, const double* b, int64_t bs,
                         double* x, int64_t xs, void* stream) {
    return dense_spmv<double>(n, k, a, as, b, bs, x, xs, stream);
}
int b200sp_dense_spmv_f32(int64_t n, int64_t k, const float* a, int64_t as, const float* b, int64_t bs,
                         float* x, int64_t xs, void* stream) {
    return dense_spmv<float>(n, k, a, as, b, bs, x, xs, stream);
}

}  // extern "C"
