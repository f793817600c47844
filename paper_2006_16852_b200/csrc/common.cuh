// Shared device helpers for libb200sp (sm_100a).
//
// Everything on this path is HBM-bound integer/FP streaming work: no tensor
// cores. The helpers here are the B200 building blocks every kernel uses:
// streaming (L1::no_allocate, read-only) loads for matrix arrays that are
// touched exactly once per apply, cached read-only loads for the gathered
// input vector (reused across neighbouring rows through L1/L2), warp-shuffle
// reductions and the thread-local error string of the C ABI.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/b200sp.h"

namespace b200sp {

constexpr int kNumSMs = 148;  // B200: 2 dies x 74 SMs
constexpr int kWarp = 32;

// ---------------------------------------------------------------------------
// error plumbing (C ABI returns codes; the message is thread-local)
// ---------------------------------------------------------------------------
void set_error(const char* fmt, ...);
int check_launch(const char* what);
void count_launch(int n = 1);
int tuning(const char* key, int dflt);  // b200sp_set_tuning knobs (sweeps)

#define B200SP_CHECK_CUDA(expr)                                              \
    do {                                                                     \
        cudaError_t _e = (expr);                                             \
        if (_e != cudaSuccess) {                                             \
            ::b200sp::set_error("%s: %s", #expr, cudaGetErrorString(_e));    \
            return B200SP_ECUDA;                                             \
        }                                                                    \
    } while (0)

#define B200SP_REQUIRE(cond, code, ...)                                      \
    do {                                                                     \
        if (!(cond)) {                                                       \
            ::b200sp::set_error(__VA_ARGS__);                                \
            return (code);                                                   \
        }                                                                    \
    } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Grid sized as a multiple of the SM count (grid-stride kernels).
inline int grid_for(int64_t work_items, int block, int per_sm = 8) {
    int64_t g = ceil_div(work_items, block);
    int64_t cap = (int64_t)kNumSMs * per_sm;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (int)g;
}

// ---------------------------------------------------------------------------
// loads
// ---------------------------------------------------------------------------
// Matrix arrays (values, column indices, row pointers) are read exactly once
// per apply: stream them past L1 so L1 stays free for the x gather.
__device__ __forceinline__ double ld_stream(const double* p) {
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ float ld_stream(const float* p) {
    float v;
    asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ int ld_stream(const int* p) {
    int v;
    asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
// 128-bit streaming loads (caller guarantees 16-byte alignment)
__device__ __forceinline__ int4 ld_stream_v4(const int* p) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}
__device__ __forceinline__ double2 ld_stream_v2(const double* p) {
    double2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
    return r;
}
__device__ __forceinline__ float4 ld_stream_v4(const float* p) {
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
    return r;
}
// load E consecutive values (E % 4 == 0, 16-byte aligned) with 128-bit loads
template <int E>
__device__ __forceinline__ void ld_stream_vec(const int* p, int (&out)[E]) {
#pragma unroll
    for (int i = 0; i < E; i += 4) {
        int4 q = ld_stream_v4(p + i);
        out[i] = q.x; out[i + 1] = q.y; out[i + 2] = q.z; out[i + 3] = q.w;
    }
}
template <int E>
__device__ __forceinline__ void ld_stream_vec(const double* p, double (&out)[E]) {
#pragma unroll
    for (int i = 0; i < E; i += 2) {
        double2 q = ld_stream_v2(p + i);
        out[i] = q.x; out[i + 1] = q.y;
    }
}
template <int E>
__device__ __forceinline__ void ld_stream_vec(const float* p, float (&out)[E]) {
#pragma unroll
    for (int i = 0; i < E; i += 4) {
        float4 q = ld_stream_v4(p + i);
        out[i] = q.x; out[i + 1] = q.y; out[i + 2] = q.z; out[i + 3] = q.w;
    }
}
// the same with L1-allocating loads: when a lane's 16-byte pieces leave the
// other half of each 32-byte sector to its next instruction, no_allocate would
// fetch every sector twice from L2
template <int E>
__device__ __forceinline__ void ld_cached_vec(const int* p, int (&out)[E]) {
#pragma unroll
    for (int i = 0; i < E; i += 4) {
        int4 q = __ldg(reinterpret_cast<const int4*>(p + i));
        out[i] = q.x; out[i + 1] = q.y; out[i + 2] = q.z; out[i + 3] = q.w;
    }
}
template <int E>
__device__ __forceinline__ void ld_cached_vec(const double* p, double (&out)[E]) {
#pragma unroll
    for (int i = 0; i < E; i += 2) {
        double2 q = __ldg(reinterpret_cast<const double2*>(p + i));
        out[i] = q.x; out[i + 1] = q.y;
    }
}
template <int E>
__device__ __forceinline__ void ld_cached_vec(const float* p, float (&out)[E]) {
#pragma unroll
    for (int i = 0; i < E; i += 4) {
        float4 q = __ldg(reinterpret_cast<const float4*>(p + i));
        out[i] = q.x; out[i + 1] = q.y; out[i + 2] = q.z; out[i + 3] = q.w;
    }
}
inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
__device__ __forceinline__ bool aligned16_dev(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// Gathered vector entries: read-only path, allocate in L1 (neighbouring rows
// of a stencil share most of their columns).
template <typename T>
__device__ __forceinline__ T ld_gather(const T* p) { return __ldg(p); }

// ---------------------------------------------------------------------------
// scalar coefficients: host value or device pointer (device scalars keep the
// solver loops free of host synchronisation)
// ---------------------------------------------------------------------------
// `guard` (nullable device flag): when it reads non-zero the launch is a
// no-op. Krylov solvers point it at their "done" flag so SpMVs captured in a
// CUDA-graph batch cost nothing once the solve has stopped.
template <typename T>
struct Coef {
    T v;
    const T* p;
    const int* guard;
    __device__ __forceinline__ T get() const { return p ? *p : v; }
    __device__ __forceinline__ bool skip() const { return guard && *(volatile const int*)guard; }
};
const int* current_guard();
template <typename T>
inline Coef<T> coef(T v, const T* p) { return Coef<T>{v, p, current_guard()}; }

// ---------------------------------------------------------------------------
// TMA (bulk async copy) + mbarrier helpers (sm_90+ PTX, used on sm_100a)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
// 1-D bulk copy global -> shared (16-byte aligned, size multiple of 16),
// completion counted on `bar` in bytes
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred P;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n @!P bra WAIT_%=;\n}" ::"r"(
            smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// IEEE products that the compiler may not fuse into a following add
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }

// ---------------------------------------------------------------------------
// warp reductions
// ---------------------------------------------------------------------------
// rows in flight per sub-warp of the classical Csr kernels (spmv.cu, hoststream.cu)
template <int SW> struct ClassicalRows { static constexpr int v = SW >= 32 ? 4 : (SW >= 8 ? 2 : 1); };

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <int SW, typename T>
__device__ __forceinline__ T subwarp_sum(T v) {
#pragma unroll
    for (int o = SW / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Block-wide sum; result valid in thread 0. `sh` needs blockDim/32 slots.
template <typename T>
__device__ __forceinline__ T block_sum(T v, T* sh) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    T r = 0;
    if (wid == 0) {
        const int nw = blockDim.x >> 5;
        r = lane < nw ? sh[lane] : T(0);
        r = warp_sum(r);
    }
    return r;
}

}  // namespace b200sp
