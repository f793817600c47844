// Grid-barrier latency probe for the persistent cooperative solvers (C1).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/barrier_probe tools/barrier_probe.cu
//   /tmp/barrier_probe
//
// Times, per barrier, (a) cooperative_groups grid.sync(), (b) a counter
// barrier (one relaxed atomicAdd per CTA + acquire spin on the counter), and
// (c) (b) plus the deterministic partial-sum exchange the solvers do (every
// CTA writes one double, after the barrier warp 0 of every CTA reads all of
// them), (d) the last arriver releasing everyone through one flag, and (e)
// the flag-in-data slot exchange with no atomic (k_ll), for several grid
// shapes. Results: profiles/r03_barrier_probe.txt.
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>

namespace cg = cooperative_groups;

__global__ void k_gridsync(int iters) {
    cg::grid_group g = cg::this_grid();
    for (int i = 0; i < iters; ++i) g.sync();
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_release(unsigned* p, unsigned v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// monotone counter barrier: the k-th barrier completes when the counter
// reaches k * gridDim.x
__device__ __forceinline__ void ctr_barrier(unsigned* ctr, unsigned& target) {
    __syncthreads();
    target += gridDim.x;
    if (threadIdx.x == 0) {
        red_release(ctr, 1u);
        while ((int)(ld_acquire(ctr) - target) < 0) {
        }
    }
    __syncthreads();
}

__global__ void k_ctr(int iters, unsigned* ctr) {
    unsigned target = 0;
    for (int i = 0; i < iters; ++i) ctr_barrier(ctr, target);
}

__global__ void k_ctr_part(int iters, unsigned* ctr, double* part, double* out) {
    unsigned target = 0;
    __shared__ double tot;
    double acc = 0;
    for (int i = 0; i < iters; ++i) {
        double* pp = part + (i & 1) * 1024;
        if (threadIdx.x == 0) pp[blockIdx.x] = (double)(blockIdx.x + i);
        ctr_barrier(ctr, target);
        if (threadIdx.x < 32) {
            double s = 0;
            for (int b = threadIdx.x; b < (int)gridDim.x; b += 32) s += ((volatile double*)pp)[b];
            for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if (threadIdx.x == 0) tot = s;
        }
        __syncthreads();
        acc += tot;
    }
    if (threadIdx.x == 0 && blockIdx.x == 0) *out = acc;
}

// all CTAs poll a flag that the last arriver flips (one atomicAdd returns the
// arrival order; the last CTA releases everyone with one store)
__global__ void k_flag(int iters, unsigned* ctr, unsigned* flag) {
    for (int i = 0; i < iters; ++i) {
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned old;
            asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(ctr) : "memory");
            if (old == (unsigned)(i + 1) * gridDim.x - 1) {
                asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flag), "r"((unsigned)(i + 1)) : "memory");
            } else {
                while (ld_acquire(flag) < (unsigned)(i + 1)) {
                }
            }
        }
        __syncthreads();
    }
}

// flag-in-data exchange (no atomics): every CTA stores {lo, epoch, hi,
// epoch} of its partial into its own 16-byte slot; every CTA's warp 0 polls
// all slots until every epoch matches (two slot sets, by epoch parity), then sums the partials in CTA order.
// Each aligned 8-byte half is single-copy atomic, so a matching epoch means
// the data half beside it is from the same store. FENCE adds the
// release/acquire pair a phase needs when other CTAs read its vector writes.
template <bool FENCE>
__global__ void k_ll(int iters, uint4* slots, double* out) {
    __shared__ double tot;
    double acc = 0;
    for (int i = 0; i < iters; ++i) {
        const unsigned e = (unsigned)i + 1;
        const double mine = (double)(blockIdx.x + i);
        uint4* const set = slots + (i & 1) * 1024;  // double-buffered: a CTA can
        // rewrite a slot set only after every CTA has left the barrier that read it
        __syncthreads();
        if (threadIdx.x == 0) {
            if (FENCE) __threadfence();
            const unsigned long long u = __double_as_longlong(mine);
            asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(set + blockIdx.x),
                         "r"((unsigned)u), "r"(e), "r"((unsigned)(u >> 32)), "r"(e)
                         : "memory");
        }
        if (threadIdx.x < 32) {
            double s = 0;
            for (int b = threadIdx.x; b < (int)gridDim.x; b += 32) {
                unsigned a0, f0, a1, f1;
                do {
                    asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                                 : "=r"(a0), "=r"(f0), "=r"(a1), "=r"(f1)
                                 : "l"(set + b)
                                 : "memory");
                } while (f0 != e || f1 != e);
                s += __longlong_as_double(((unsigned long long)a1 << 32) | a0);
            }
            for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if (FENCE) __threadfence();
            if (threadIdx.x == 0) tot = s;
        }
        __syncthreads();
        acc += tot;
    }
    if (threadIdx.x == 0 && blockIdx.x == 0) *out = acc;
}

// k_ll with the polls of a lane's slots issued together (up to 8 slots per
// lane, 256 CTAs): one round trip per poll round instead of one per slot
template <bool FENCE>
__global__ void k_ll2(int iters, uint4* slots, double* out) {
    __shared__ double tot;
    double acc = 0;
    for (int i = 0; i < iters; ++i) {
        const unsigned e = (unsigned)i + 1;
        const double mine = (double)(blockIdx.x + i);
        uint4* const set = slots + (i & 1) * 1024;
        __syncthreads();
        if (threadIdx.x == 0) {
            if (FENCE) __threadfence();
            const unsigned long long u = __double_as_longlong(mine);
            asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(set + blockIdx.x),
                         "r"((unsigned)u), "r"(e), "r"((unsigned)(u >> 32)), "r"(e)
                         : "memory");
        }
        if (threadIdx.x < 32) {
            double v[8];
            unsigned need = 0;
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (threadIdx.x + 32 * q < (int)gridDim.x) need |= 1u << q;
            while (need) {
                unsigned a0[8], f0[8], a1[8], f1[8];
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    if (need >> q & 1)
                        asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                                     : "=r"(a0[q]), "=r"(f0[q]), "=r"(a1[q]), "=r"(f1[q])
                                     : "l"(set + threadIdx.x + 32 * q)
                                     : "memory");
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    if ((need >> q & 1) && f0[q] == e && f1[q] == e) {
                        v[q] = __longlong_as_double(((unsigned long long)a1[q] << 32) | a0[q]);
                        need &= ~(1u << q);
                    }
            }
            double s = 0;
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (threadIdx.x + 32 * q < (int)gridDim.x) s += v[q];
            for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if (FENCE) __threadfence();
            if (threadIdx.x == 0) tot = s;
        }
        __syncthreads();
        acc += tot;
    }
    if (threadIdx.x == 0 && blockIdx.x == 0) *out = acc;
}

static float time_launch(const void* fn, int grid, int block, void** args, bool coop) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    if (coop)
        cudaLaunchCooperativeKernel(fn, grid, block, args, 0, 0);
    else
        cudaLaunchKernel(fn, grid, block, args, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
    return ms;
}

int main() {
    unsigned *ctr, *flag;
    double *part, *out;
    cudaMalloc(&ctr, 4);
    cudaMalloc(&flag, 4);
    cudaMalloc(&part, 4096 * 8);
    cudaMalloc(&out, 8);
    const int shapes[][2] = {{148, 256}, {256, 256}, {128, 256}, {148, 512}, {64, 256}, {32, 1024}};
    for (auto& s : shapes) {
        const int grid = s[0], block = s[1];
        for (int iters : {10, 2000}) {
            void* a0[] = {&iters};
            float t0 = time_launch((const void*)k_gridsync, grid, block, a0, true);
            cudaMemset(ctr, 0, 4);
            void* a1[] = {&iters, &ctr};
            float t1 = time_launch((const void*)k_ctr, grid, block, a1, true);
            cudaMemset(ctr, 0, 4);
            void* a2[] = {&iters, &ctr, &part, &out};
            float t2 = time_launch((const void*)k_ctr_part, grid, block, a2, true);
            cudaMemset(ctr, 0, 4);
            cudaMemset(flag, 0, 4);
            void* a3[] = {&iters, &ctr, &flag};
            float t3 = time_launch((const void*)k_flag, grid, block, a3, true);
            cudaMemset(part, 0, 4096 * 8);
            void* a4[] = {&iters, &part, &out};
            float t4 = time_launch((const void*)k_ll<false>, grid, block, a4, true);
            double h4 = 0;
            cudaMemcpy(&h4, out, 8, cudaMemcpyDeviceToHost);
            cudaMemset(part, 0, 4096 * 8);
            float t5 = time_launch((const void*)k_ll<true>, grid, block, a4, true);
            double h5 = 0;
            cudaMemcpy(&h5, out, 8, cudaMemcpyDeviceToHost);
            cudaMemset(part, 0, 4096 * 8);
            float t6 = time_launch((const void*)k_ll2<false>, grid, block, a4, true);
            double h6 = 0;
            cudaMemcpy(&h6, out, 8, cudaMemcpyDeviceToHost);
            cudaMemset(part, 0, 4096 * 8);
            float t7 = time_launch((const void*)k_ll2<true>, grid, block, a4, true);
            double h7 = 0;
            cudaMemcpy(&h7, out, 8, cudaMemcpyDeviceToHost);
            double want = 0;
            for (int i = 0; i < iters; ++i) want += (double)grid * (grid - 1) / 2 + (double)grid * i;
            if (iters == 2000)
                printf("grid %4d x %4d: grid.sync %.3f us | counter %.3f us | counter+partials %.3f us | flag %.3f us"
                       " | ll %.3f us (%s) | ll+fence %.3f us (%s)\n",
                       grid, block, t0 * 1e3 / iters, t1 * 1e3 / iters, t2 * 1e3 / iters, t3 * 1e3 / iters,
                       t4 * 1e3 / iters, h4 == want ? "ok" : "WRONG", t5 * 1e3 / iters, h5 == want ? "ok" : "WRONG");
            if (iters == 2000)
                printf("                  ll2 %.3f us (%s) | ll2+fence %.3f us (%s)\n", t6 * 1e3 / iters,
                       h6 == want ? "ok" : "WRONG", t7 * 1e3 / iters, h7 == want ? "ok" : "WRONG");
        }
    }
    return 0;
}
