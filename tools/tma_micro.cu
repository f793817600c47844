// Microbenchmark: 1-D bulk copies (cp.async.bulk global->shared) on B200.
// One CTA per SM streams a large buffer through a ring of `stages` shared
// memory stages; each stage is filled by `copies` bulk copies of equal size.
// Consumers (all threads) touch one word per 16 B of the stage, then release it.
// Reports GB/s for a sweep of (stage bytes, copies per stage, stages).
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/tma_micro.cu -o /tmp/tma_micro
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
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

constexpr int NT = 256;

__global__ void __launch_bounds__(NT + 32, 1)
stream_kernel(const unsigned char* src, int64_t total, int stage_bytes, int copies, int stages, unsigned long long* sink) {
    extern __shared__ __align__(128) unsigned char s_raw[];
    uint64_t* full = reinterpret_cast<uint64_t*>(s_raw);
    uint64_t* empty = full + stages;
    unsigned char* st0 = s_raw + 256;
    const int t = threadIdx.x;
    const int64_t nchunks = total / stage_bytes;
    if (t == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NT / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (t >= NT) {
        if (t != NT) return;
        int it = 0;
        const int per = stage_bytes / copies;
        for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++it) {
            const int s = it % stages;
            if (it >= stages) mbar_wait(&empty[s], (uint32_t)(((it / stages) - 1) & 1));
            mbar_arrive_expect_tx(&full[s], (uint32_t)stage_bytes);
            for (int k = 0; k < copies; ++k)
                tma_load_1d(st0 + (int64_t)s * stage_bytes + k * per, src + c * stage_bytes + k * per, per, &full[s]);
        }
        return;
    }
    unsigned long long acc = 0;
    int it = 0;
    for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++it) {
        const int s = it % stages;
        mbar_wait(&full[s], (uint32_t)((it / stages) & 1));
        const uint32_t* w = reinterpret_cast<const uint32_t*>(st0 + (int64_t)s * stage_bytes);
        for (int i = t; i < stage_bytes / 16; i += NT) acc += w[i * 4];
        __syncwarp();
        if ((t & 31) == 0) mbar_arrive(&empty[s]);
    }
    if (acc == 0x1234567) sink[0] = acc;
}

int main() {
    const int64_t total = 1LL << 30;  // 1 GiB
    unsigned char* src;
    unsigned long long* sink;
    cudaMalloc(&src, total);
    cudaMalloc(&sink, 8);
    cudaMemset(src, 1, total);
    unsigned char* flush;
    cudaMalloc(&flush, 256 << 20);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    const int sizes[] = {4096, 8192, 16384, 32768, 65536, 98304};
    const int copies_l[] = {1, 2, 4, 8};
    const int stages_l[] = {2, 3, 4, 6, 8, 12};
    for (int sb : sizes)
        for (int cp : copies_l)
            for (int ns : stages_l) {
                if (256 + (int64_t)ns * sb > 226 * 1024) continue;
                if (sb / cp < 512) continue;
                float best = 1e30f;
                for (int r = 0; r < 5; ++r) {
                    cudaMemset(flush, r, 256 << 20);
                    cudaEventRecord(e0);
                    stream_kernel<<<148, NT + 32, 256 + ns * sb>>>(src, total, sb, cp, ns, sink);
                    cudaEventRecord(e1);
                    cudaEventSynchronize(e1);
                    float ms;
                    cudaEventElapsedTime(&ms, e0, e1);
                    if (ms < best) best = ms;
                }
                cudaError_t err = cudaGetLastError();
                printf("stage %6d B copies %d stages %2d: %8.1f us %7.1f GB/s %s\n", sb, cp, ns, best * 1e3,
                       total / (best * 1e-3) / 1e9, err == cudaSuccess ? "" : cudaGetErrorString(err));
            }
    return 0;
}
