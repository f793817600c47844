// Floor of the power-law SpMV (C3): stream 67M column indices + values and
// gather x[col] at random from a 4M-entry (33.5 MB, L2-resident) vector,
// summing per thread -- no row structure at all. Compared with the C3 SpMV
// kernels this separates the random-gather cost from the format overheads.
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/gather_probe.cu -o tools/gather_probe.bin
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void fill(int64_t nnz, int n, int* ci, double* v, unsigned seed) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x) {
        unsigned h = (unsigned)i * 2654435761u ^ seed;
        h ^= h >> 13;
        h *= 0x5bd1e995u;
        h ^= h >> 15;
        ci[i] = (int)(h % (unsigned)n);
        v[i] = 1.0;
    }
}

template <int UNR>
__global__ void gather(int64_t nnz, const int* __restrict__ ci, const double* __restrict__ v,
                       const double* __restrict__ x, double* out) {
    double acc = 0;
    const int64_t st = (int64_t)gridDim.x * blockDim.x;
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    for (; i + (UNR - 1) * st < nnz; i += UNR * st) {
        int c[UNR];
        double w[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            c[u] = __ldg(ci + i + u * st);
            w[u] = __ldg(v + i + u * st);
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) acc += w[u] * __ldg(x + c[u]);
    }
    for (; i < nnz; i += st) acc += v[i] * x[ci[i]];
    if (acc == 12345.678) *out = acc;
}

int main() {
    const int n = 4194304;
    const int64_t nnz = 66685618;
    int* ci;
    double *v, *x, *out;
    cudaMalloc(&ci, nnz * 4);
    cudaMalloc(&v, nnz * 8);
    cudaMalloc(&x, (size_t)n * 8);
    cudaMalloc(&out, 8);
    cudaMemset(x, 0, (size_t)n * 8);
    fill<<<1184, 256>>>(nnz, n, ci, v, 7u);
    unsigned char* flush;
    cudaMalloc(&flush, 256 << 20);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const double bytes = nnz * 12.0 + n * 16.0;  // the Csr-formula algorithmic bytes of C3
    for (int per_sm : {8, 16, 32}) {
        for (int unr : {1, 4, 8}) {
            float best = 1e30f;
            for (int r = 0; r < 5; ++r) {
                cudaMemset(flush, r, 256 << 20);
                cudaEventRecord(a);
                const int grid = 148 * per_sm;
                if (unr == 1) gather<1><<<grid, 256>>>(nnz, ci, v, x, out);
                else if (unr == 4) gather<4><<<grid, 256>>>(nnz, ci, v, x, out);
                else gather<8><<<grid, 256>>>(nnz, ci, v, x, out);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (ms < best) best = ms;
            }
            printf("per_sm %2d unroll %d: %7.1f us  %6.1f G gathers/s  %7.1f GB/s of C3 bytes\n", per_sm, unr,
                   best * 1e3, nnz / (best * 1e-3) / 1e9, bytes / (best * 1e-3) / 1e9);
        }
    }
    return 0;
}
