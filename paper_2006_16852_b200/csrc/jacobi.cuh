// Block-Jacobi storage and the warp-per-block apply used by the solvers.
//
// Reference: _JacobiApplyKernel / JacobiOperator (src/precond.py:98-152):
// z_blk = inv_blk (widened to f64) @ r_blk, per diagonal block.
// Layout in HBM: block b (rows starts[b] .. starts[b+1]-1, size <= 32) stores
// its inverse column-major -- element (row l, col c) at c*bs + l -- at byte
// offset offs[b], in fp64 (prec 0) or fp32 (prec 1, adaptive precision).
// A warp owns a block, lane l owns row l: each step c broadcasts r[c] with a
// shuffle and reads one fully coalesced column of the inverse.
#pragma once

#include "common.cuh"

namespace b200sp {

struct JacobiView {
    int64_t nblocks;                  // 0 => identity (no preconditioner)
    const int* starts;                // nblocks + 1
    const long long* offs;            // byte offset of each block's inverse
    const unsigned char* prec;        // 0 = fp64 storage, 1 = fp32 storage
    const unsigned char* storage;
};

// Row blocks walked by warps: Jacobi blocks, or 32-row chunks without one.
struct RowBlocks {
    int64_t n;
    JacobiView J;
    __device__ __forceinline__ int64_t count() const { return J.nblocks ? J.nblocks : (n + 31) / 32; }
    __device__ __forceinline__ void range(int64_t b, int64_t& r0, int& bs) const {
        if (J.nblocks) {
            r0 = J.starts[b];
            bs = J.starts[b + 1] - (int)r0;
        } else {
            r0 = b * 32;
            bs = (int)min((int64_t)32, n - r0);
        }
    }
};

// z for this lane's row of block b given this lane's r value (0 for lanes
// beyond the block). Sequential in c.
template <typename T>
__device__ __forceinline__ T jacobi_row(const JacobiView& J, int64_t b, int bs, int lane, T rv) {
    const unsigned char* base = J.storage + J.offs[b];
    T acc = 0;
    if (bs == 32 && J.prec[b] == 0) {
        // full fp64 block: 8 columns' loads in flight per lane before their
        // FMAs (the loop form kept about two in flight: 4.4-4.8 TB/s under
        // ncu); same products, same order
        const double* inv = reinterpret_cast<const double*>(base);
#pragma unroll
        for (int c0 = 0; c0 < 32; c0 += 8) {
            double iv[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) iv[j] = ld_stream(inv + (c0 + j) * 32 + lane);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const T rc = __shfl_sync(0xffffffffu, rv, c0 + j);
                acc += (T)iv[j] * rc;
            }
        }
    } else if (bs == 32) {  // full fp32-stored block (adaptive precision): the same batching
        const float* inv = reinterpret_cast<const float*>(base);
#pragma unroll
        for (int c0 = 0; c0 < 32; c0 += 8) {
            float iv[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) iv[j] = ld_stream(inv + (c0 + j) * 32 + lane);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const T rc = __shfl_sync(0xffffffffu, rv, c0 + j);
                acc += (T)(double)iv[j] * rc;
            }
        }
    } else if (J.prec[b] == 0) {
        const double* inv = reinterpret_cast<const double*>(base);
        for (int c = 0; c < bs; ++c) {
            const T rc = __shfl_sync(0xffffffffu, rv, c);
            if (lane < bs) acc += (T)ld_stream(inv + c * bs + lane) * rc;
        }
    } else {
        const float* inv = reinterpret_cast<const float*>(base);
        for (int c = 0; c < bs; ++c) {
            const T rc = __shfl_sync(0xffffffffu, rv, c);
            if (lane < bs) acc += (T)(double)ld_stream(inv + c * bs + lane) * rc;
        }
    }
    return acc;
}

}  // namespace b200sp
