// Row-partitioned (distributed) matrix support: ghost-column discovery,
// global -> local column mapping, owned/ghost split of the local rows,
// halo packing, and the control step of the distributed CG.
//
// Layout of a rank's vector: [owned rows (n_local) | ghost values (G)], the
// ghosts sorted by global column (so each neighbour's ghosts are one
// contiguous segment). The local matrix is split into A_own (columns
// < n_local) and A_ghost (columns shifted by -n_local): q = A_own p_own runs
// while the halo exchange is in flight, q += A_ghost p_ghost after it lands.
#include <cstddef>

#include "krylov.cuh"

namespace b200sp {

__global__ void flag_out_of_range_kernel(int64_t nnz, const int* __restrict__ ci, int64_t lo, int64_t hi,
                                         int* __restrict__ flag) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x)
        flag[k] = (ci[k] < lo || ci[k] >= hi) ? 1 : 0;
}

__global__ void compact_cols_kernel(int64_t nnz, const int* __restrict__ ci, const int* __restrict__ flag,
                                    const int* __restrict__ pos, int* __restrict__ out) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x)
        if (flag[k]) out[pos[k]] = ci[k];
}

// owned column c -> c - lo; ghost column -> n_local + index in the sorted ghost list
__global__ void map_cols_kernel(int64_t nnz, int* __restrict__ ci, int64_t lo, int64_t hi,
                                const int* __restrict__ ghosts, int64_t nghost) {
    const int64_t nl = hi - lo;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = ci[k];
        if (c >= lo && c < hi) {
            ci[k] = (int)(c - lo);
        } else {
            int64_t a = 0, b = nghost;
            while (a < b) {
                const int64_t m = (a + b) >> 1;
                if (ghosts[m] < c) a = m + 1;
                else b = m;
            }
            ci[k] = (int)(nl + a);
        }
    }
}

__global__ void split_count_kernel(int64_t n, const int* __restrict__ rp, const int* __restrict__ ci, int thr,
                                   int* __restrict__ len_lo, int* __restrict__ len_hi) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        int lo = 0, hi = 0;
        for (int k = rp[r]; k < rp[r + 1]; ++k) (ci[k] < thr ? lo : hi)++;
        len_lo[r] = lo;
        len_hi[r] = hi;
    }
}

template <typename T>
__global__ void split_fill_kernel(int64_t n, const int* __restrict__ rp, const int* __restrict__ ci,
                                  const T* __restrict__ v, int thr, const int* __restrict__ rp_lo,
                                  const int* __restrict__ rp_hi, int* __restrict__ ci_lo, T* __restrict__ v_lo,
                                  int* __restrict__ ci_hi, T* __restrict__ v_hi) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        int a = rp_lo[r], b = rp_hi[r];
        for (int k = rp[r]; k < rp[r + 1]; ++k) {
            if (ci[k] < thr) {
                ci_lo[a] = ci[k];
                v_lo[a++] = v[k];
            } else {
                ci_hi[b] = ci[k] - thr;
                v_hi[b++] = v[k];
            }
        }
    }
}

template <typename T>
__global__ void gather_kernel(int64_t count, const int* __restrict__ idx, const T* __restrict__ src,
                              T* __restrict__ dst) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[idx[i]];
}

__global__ void krylov_set_dist_kernel(KrylovCtl* c, int dist) { c->dist = dist; }

}  // namespace b200sp

using namespace b200sp;

#define D_LAUNCH(kernel, work, ...)                                                                   \
    do {                                                                                              \
        if ((work) <= 0) return B200SP_OK;                                                            \
        kernel<<<grid_for((work), 256, 8), 256, 0, as_stream(stream)>>>(__VA_ARGS__);                 \
        count_launch();                                                                               \
        return check_launch(#kernel);                                                                 \
    } while (0)

extern "C" {

int b200sp_flag_out_of_range(int64_t nnz, const int32_t* ci, int64_t lo, int64_t hi, int32_t* flag, void* stream) {
    D_LAUNCH(flag_out_of_range_kernel, nnz, nnz, ci, lo, hi, flag);
}
int b200sp_compact_cols(int64_t nnz, const int32_t* ci, const int32_t* flag, const int32_t* pos, int32_t* out,
                        void* stream) {
    D_LAUNCH(compact_cols_kernel, nnz, nnz, ci, flag, pos, out);
}
int b200sp_map_cols(int64_t nnz, int32_t* ci, int64_t lo, int64_t hi, const int32_t* ghosts, int64_t nghost,
                    void* stream) {
    D_LAUNCH(map_cols_kernel, nnz, nnz, ci, lo, hi, ghosts, nghost);
}
int b200sp_split_count(int64_t n, const int32_t* rp, const int32_t* ci, int32_t thr, int32_t* len_lo,
                       int32_t* len_hi, void* stream) {
    D_LAUNCH(split_count_kernel, n, n, rp, ci, thr, len_lo, len_hi);
}
int b200sp_split_fill_f64(int64_t n, const int32_t* rp, const int32_t* ci, const double* v, int32_t thr,
                          const int32_t* rp_lo, const int32_t* rp_hi, int32_t* ci_lo, double* v_lo, int32_t* ci_hi,
                          double* v_hi, void* stream) {
    D_LAUNCH(split_fill_kernel<double>, n, n, rp, ci, v, thr, rp_lo, rp_hi, ci_lo, v_lo, ci_hi, v_hi);
}
int b200sp_split_fill_f32(int64_t n, const int32_t* rp, const int32_t* ci, const float* v, int32_t thr,
                          const int32_t* rp_lo, const int32_t* rp_hi, int32_t* ci_lo, float* v_lo, int32_t* ci_hi,
                          float* v_hi, void* stream) {
    D_LAUNCH(split_fill_kernel<float>, n, n, rp, ci, v, thr, rp_lo, rp_hi, ci_lo, v_lo, ci_hi, v_hi);
}
int b200sp_gather_f64(int64_t count, const int32_t* idx, const double* src, double* dst, void* stream) {
    D_LAUNCH(gather_kernel<double>, count, count, idx, src, dst);
}
int b200sp_gather_f32(int64_t count, const int32_t* idx, const float* src, float* dst, void* stream) {
    D_LAUNCH(gather_kernel<float>, count, count, idx, src, dst);
}

int b200sp_krylov_set_dist(void* ctl, int32_t dist, void* stream) {
    krylov_set_dist_kernel<<<1, 1, 0, as_stream(stream)>>>((KrylovCtl*)ctl, dist);
    count_launch();
    return check_launch("krylov_set_dist");
}
int64_t b200sp_krylov_red_offset(void) { return (int64_t)offsetof(KrylovCtl, red); }

}  // extern "C"
