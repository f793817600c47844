// Row-partitioned (distributed) matrix support: ghost-column discovery,
// global -> local column mapping, owned/ghost split of the local rows,
// halo packing, and the control step of the distributed CG.
//
// Layout of a rank's vector: [owned rows (n_local) | ghost values (G)], the
// ghosts sorted by global column (so each neighbour's ghosts are one
// contiguous segment). The local matrix is split into A_own (columns
// < n_local) and A_ghost (columns shifted by -n_local): q = A_own p_own runs
// while the halo exchange is in flight, q += A_ghost p_ghost after it lands.
#include <cuda.h>

#include <cstddef>
#include <cstring>

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

// ---------------------------------------------------------------------------
// Halo exchange through peer memory (CUDA IPC; NVLink / NVSwitch between
// GPUs). The CG step that updates p (CgStep1, steps.py:93-119) also stores
// each boundary row it produces straight into the ghost slots of the
// neighbour that needs it, so the exchange rides on the kernel that
// computes the values -- no pack, no separate transfer. The grid's last CTA
// (ticket) then raises this rank's flag in every destination's flag array
// (release at system scope). A destination's ghost SpMV is ordered after a
// one-thread wait kernel that acquires its flags. Sends must be row ranges
// (slab partitions); buffer reuse across iterations is ordered by the two
// all-reduces every iteration performs.
// ---------------------------------------------------------------------------
constexpr int PEER_MAX = 4;
struct PeerPut {
    int n;
    int64_t lo[PEER_MAX], hi[PEER_MAX];  // local rows [lo, hi) go to ...
    void* dst[PEER_MAX];                 // ... the peer's ghost slots (mapped peer memory)
    int* flag[PEER_MAX];                 // this rank's flag slot in the peer's flag array
};
struct PeerWait {
    int n;
    const int* flag[2 * PEER_MAX];
};

__device__ __forceinline__ void st_release_sys(int* p, int v) {
    asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire_sys(const int* p) {
    int v;
    asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

template <typename T>
__global__ void __launch_bounds__(256)
cg_step1_put_kernel(int64_t n, T* __restrict__ p, const T* __restrict__ z, const KrylovCtl* c, PeerPut pp,
                    int epoch, unsigned* ticket, int* epoch_dev) {
    if (c->done) return;
    // device-managed epoch (CUDA-graph replays): this launch's = stored + 1,
    // published by the last CTA once every CTA has read the old value
    if (epoch_dev) epoch = *(volatile int*)epoch_dev + 1;
    const T beta = (T)c->beta;
    bool wrote = false;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const T v = z[i] + beta * p[i];
        p[i] = v;
#pragma unroll
        for (int k = 0; k < PEER_MAX; ++k)
            if (k < pp.n && i >= pp.lo[k] && i < pp.hi[k]) {
                static_cast<T*>(pp.dst[k])[i - pp.lo[k]] = v;
                wrote = true;
            }
    }
    if (wrote) __threadfence_system();  // this thread's peer stores before the CTA's arrival
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned t = atomicAdd(ticket, 1u);
        if (t == gridDim.x - 1) {  // every CTA's stores are out: raise the flags
            __threadfence_system();
            *ticket = 0;
            for (int k = 0; k < pp.n; ++k) st_release_sys(pp.flag[k], epoch);
            if (epoch_dev) *epoch_dev = epoch;
        }
    }
}

// All-reduce of the k <= 4 local sums parked in ctl.red, through peer
// memory: one thread stores them into slot [parity][rank] of every rank's
// slot array (its own included), raises its flag there, waits for every
// rank's flag and sums the slots in rank order -- the same order on every
// rank, so every rank gets the identical result (as with NCCL). Slots are
// double-buffered by epoch parity: a rank can only write epoch e+1 after
// every rank raised e+1's predecessor flag, i.e. finished reading epoch e-1.
constexpr int PEER_RED_MAX = 8;
struct PeerRed {
    int world, rank;
    double* slots[PEER_RED_MAX];  // every rank's slot array (mapped; own local)
    int* flags[PEER_RED_MAX];     // every rank's flag array
};

// Every spin on a peer's flag is bounded (b200sp_set_tuning("peer_timeout_ms"),
// default 30 s): a rank that died between its store and the matching wait
// must not leave the surviving GPUs spinning in a kernel that never returns.
// On timeout the wait marks the solve as broken down (BD_PEER_TIMEOUT, the
// host reports a failed solve) and the all-reduce returns NaN sums.
__device__ __forceinline__ bool spin_until(const int* flag, int epoch, unsigned long long deadline, int ns) {
    while (ld_acquire_sys(flag) < epoch) {
        if (global_ns() > deadline) return false;
        __nanosleep(ns);
    }
    return true;
}

__global__ void peer_allreduce_kernel(double* red, int k, PeerRed pr, int epoch, unsigned long long timeout_ns,
                                      int* epoch_dev) {
    if (epoch_dev) epoch = *epoch_dev + 1;
    const int par = epoch & 1;
    double v[4];
    for (int i = 0; i < k; ++i) v[i] = red[i];
    for (int j = 0; j < pr.world; ++j) {
        double* dst = pr.slots[j] + ((size_t)par * pr.world + pr.rank) * 4;
        for (int i = 0; i < k; ++i) dst[i] = v[i];
    }
    __threadfence_system();
    for (int j = 0; j < pr.world; ++j) st_release_sys(pr.flags[j] + pr.rank, epoch);
    const int* mine = pr.flags[pr.rank];
    const unsigned long long deadline = global_ns() + timeout_ns;
    for (int j = 0; j < pr.world; ++j)
        if (!spin_until(mine + j, epoch, deadline, 64)) {
            for (int i = 0; i < k; ++i) red[i] = __longlong_as_double(0x7ff8000000000000ll);
            return;
        }
    const volatile double* sl = pr.slots[pr.rank] + (size_t)par * pr.world * 4;
    for (int i = 0; i < k; ++i) {
        double s = 0;
        for (int j = 0; j < pr.world; ++j) s += sl[j * 4 + i];
        red[i] = s;
    }
    if (epoch_dev) *epoch_dev = epoch;
}

// ---------------------------------------------------------------------------
// Plain distributed SpMV through peer memory (DistCsr.apply_peer): no CG step
// precedes the SpMV, so a copy kernel puts the boundary rows of x straight
// into the neighbours' ghost slots. Ghost-slot reuse is ordered by ACK flags
// (no all-reduce separates two SpMVs): before writing epoch e, every CTA
// waits until each destination has acknowledged epoch e - 1 (it finished its
// ghost SpMV); after its ghost SpMV a rank raises its ack in every source's
// ack array. Epochs live on the device, so the step is graph-capturable.
// ---------------------------------------------------------------------------
struct PeerAck {
    int n;
    const int* wait[PEER_MAX];  // my slot in each destination's ack array... read side: acks FROM destinations
};

template <typename T>
__global__ void __launch_bounds__(256)
peer_put_kernel(const T* __restrict__ xo, PeerPut pp, PeerAck acks, int* epoch_dev, unsigned* ticket,
                unsigned long long timeout_ns) {
    __shared__ int s_epoch, s_ok;
    if (threadIdx.x == 0) {
        const int e = *(volatile int*)epoch_dev + 1;
        s_epoch = e;
        s_ok = 1;
        const unsigned long long deadline = global_ns() + timeout_ns;
        for (int k = 0; k < acks.n; ++k)
            while (ld_acquire_sys(acks.wait[k]) < e - 1) {
                if (global_ns() > deadline) {
                    s_ok = 0;
                    break;
                }
                __nanosleep(64);
            }
    }
    __syncthreads();
    const int epoch = s_epoch;
    if (!s_ok) return;  // a destination stopped responding: the flags stay low, the receiver's wait times out
    bool wrote = false;
    for (int k = 0; k < pp.n; ++k) {
        const int64_t cnt = pp.hi[k] - pp.lo[k];
        T* dst = static_cast<T*>(pp.dst[k]);
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x) {
            dst[i] = xo[pp.lo[k] + i];
            wrote = true;
        }
    }
    if (wrote) __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned t = atomicAdd(ticket, 1u);
        if (t == gridDim.x - 1) {
            __threadfence_system();
            *ticket = 0;
            for (int k = 0; k < pp.n; ++k) st_release_sys(pp.flag[k], epoch);
            *epoch_dev = epoch;
        }
    }
}

// after the ghost SpMV: acknowledge epoch *epoch_dev to every source
__global__ void peer_ack_kernel(PeerWait ackout, const int* epoch_dev) {
    const int e = *(volatile const int*)epoch_dev;
    for (int k = 0; k < ackout.n; ++k) st_release_sys(const_cast<int*>(ackout.flag[k]), e);
}

// wait for the sources' flags of the current epoch (no solver control block)
__global__ void peer_wait_plain_kernel(PeerWait w, const int* epoch_dev, unsigned long long timeout_ns) {
    const int e = *(volatile const int*)epoch_dev;
    const unsigned long long deadline = global_ns() + timeout_ns;
    for (int k = 0; k < w.n; ++k)
        while (ld_acquire_sys(w.flag[k]) < e) {
            if (global_ns() > deadline) return;
            __nanosleep(64);
        }
}

__global__ void peer_wait_kernel(KrylovCtl* c, PeerWait w, int epoch, unsigned long long timeout_ns,
                                 const int* epoch_dev) {
    if (c->done) return;
    if (epoch_dev) epoch = *(volatile const int*)epoch_dev;  // this rank's put of the same step published it
    const unsigned long long deadline = global_ns() + timeout_ns;
    for (int k = 0; k < w.n; ++k)
        if (!spin_until(w.flag[k], epoch, deadline, 256)) {
            c->breakdown = BD_PEER_TIMEOUT;
            c->breakdown_it = c->it + 1;
            c->done = 1;
            return;
        }
}

inline unsigned long long peer_timeout_ns() {
    return (unsigned long long)tuning("peer_timeout_ms", 30000) * 1000000ull;
}

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

int32_t b200sp_peer_max(void) { return PEER_MAX; }

#define PEER_PUT_DEF(SUF, T)                                                                                  \
    int b200sp_cg_step1_put_##SUF(int64_t n, T* p, const T* z, const void* ctl, int32_t nput, const int64_t* lo, \
                                  const int64_t* hi, void* const* dst, int32_t* const* flag, int32_t epoch,     \
                                  uint32_t* ticket, int32_t* epoch_dev, void* stream) {                         \
        B200SP_REQUIRE(nput >= 0 && nput <= PEER_MAX, B200SP_EINVAL, "cg_step1_put: at most %d peers (got %d)", \
                       PEER_MAX, nput);                                                                         \
        B200SP_REQUIRE(epoch > 0 || epoch_dev, B200SP_EINVAL, "cg_step1_put: epoch must be positive");         \
        if (n <= 0) return B200SP_OK;                                                                           \
        PeerPut pp{};                                                                                           \
        pp.n = nput;                                                                                            \
        for (int k = 0; k < nput; ++k) {                                                                        \
            pp.lo[k] = lo[k];                                                                                   \
            pp.hi[k] = hi[k];                                                                                   \
            pp.dst[k] = dst[k];                                                                                 \
            pp.flag[k] = flag[k];                                                                               \
        }                                                                                                       \
        cg_step1_put_kernel<T><<<grid_for(n, 256, 8), 256, 0, as_stream(stream)>>>(n, p, z, (const KrylovCtl*)ctl, \
                                                                                    pp, epoch, ticket, epoch_dev); \
        count_launch();                                                                                         \
        return check_launch("cg_step1_put");                                                                    \
    }
PEER_PUT_DEF(f64, double)
PEER_PUT_DEF(f32, float)
#undef PEER_PUT_DEF

int b200sp_peer_allreduce(double* red, int32_t k, int32_t world, int32_t rank, double* const* slots,
                          int32_t* const* flags, int32_t epoch, int32_t* epoch_dev, void* stream) {
    B200SP_REQUIRE(k >= 1 && k <= 4, B200SP_EINVAL, "peer_allreduce: 1..4 values (got %d)", k);
    B200SP_REQUIRE(world >= 1 && world <= PEER_RED_MAX && rank >= 0 && rank < world, B200SP_EINVAL,
                   "peer_allreduce: world must be 1..%d (got %d, rank %d)", PEER_RED_MAX, world, rank);
    B200SP_REQUIRE(epoch > 0 || epoch_dev, B200SP_EINVAL, "peer_allreduce: epoch must be positive");
    PeerRed pr{};
    pr.world = world;
    pr.rank = rank;
    for (int j = 0; j < world; ++j) {
        pr.slots[j] = slots[j];
        pr.flags[j] = flags[j];
    }
    peer_allreduce_kernel<<<1, 1, 0, as_stream(stream)>>>(red, k, pr, epoch, peer_timeout_ns(), epoch_dev);
    count_launch();
    return check_launch("peer_allreduce");
}

#define PEER_PUT_X(SUF, T)                                                                                    \
    int b200sp_peer_put_##SUF(const T* x_owned, int32_t nput, const int64_t* lo, const int64_t* hi,            \
                              void* const* dst, int32_t* const* flag, int32_t nack, const int32_t* const* ack_in, \
                              int32_t* epoch_dev, uint32_t* ticket, void* stream) {                             \
        B200SP_REQUIRE(nput >= 0 && nput <= PEER_MAX && nack >= 0 && nack <= PEER_MAX, B200SP_EINVAL,           \
                       "peer_put: at most %d peers", PEER_MAX);                                                 \
        PeerPut pp{};                                                                                           \
        pp.n = nput;                                                                                            \
        int64_t most = 0;                                                                                       \
        for (int k = 0; k < nput; ++k) {                                                                        \
            pp.lo[k] = lo[k];                                                                                   \
            pp.hi[k] = hi[k];                                                                                   \
            pp.dst[k] = dst[k];                                                                                 \
            pp.flag[k] = flag[k];                                                                               \
            most = hi[k] - lo[k] > most ? hi[k] - lo[k] : most;                                                 \
        }                                                                                                       \
        PeerAck a{};                                                                                            \
        a.n = nack;                                                                                             \
        for (int k = 0; k < nack; ++k) a.wait[k] = ack_in[k];                                                   \
        const unsigned grid = (unsigned)(most > 0 ? grid_for(most, 256, 4) : 1);                                \
        peer_put_kernel<T><<<grid, 256, 0, as_stream(stream)>>>(x_owned, pp, a, epoch_dev, ticket,              \
                                                               peer_timeout_ns());                              \
        count_launch();                                                                                         \
        return check_launch("peer_put");                                                                        \
    }
PEER_PUT_X(f64, double)
PEER_PUT_X(f32, float)
#undef PEER_PUT_X

int b200sp_peer_ack(int32_t nack, const int32_t* const* ack_out, const int32_t* epoch_dev, void* stream) {
    B200SP_REQUIRE(nack >= 0 && nack <= 2 * PEER_MAX, B200SP_EINVAL, "peer_ack: at most %d sources", 2 * PEER_MAX);
    if (nack == 0) return B200SP_OK;
    PeerWait w{};
    w.n = nack;
    for (int k = 0; k < nack; ++k) w.flag[k] = ack_out[k];
    peer_ack_kernel<<<1, 1, 0, as_stream(stream)>>>(w, epoch_dev);
    count_launch();
    return check_launch("peer_ack");
}

int b200sp_peer_wait_plain(int32_t nwait, const int32_t* const* flags, const int32_t* epoch_dev, void* stream) {
    B200SP_REQUIRE(nwait >= 0 && nwait <= 2 * PEER_MAX, B200SP_EINVAL, "peer_wait_plain: at most %d flags",
                   2 * PEER_MAX);
    if (nwait == 0) return B200SP_OK;
    PeerWait w{};
    w.n = nwait;
    for (int k = 0; k < nwait; ++k) w.flag[k] = flags[k];
    peer_wait_plain_kernel<<<1, 1, 0, as_stream(stream)>>>(w, epoch_dev, peer_timeout_ns());
    count_launch();
    return check_launch("peer_wait_plain");
}

int b200sp_peer_wait(void* ctl, int32_t nwait, const int32_t* const* flags, int32_t epoch, const int32_t* epoch_dev,
                     void* stream) {
    B200SP_REQUIRE(nwait >= 0 && nwait <= 2 * PEER_MAX, B200SP_EINVAL, "peer_wait: at most %d flags (got %d)",
                   2 * PEER_MAX, nwait);
    if (nwait == 0) return B200SP_OK;
    PeerWait w{};
    w.n = nwait;
    for (int k = 0; k < nwait; ++k) w.flag[k] = flags[k];
    peer_wait_kernel<<<1, 1, 0, as_stream(stream)>>>((KrylovCtl*)ctl, w, epoch, peer_timeout_ns(), epoch_dev);
    count_launch();
    return check_launch("peer_wait");
}

// ---- CUDA IPC + peer access (the peer-memory halo / all-reduce setup) ------
// Buffers are exported as (allocation handle, offset) and opened in the
// CALLER's current device context with lazy peer access: no CUDA context is
// created on the owner's device. Peer access is enabled explicitly first so
// that a topology without P2P is detected (and the host falls back to NCCL)
// instead of failing inside a kernel.
typedef CUresult (*PfnMemGetAddressRange)(CUdeviceptr*, size_t*, CUdeviceptr);

static PfnMemGetAddressRange address_range_fn() {
    static PfnMemGetAddressRange fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PfnMemGetAddressRange)p;
    }
    return fn;
}

int32_t b200sp_ipc_handle_bytes(void) { return (int32_t)sizeof(cudaIpcMemHandle_t); }

int b200sp_ipc_export(const void* ptr, void* handle, int64_t* offset) {
    PfnMemGetAddressRange range = address_range_fn();
    B200SP_REQUIRE(range != nullptr, B200SP_ECUDA, "ipc_export: cuMemGetAddressRange unavailable");
    CUdeviceptr base = 0;
    size_t size = 0;
    B200SP_REQUIRE(range(&base, &size, (CUdeviceptr)ptr) == CUDA_SUCCESS, B200SP_ECUDA,
                   "ipc_export: %p is not device memory", ptr);
    cudaIpcMemHandle_t h;
    B200SP_CHECK_CUDA(cudaIpcGetMemHandle(&h, (void*)base));
    std::memcpy(handle, &h, sizeof(h));
    *offset = (int64_t)((CUdeviceptr)ptr - base);
    return B200SP_OK;
}

int b200sp_ipc_open(const void* handle, int64_t offset, void** ptr, void** base) {
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    void* b = nullptr;
    B200SP_CHECK_CUDA(cudaIpcOpenMemHandle(&b, h, cudaIpcMemLazyEnablePeerAccess));
    *base = b;
    *ptr = (char*)b + offset;
    return B200SP_OK;
}

int b200sp_ipc_close(void* base) {
    B200SP_CHECK_CUDA(cudaIpcCloseMemHandle(base));
    return B200SP_OK;
}

// can = 1 when the current device can load/store `peer`'s memory (same
// device, or cudaDeviceCanAccessPeer); peer access is then enabled
int b200sp_peer_enable(int32_t peer, int32_t* can) {
    int cur = 0;
    B200SP_CHECK_CUDA(cudaGetDevice(&cur));
    if (peer == cur) {
        *can = 1;
        return B200SP_OK;
    }
    int ok = 0;
    B200SP_CHECK_CUDA(cudaDeviceCanAccessPeer(&ok, cur, peer));
    *can = ok;
    if (!ok) return B200SP_OK;
    const cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) {
        (void)cudaGetLastError();
        return B200SP_OK;
    }
    B200SP_CHECK_CUDA(e);
    return B200SP_OK;
}

}  // extern "C"
