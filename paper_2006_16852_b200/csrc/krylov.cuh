// Shared pieces of the device-resident Krylov solvers.
//
// A solve keeps ALL of its control state on the device (KrylovCtl): the
// iteration counter, per-solve scalars (rho, alpha, omega, ...), the stopping
// status and the stopping criteria. Every reduction ends in a deterministic
// "last block" epilogue (ticket counter, partials summed in block order) that
// also takes the solver's scalar decisions -- the reference's host-side
// _safe_div / breakdown tests / criterion checks (src/solvers/steps.py:21-28,
// src/solvers/krylov.py:56-76, src/stop.py:118-246) -- so a whole batch of
// iterations runs as one CUDA graph with no host round trip.
#pragma once

#include "common.cuh"
#include "jacobi.cuh"

namespace b200sp {

constexpr int KRY_BLOCK = 256;
constexpr int KRY_MAX_GRID = kNumSMs * 8;
constexpr int KRY_MAX_CRIT = 8;
constexpr int KRY_NRED = 4;  // partial-sum slots per reduction

enum CritType : int { CRIT_ITERATION = 1, CRIT_RNR = 2, CRIT_TIME = 3 };
enum Breakdown : int { BD_NONE = 0, BD_CG_SIGMA = 1, BD_RHO = 2, BD_GAMMA = 3, BD_TT = 4, BD_HESSENBERG = 5,
                       BD_PEER_TIMEOUT = 6 };
constexpr int EXACT_CONVERGENCE_ID = 254;  // src/solvers/gmres.py:31

struct KrylovCtl {
    // status (m = 1): src/stop.py:30-31 STOPPING_STATUS_DTYPE
    int it;            // completed iterations (half-iterations for BiCGSTAB)
    int stopped;
    int stopping_id;
    int finalized;
    int done;          // no more work: stopped (and committed) or breakdown
    int breakdown;     // Breakdown code
    int breakdown_it;  // BreakdownInfo.iteration
    int mid_final;     // BiCGSTAB: stopped at the mid check, x += alpha y pending
    int n_crit;
    int needs_residual;
    int hist_cap;
    int jpos;          // GMRES segment position j
    int kdim;          // GMRES restart length
    int committed;     // GMRES: partial segment folded into x
    int pad[2];
    int crit_type[KRY_MAX_CRIT];
    double crit_param[KRY_MAX_CRIT];
    double baseline;   // ||r0||
    double rho, rho_prev, sigma, alpha, beta, omega, gamma, ts, tt, rnorm, snorm, hnorm;
    unsigned ticket[4];
    int dist;          // distributed solve: epilogues park local sums in red[]
    int pad2;
    double red[4];     // local reduction results, all-reduced across ranks in place
    double rho_t;      // FCG: t.z with t = r_new - r_old (src/solvers/krylov.py:80-125)
    unsigned long long t_start;  // %globaltimer (ns) when the solve's control block was initialised
};

__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// One child of Combined: Iteration `it >= max` (src/stop.py:95-106), RNR
// `||r|| <= factor ||r0||` (src/stop.py:187-196), TimeLimit `elapsed >= limit`
// (src/stop.py:134-147) -- all evaluated at EVERY check, on the device: the
// wall clock is the GPU's global nanosecond timer, started by ctl_init.
// A distributed solve needs every rank to take the same decision: each rank
// parks its local "limit reached" flag in red[3] next to its partial sums,
// the all-reduce adds them, and the time child fires on every rank once any
// rank's clock has passed the limit.
__device__ __forceinline__ bool time_expired_local(const KrylovCtl* c, int i) {
    return (double)(global_ns() - c->t_start) >= c->crit_param[i] * 1e9;
}
__device__ __forceinline__ bool crit_fires(const KrylovCtl* c, int i, int it, double nrm) {
    const int t = c->crit_type[i];
    if (t == CRIT_ITERATION) return it >= (int)c->crit_param[i];
    if (t == CRIT_RNR) return nrm <= c->crit_param[i] * c->baseline;
    if (t == CRIT_TIME) return c->dist ? c->red[3] > 0.0 : time_expired_local(c, i);
    return false;
}
// local partial sums of a check phase, parked for the cross-rank all-reduce
__device__ __forceinline__ void park_check(KrylovCtl* c, double s0, double s1) {
    double flag = 0.0;
    for (int i = 0; i < c->n_crit; ++i)
        if (c->crit_type[i] == CRIT_TIME && time_expired_local(c, i)) flag = 1.0;
    c->red[0] = s0;
    c->red[1] = s1;
    c->red[2] = 0.0;
    c->red[3] = flag;
}

// ---------------------------------------------------------------------------
// criteria: Combined ORs the children in order; child i stamps id i+1
// (src/stop.py:226-246); RNR stops when ||r|| <= factor * ||r0||
// (src/stop.py:187-196); Iteration when it >= max (src/stop.py:95-106).
// ---------------------------------------------------------------------------
__device__ inline void crit_check(KrylovCtl* c, int it, double nrm) {
    if (c->stopped) return;
    for (int i = 0; i < c->n_crit; ++i) {
        if (crit_fires(c, i, it, nrm)) {
            c->stopped = 1;
            c->stopping_id = i + 1;
            c->finalized = 1;  // solvers pass set_finalized=True
            return;
        }
    }
}

__device__ __forceinline__ double safe_div(double num, double den) {
    // num/den with 0/0 -> 0 (src/solvers/steps.py:21-28)
    if (den == 0.0 && num == 0.0) return 0.0;
    return num / den;
}

// ---------------------------------------------------------------------------
// deterministic grid reduction of NV values with a last-block epilogue.
// Returns true in thread 0 of the last block, with the totals in `tot`.
// ---------------------------------------------------------------------------
template <int NV>
__device__ bool grid_reduce(double (&v)[NV], double* part, unsigned* ticket, double (&tot)[NV]) {
    __shared__ double sh[KRY_BLOCK / 32];
    __shared__ bool last;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        const double s = block_sum(v[k], sh);
        if (threadIdx.x == 0) part[k * KRY_MAX_GRID + blockIdx.x] = s;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return false;
    __threadfence();
    if (threadIdx.x < 32) {
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            double s = 0;
            for (int b = threadIdx.x; b < (int)gridDim.x; b += 32) s += ((volatile double*)part)[k * KRY_MAX_GRID + b];
            tot[k] = warp_sum(s);
        }
    }
    if (threadIdx.x == 0) *ticket = 0;
    return threadIdx.x == 0;
}

inline int kry_grid(int64_t units, int per_block) {
    int64_t g = ceil_div(units, per_block);
    // knob "kry_grid_div": fewer reduction blocks (a different, equally valid
    // summation partition -- used to measure the solvers' rounding sensitivity)
    const int div = tuning("kry_grid_div", 1);
    const int64_t cap = KRY_MAX_GRID / (div > 1 ? div : 1);
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (int)g;
}

}  // namespace b200sp
