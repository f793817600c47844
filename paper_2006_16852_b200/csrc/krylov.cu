// Device-resident Krylov iterations: CG, BiCGSTAB, restarted GMRES (m = 1).
//
// Each solver is a fixed sequence of kernels per iteration whose scalar
// control (criteria, breakdown tests, alpha/beta/omega, Givens rotations)
// runs in the last-block epilogue of the reduction that produces its inputs
// (see krylov.cuh). Vectors are contiguous except x / b (user columns, row
// stride xs / bs). Element-wise kernels walk "row blocks" warp-per-block:
// Jacobi blocks when a block-Jacobi preconditioner is present (so z = M r is
// fused into the update that produces r), else 32-row chunks.
//
// Reference loops restated:
//   CG        src/solvers/krylov.py:36-77   + steps.py:87-158
//   BiCGSTAB  src/solvers/krylov.py:190-271 + steps.py:238-243, :348-480
//   GMRES     src/solvers/gmres.py:75-340

#include <cstring>

#include "krylov.cuh"

namespace b200sp {

__device__ __forceinline__ void hist_put(const KrylovCtl* c, double* hist, int it, double v) {
    if (hist && it < c->hist_cap) hist[it] = v;
}

// ===========================================================================
// CG
// ===========================================================================
// control steps (run by the last block, or by cg_finish_kernel after the
// cross-rank all-reduce of a distributed solve)
__device__ inline void cg_init_ctl(KrylovCtl* c, const double* tot, double* hist) {
    c->it = 0;
    c->rho = tot[0];
    c->rho_prev = 1.0;
    c->rnorm = sqrt(tot[1]);
    c->baseline = c->rnorm;
    hist_put(c, hist, 0, c->rnorm);
    crit_check(c, 0, c->rnorm);
    c->done = c->stopped;
    c->beta = safe_div(c->rho, c->rho_prev);
}

__device__ inline void cg_sigma_ctl(KrylovCtl* c, const double* tot) {
    c->sigma = tot[0];
    if (c->sigma <= 0.0 && c->rho != 0.0) {  // krylov.py:64-70
        c->breakdown = BD_CG_SIGMA;
        c->breakdown_it = c->it + 1;
        c->done = 1;
        return;
    }
    c->alpha = safe_div(c->rho, c->sigma);
}

__device__ inline void cg_step2_ctl(KrylovCtl* c, const double* tot, double* hist) {
    c->rho_prev = c->rho;
    c->rho = tot[0];
    c->it += 1;
    c->rnorm = sqrt(tot[1]);
    hist_put(c, hist, c->it, c->rnorm);
    crit_check(c, c->it, c->rnorm);
    c->done = c->stopped;
    c->beta = safe_div(c->rho, c->rho_prev);
}

// after r = b - A x: z = M r, p = 0, rho = r.z, baseline = ||r||, check(0)
template <typename T>
__global__ void __launch_bounds__(KRY_BLOCK)
cg_init_kernel(RowBlocks rb, const T* __restrict__ r, T* __restrict__ z, T* __restrict__ p, KrylovCtl* c,
               double* part, double* hist) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    double rz = 0, rr = 0;
    for (int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < rb.count(); b += nw) {
        int64_t r0;
        int bs;
        rb.range(b, r0, bs);
        const T rv = lane < bs ? r[r0 + lane] : T(0);
        T zv = rv;
        if (rb.J.nblocks) zv = jacobi_row<T>(rb.J, b, bs, lane, rv);
        if (lane < bs) {
            if (rb.J.nblocks) z[r0 + lane] = zv;
            p[r0 + lane] = T(0);
            rz += (double)rv * (double)zv;
            rr += (double)rv * (double)rv;
        }
    }
    double v[2] = {rz, rr}, tot[2];
    if (!grid_reduce<2>(v, part, &c->ticket[0], tot)) return;
    if (c->dist) {
        park_check(c, tot[0], tot[1]);
        return;
    }
    cg_init_ctl(c, tot, hist);
}

// p = z + beta p    (CgStep1, steps.py:93-119)
template <typename T>
__global__ void __launch_bounds__(KRY_BLOCK)
cg_step1_kernel(int64_t n, T* __restrict__ p, const T* __restrict__ z, const KrylovCtl* c) {
    if (c->done) return;
    const T beta = (T)c->beta;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = z[i] + beta * p[i];
}

// sigma = p.q; breakdown if sigma <= 0 and rho != 0 (krylov.py:64-70); alpha
template <typename T>
__global__ void __launch_bounds__(KRY_BLOCK)
cg_sigma_kernel(int64_t n, const T* __restrict__ p, const T* __restrict__ q, KrylovCtl* c, double* part) {
    if (c->done) return;
    double s = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        s += (double)p[i] * (double)q[i];
    double v[1] = {s}, tot[1];
    if (!grid_reduce<1>(v, part, &c->ticket[1], tot)) return;
    if (c->dist) {
        c->red[0] = tot[0];
        return;
    }
    cg_sigma_ctl(c, tot);
}

// x += alpha p; r -= alpha q; z = M r; rho = r.z; ||r||; it++; check   (CgStep2)
template <typename T>
__global__ void __launch_bounds__(KRY_BLOCK)
cg_step2_kernel(RowBlocks rb, T* __restrict__ x, int64_t xs, T* __restrict__ r, const T* __restrict__ p,
                const T* __restrict__ q, T* __restrict__ z, KrylovCtl* c, double* part, double* hist) {
    if (c->done) return;
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const T alpha = (T)c->alpha;
    double rz = 0, rr = 0;
    if (!rb.J.nblocks) {
        // no preconditioner: plain element loop, 4 rows in flight per thread
        const int64_t n = rb.n, st = (int64_t)gridDim.x * blockDim.x;
        int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
        for (; i + 3 * st < n; i += 4 * st) {
            T pv[4], qv[4], xv[4], rv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int64_t k = i + u * st;
                pv[u] = p[k];
                qv[u] = q[k];
                xv[u] = x[k * xs];
                rv[u] = r[k];
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int64_t k = i + u * st;
                x[k * xs] = xv[u] + alpha * pv[u];
                const T nr = rv[u] - alpha * qv[u];
                r[k] = nr;
                rr += (double)nr * (double)nr;
            }
        }
        for (; i < n; i += st) {
            x[i * xs] = x[i * xs] + alpha * p[i];
            const T nr = r[i] - alpha * q[i];
            r[i] = nr;
            rr += (double)nr * (double)nr;
        }
        rz = rr;
    }
    for (int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; rb.J.nblocks && b < rb.count(); b += nw) {
        int64_t r0;
        int bs;
        rb.range(b, r0, bs);
        T rv = T(0);
        if (lane < bs) {
            const int64_t i = r0 + lane;
            x[i * xs] = x[i * xs] + alpha * p[i];
            rv = r[i] - alpha * q[i];
            r[i] = rv;
        }
        T zv = rv;
        if (rb.J.nblocks) {
            zv = jacobi_row<T>(rb.J, b, bs, lane, rv);
            if (lane < bs) z[r0 + lane] = zv;
        }
        rz += (double)rv * (double)zv;
        rr += (double)rv * (double)rv;
    }
    double v[2] = {rz, rr}, tot[2];
    if (!grid_reduce<2>(v, part, &c->ticket[2], tot)) return;
    if (c->dist) {
        park_check(c, tot[0], tot[1]);
        return;
    }
    cg_step2_ctl(c, tot, hist);
}

// ===========================================================================
// FCG (src/solvers/krylov.py:80-125; FcgStep1 = CgStep1 with beta =
// rho_t / prev_rho, FcgStep2 steps.py:167-199). Step 1 and the fused SpMV +
// sigma are CG's; step 2 also forms t = r_new - r_old and reduces
// (r.z, t.z, r.r) for rho, rho_t and the criterion.
// ===========================================================================
__global__ void fcg_init_ctl_kernel(KrylovCtl* c) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {  // fcg_init: prev_rho = 1, rho_t = 0
        c->rho_t = 0.0;
        c->beta = safe_div(0.0, c->rho_prev);
    }
}

template <typename T>
__global__ void __launch_bounds__(KRY_BLOCK)
fcg_step2_kernel(RowBlocks rb, T* __restrict__ x, int64_t xs, T* __restrict__ r, const T* __restrict__ p,
                 const T* __restrict__ q, T* __restrict__ t, T* __restrict__ z, KrylovCtl* c, double* part,
                 double* hist) {
    if (c->done) return;
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const T alpha = (T)c->alpha;
    double rz = 0, tz = 0, rr = 0;
    for (int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < rb.count(); b += nw) {
        int64_t r0;
        int bs;
        rb.range(b, r0, bs);
        T rv = T(0), tv = T(0);
        if (lane < bs) {
            const int64_t i = r0 + lane;
            x[i * xs] = x[i * xs] + mul_rn(alpha, p[i]);
            const T ro = r[i];
            rv = ro - mul_rn(alpha, q[i]);
            tv = rv - ro;
            t[i] = tv;
            r[i] = rv;
        }
        T zv = rv;
        if (rb.J.nblocks) {
            zv = jacobi_row<T>(rb.J, b, bs, lane, rv);
            if (lane < bs) z[r0 + lane] = zv;
        }
        rz += (double)rv * (double)zv;
        tz += (double)tv * (double)zv;
        rr += (double)rv * (double)rv;
    }
    double v[3] = {rz, tz, rr}, tot[3];
    if (!grid_reduce<3>(v, part, &c->ticket[2], tot)) return;
    c->rho_prev = c->rho;
    c->rho = tot[0];
    c->rho_t = tot[1];
    c->it += 1;
    c->rnorm = sqrt(tot[2]);
    hist_put(c, hist, c->it, c->rnorm);
    crit_check(c, c->it, c->rnorm);
    c->done = c->stopped;
    c->beta = safe_div(c->rho_t, c->rho_prev);
}

// distributed solves: the control step after red[] has been all-reduced
// (phase 0 = init, 1 = sigma, 2 = step2)
__global__ void cg_finish_kernel(KrylovCtl* c, double* hist, int phase) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    if (phase != 0 && c->done) return;
    if (phase == 0) cg_init_ctl(c, c->red, hist);
    else if (phase == 1) cg_sigma_ctl(c, c->red);
    else cg_step2_ctl(c, c->red, hist);
}

// ===========================================================================
// Persistent cooperative CG for small systems (C1: 65,536 rows, L2-resident):
// the whole solve is ONE launch. Per iteration three grid-wide barriers:
//   p = z + beta p | q = A p, sigma partials | x, r update, rr partials
// Every block re-sums the per-block partials in the same order, so all blocks
// compute bitwise-identical alpha / beta / stop decisions without another
// barrier; block 0 publishes the status. Same arithmetic as the batched
// kernels above (Csr rows summed left to right per thread).
// ===========================================================================
// Grid-wide exchange for the persistent cooperative kernels: block partials
// -> grid totals with ONE counter barrier (measured 6.1 vs 7.7 us per C1 CG
// iteration against cooperative_groups grid.sync + a separate partial read,
// profiles/r03_coop_c1.txt). Warp 0 holds the block sum after block_sum;
// lane 0 stores it, fences (this block's vector stores, ordered before it by
// the block barrier, and the partial) and arrives on a monotone counter,
// then spins until all gridDim.x CTAs have arrived; warp 0 sums the partials
// in CTA order (so every CTA gets bitwise the same totals) and one block
// barrier broadcasts them. Partial slots alternate between the phases of an
// iteration, so a slot is rewritten only after the next barrier, by which
// time every CTA has read it. The counter is KrylovCtl::ticket[3]: zeroed by
// ctl_init, reset by the last CTA out (coop_exit).
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void coop_arrive_wait(unsigned* ctr, unsigned target) {
    __threadfence();
    atomicAdd(ctr, 1u);
    // acquire polling (measured faster than relaxed polling + one fence)
    while ((int)(ld_acquire_u32(ctr) - target) < 0) {
    }
}
template <int NV>
__device__ __forceinline__ void coop_exchange(double (&v)[NV], double (&tot)[NV], double* part, unsigned* ctr,
                                              unsigned& target, double* sh, double* sh_tot) {
    double bs[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) bs[k] = block_sum(v[k], sh);
    if (gridDim.x == 1) {  // one block: the totals never leave the chip
        if (threadIdx.x == 0)
#pragma unroll
            for (int k = 0; k < NV; ++k) sh_tot[k] = bs[k];
    } else {
        target += gridDim.x;
        if (threadIdx.x < 32) {
            if (threadIdx.x == 0) {
#pragma unroll
                for (int k = 0; k < NV; ++k) part[k * KRY_MAX_GRID + blockIdx.x] = bs[k];
                coop_arrive_wait(ctr, target);
            }
            __syncwarp();
#pragma unroll
            for (int k = 0; k < NV; ++k) {
                double s = 0;
                for (int b = threadIdx.x; b < (int)gridDim.x; b += 32) s += ((volatile double*)part)[k * KRY_MAX_GRID + b];
                s = warp_sum(s);
                if (threadIdx.x == 0) sh_tot[k] = s;
            }
        }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < NV; ++k) tot[k] = sh_tot[k];
}
// plain grid barrier on the same counter
__device__ __forceinline__ void coop_barrier(unsigned* ctr, unsigned& target) {
    __syncthreads();
    if (gridDim.x > 1) {
        target += gridDim.x;
        if (threadIdx.x == 0) coop_arrive_wait(ctr, target);
        __syncthreads();
    }
}
// Exchange with no memory fence, for a barrier after which no CTA reads
// another CTA's vector stores (CG's sigma barrier: the next gathers happen
// only after the rho barrier, whose fence orders them). The partial travels
// in a flagged 16-byte slot {lo, epoch, hi, epoch} (each aligned 8-byte half
// is single-copy atomic, so a matching epoch certifies the data word beside
// it); the counter is only a relaxed hint of when to start reading, and a
// slot whose epoch does not match yet is re-read. Epochs are 1, 2, ... per
// launch; coop_slots_clear zeroes the slots before the first use. One slot
// set suffices when the barriers alternate with fenced ones: a CTA rewrites
// its slot only after the next barrier, when every CTA has read it.
__device__ __forceinline__ void coop_slots_clear(uint4* slots, unsigned* ctr, unsigned& target) {
    if (threadIdx.x == 0) slots[blockIdx.x] = make_uint4(0, 0, 0, 0);
    coop_barrier(ctr, target);
}
__device__ __forceinline__ void coop_exchange_nofence(double v, double& tot, uint4* slots, unsigned epoch, unsigned* ctr,
                                                      unsigned& target, double* sh, double* sh_tot) {
    const double bs = block_sum(v, sh);
    if (gridDim.x == 1) {
        if (threadIdx.x == 0) sh_tot[0] = bs;
    } else {
        target += gridDim.x;
        if (threadIdx.x < 32) {
            if (threadIdx.x == 0) {
                const unsigned long long u = (unsigned long long)__double_as_longlong(bs);
                asm volatile("st.relaxed.gpu.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(slots + blockIdx.x),
                             "r"((unsigned)u), "r"(epoch), "r"((unsigned)(u >> 32)), "r"(epoch)
                             : "memory");
                asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
                unsigned cv;
                do {
                    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(cv) : "l"(ctr) : "memory");
                } while ((int)(cv - target) < 0);
            }
            __syncwarp();
            double s = 0;
            for (int b = threadIdx.x; b < (int)gridDim.x; b += 32) {
                unsigned a0, f0, a1, f1;
                do {
                    asm volatile("ld.relaxed.gpu.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                                 : "=r"(a0), "=r"(f0), "=r"(a1), "=r"(f1)
                                 : "l"(slots + b)
                                 : "memory");
                } while (f0 != epoch || f1 != epoch);
                s += __longlong_as_double((long long)(((unsigned long long)a1 << 32) | a0));
            }
            s = warp_sum(s);
            if (threadIdx.x == 0) sh_tot[0] = s;
        }
    }
    __syncthreads();
    tot = sh_tot[0];
}

// kernel exit: every CTA arrives once more; the last one out resets the
// counter (and, for kernels that keep the control block in shared memory,
// publishes it -- every CTA holds the same copy)
__device__ __forceinline__ void coop_exit(unsigned* ctr, unsigned target, KrylovCtl* c = nullptr,
                                          const KrylovCtl* sc = nullptr) {
    if (threadIdx.x != 0) return;
    if (gridDim.x == 1) {
        if (sc) *c = *sc;
        return;
    }
    __threadfence();
    if (atomicAdd(ctr, 1u) == target + gridDim.x - 1) {
        __threadfence();
        if (sc) {
            *c = *sc;
            c->ticket[3] = 0;
        } else {
            *ctr = 0;
        }
    }
}

__device__ __forceinline__ double fma_t(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ float fma_t(float a, float b, float c) { return __fmaf_rn(a, b, c); }


// Two grid barriers per iteration: p = r + beta p is not a phase of its own
// but recomputed inside the SpMV for every column it gathers (r and the
// previous p of the neighbours are final since the last barrier) and written
// for the thread's own rows into the other of two p buffers -- the same
// fused multiply-add as CgStep1 (steps.py:93-119), so the same values.
template <typename T>
__global__ void __launch_bounds__(KRY_BLOCK)
cg_coop_kernel(int64_t n, const int* __restrict__ rp, const int* __restrict__ ci, const T* __restrict__ av,
               T* __restrict__ x, T* __restrict__ r, T* p_a, T* p_b, T* __restrict__ q, KrylovCtl* c,
               double* part, double* hist) {
    unsigned* const ctr = &c->ticket[3];
    unsigned target = 0;
    __shared__ double sh[KRY_BLOCK / 32];
    __shared__ double sh_tot[2];
    const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t gs = (int64_t)gridDim.x * blockDim.x;
    // initial state comes from cg_init (run before): rho, rho_prev, beta, done
    double rho = c->rho, beta = c->beta;
    int it = c->it;
    bool done = c->done;
    T* pin = p_a;   // p of the previous iteration
    T* pout = p_b;  // p of this one
    while (!done) {
        const T tb = (T)beta;
        double sg = 0;
        for (int64_t i = gt; i < n; i += gs) {
            T s = 0;
            for (int k = rp[i]; k < rp[i + 1]; ++k) {
                const int j = ci[k];
                s += av[k] * fma_t(tb, pin[j], r[j]);
            }
            q[i] = s;
            const T pi = fma_t(tb, pin[i], r[i]);
            pout[i] = pi;
            sg += (double)pi * (double)s;
        }
        double v1[1] = {sg}, t1[1];
        coop_exchange<1>(v1, t1, part, ctr, target, sh, sh_tot);
        const double sigma = t1[0];
        T* const p = pout;
        if (sigma <= 0.0 && rho != 0.0) {  // breakdown (krylov.py:64-70)
            if (gt == 0) {
                c->sigma = sigma;
                c->breakdown = BD_CG_SIGMA;
                c->breakdown_it = it + 1;
                c->done = 1;
            }
            break;
        }
        const double alpha = safe_div(rho, sigma);
        const T ta = (T)alpha;
        double rr = 0;
        for (int64_t i = gt; i < n; i += gs) {
            x[i] = x[i] + ta * p[i];
            const T nr = r[i] - ta * q[i];
            r[i] = nr;
            rr += (double)nr * (double)nr;
        }
        double v2[1] = {rr}, t2[1];
        coop_exchange<1>(v2, t2, part + 2 * KRY_MAX_GRID, ctr, target, sh, sh_tot);
        const double rho_prev = rho;
        rho = t2[0];
        it += 1;
        const double nrm = sqrt(rho);
        // identical decision in every block (same inputs, same order)
        bool stop = false;
        int sid = 0;
        for (int i = 0; i < c->n_crit && !stop; ++i) {
            if (crit_fires(c, i, it, nrm)) stop = true, sid = i + 1;
        }
        beta = safe_div(rho, rho_prev);
        if (gt == 0) {
            c->it = it;
            c->rho_prev = rho_prev;
            c->rho = rho;
            c->rnorm = nrm;
            c->sigma = sigma;
            c->alpha = alpha;
            c->beta = beta;
            hist_put(c, hist, it, nrm);
            if (stop) {
                c->stopped = 1;
                c->stopping_id = sid;
                c->finalized = 1;
                c->done = 1;
            }
        }
        // no barrier needed here: every thread updates its own rows in every
        // phase, and a partial slot is rewritten only after the next barrier,
        // by which time every block has finished reading it
        done = stop;
        pout = pin;
        pin = p;
    }
    coop_exit(ctr, target);
}

// Register-resident variant (C1): the same arithmetic, row ownership and
// summation order as cg_coop_kernel (rows gt + k*gs, k < RPT, so bitwise the
// same iterates), but everything a thread owns lives in registers for the
// whole solve -- its rows' x, r, p and q, their row bounds, the first W
// column indices and values of each row, and the criteria -- so an iteration
// touches global memory only for the neighbour gathers (p, r of the columns)
// and the stores the neighbours read (p, r). The loop-carried dependency
// chain per iteration drops from four L2 round trips (row bounds -> columns
// -> gathers, then x/p/r/q) plus the control block to one.
template <typename T, int RPT, int W, int BS>
__global__ void __launch_bounds__(BS)
cg_coop_res_kernel(int64_t n, const int* __restrict__ rp, const int* __restrict__ ci, const T* __restrict__ av,
                   T* __restrict__ x, T* r, T* p_a, T* p_b, T* __restrict__ q, KrylovCtl* c, double* part,
                   double* hist, int nofence) {
    unsigned* const ctr = &c->ticket[3];
    unsigned target = 0;
    __shared__ double sh[BS / 32];
    __shared__ double sh_tot[2];
    const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t gs = (int64_t)gridDim.x * blockDim.x;
    T xo[RPT], ro[RPT], po[RPT], qo[RPT];
    int kb[RPT], ke[RPT];
    int cj[RPT][W];
    T cv[RPT][W];
#pragma unroll
    for (int k = 0; k < RPT; ++k) {
        const int64_t i = gt + k * gs;
        kb[k] = ke[k] = 0;
        xo[k] = ro[k] = po[k] = qo[k] = 0;
        if (i < n) {
            kb[k] = rp[i];
            ke[k] = rp[i + 1];
            xo[k] = x[i];
            ro[k] = r[i];
            po[k] = p_a[i];
        }
#pragma unroll
        for (int w = 0; w < W; ++w) {
            cj[k][w] = 0;
            cv[k][w] = 0;
            if (kb[k] + w < ke[k]) {
                cj[k][w] = ci[kb[k] + w];
                cv[k][w] = av[kb[k] + w];
            }
        }
    }
    // criteria are constant during the solve (TimeLimit never takes this path)
    const int n_crit = c->n_crit;
    int ctype[KRY_MAX_CRIT];
    double cparam[KRY_MAX_CRIT];
#pragma unroll
    for (int i = 0; i < KRY_MAX_CRIT; ++i) {
        ctype[i] = i < n_crit ? c->crit_type[i] : 0;
        cparam[i] = i < n_crit ? c->crit_param[i] : 0.0;
    }
    const double baseline = c->baseline;
    const int hist_cap = c->hist_cap;  // thread 0 must not stall on a control-block load
    double rho = c->rho, beta = c->beta;
    int it = c->it;
    bool done = c->done;
    const T* pin = p_a;
    T* pout = p_b;
    uint4* const slots = (uint4*)(part + KRY_NRED * KRY_MAX_GRID);
    if (nofence) coop_slots_clear(slots, ctr, target);
    while (!done) {
        const T tb = (T)beta;
        double sg = 0;
#pragma unroll
        for (int k = 0; k < RPT; ++k) {
            const int64_t i = gt + k * gs;
            if (i < n) {
                T s = 0;
#pragma unroll
                for (int w = 0; w < W; ++w) {
                    if (kb[k] + w < ke[k]) {
                        const int j = cj[k][w];
                        s += cv[k][w] * fma_t(tb, pin[j], r[j]);
                    }
                }
                for (int kk = kb[k] + W; kk < ke[k]; ++kk) {
                    const int j = ci[kk];
                    s += av[kk] * fma_t(tb, pin[j], r[j]);
                }
                qo[k] = s;
                const T pi = fma_t(tb, po[k], ro[k]);
                po[k] = pi;
                pout[i] = pi;
                sg += (double)pi * (double)s;
            }
        }
        double sigma;
        if (nofence) {
            coop_exchange_nofence(sg, sigma, slots, (unsigned)it + 1, ctr, target, sh, sh_tot);
        } else {
            double v1[1] = {sg}, t1[1];
            coop_exchange<1>(v1, t1, part, ctr, target, sh, sh_tot);
            sigma = t1[0];
        }
        if (sigma <= 0.0 && rho != 0.0) {  // breakdown (krylov.py:64-70)
            if (gt == 0) {
                c->sigma = sigma;
                c->breakdown = BD_CG_SIGMA;
                c->breakdown_it = it + 1;
                c->done = 1;
            }
            break;
        }
        const double alpha = safe_div(rho, sigma);
        const T ta = (T)alpha;
        double rr = 0;
#pragma unroll
        for (int k = 0; k < RPT; ++k) {
            const int64_t i = gt + k * gs;
            if (i < n) {
                xo[k] = xo[k] + ta * po[k];
                const T nr = ro[k] - ta * qo[k];
                ro[k] = nr;
                r[i] = nr;
                rr += (double)nr * (double)nr;
            }
        }
        double v2[1] = {rr}, t2[1];
        coop_exchange<1>(v2, t2, part + 2 * KRY_MAX_GRID, ctr, target, sh, sh_tot);
        const double rho_prev = rho;
        rho = t2[0];
        it += 1;
        const double nrm = sqrt(rho);
        bool stop = false;
        int sid = 0;
#pragma unroll
        for (int i = 0; i < KRY_MAX_CRIT; ++i) {  // unrolled: the criteria stay in registers
            const bool f = ctype[i] == CRIT_ITERATION ? it >= (int)cparam[i]
                           : ctype[i] == CRIT_RNR     ? nrm <= cparam[i] * baseline
                                                      : false;
            if (!stop && i < n_crit && f) stop = true, sid = i + 1;
        }
        beta = safe_div(rho, rho_prev);
        if (gt == 0) {
            c->it = it;
            c->rho_prev = rho_prev;
            c->rho = rho;
            c->rnorm = nrm;
            c->sigma = sigma;
            c->alpha = alpha;
            c->beta = beta;
            if (hist && it < hist_cap) hist[it] = nrm;
            if (stop) {
                c->stopped = 1;
                c->stopping_id = sid;
                c->finalized = 1;
                c->done = 1;
            }
        }
        done = stop;
        T* const pt = pout;
        pout = (T*)pin;
        pin = pt;
    }
#pragma unroll
    for (int k = 0; k < RPT; ++k) {
        const int64_t i = gt + k * gs;
        if (i < n) {
            x[i] = xo[k];
            q[i] = qo[k];
        }
    }
    coop_exit(ctr, target);
}

// ===========================================================================
// BiCGSTAB (half-iteration counting, mid check on s with finalize)
// ===========================================================================
// cycle start: rho = rt.r; breakdown if rho == 0 with r != 0; beta
__device__ inline void bicg_cycle_start(KrylovCtl* c, double rho_new, double rr) {
    if (c->done) return;
    if (rho_new == 0.0 && rr != 0.0) {  // krylov.py:227-231
        c->breakdown = BD_RHO;
        c->breakdown_it = c->it + 1;
        c->done = 1;
        return;
    }
    c->rho = rho_new;
    c->beta = safe_div(c->rho, c->rho_prev) * safe_div(c->alpha, c->omega);
}

__device__ inline void bicg_gamma_ctl(KrylovCtl* c, const double* tot) {
    c->gamma = tot[0];
    if (c->gamma == 0.0 && c->rho != 0.0) {  // krylov.py:235-239
        c->breakdown = BD_GAMMA;
        c->breakdown_it = c->it + 1;
        c->done = 1;
        return;
    }
    c->alpha = safe_div(c->rho, c->gamma);
}

__device__ inline void bicg_tst_ctl(KrylovCtl* c, const double* tot) {
    c->ts = tot[0];
    c->tt = tot[1];
    if (c->tt == 0.0 && c->ts != 0.0) {  // krylov.py:262-265
        c->breakdown = BD_TT;
        c->breakdown_it = c->it + 1;
        c->done = 1;
        return;
    }
    c->omega = safe_div(c->ts, c->tt);
}

// after r = b - A x: rt = b, zero p v s t y z, baseline, check(0), cycle start
template <typename T>
__global__ void __launch_bounds__(KRY_BLOCK)
bicg_init_kernel(int64_t n, const T* __restrict__ b, int64_t bstr, const T* __restrict__ r, T* __restrict__ rt,
                 T* __restrict__ p, T* __restrict__ v, T* __restrict__ s, T* __restrict__ t, T* __restrict__ y,
                 T* __restrict__ z, KrylovCtl* c, double* part, double* hist) {
    double rr = 0, rtr = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const T bv = b[i * bstr];
        const T rv = r[i];
        rt[i] = bv;
        p[i] = v[i] = s[i] = t[i] = T(0);
        if (y != p) y[i] = T(0);
        if (z != s) z[i] = T(0);
        rr += (double)rv * (double)rv;
        rtr += (double)bv * (double)rv;
    }
    double vv[2] = {rr, rtr}, tot[2];
    if (!grid_reduce<2>(vv, part, &c->ticket[0], tot)) return;
    c->it = 0;
    c->rho_prev = 1.0;
    c->alpha = 1.0;
    c->omega = 1.0;
    c->rho = 0.0;
    c->ts = c->tt = 0.0;
    c->rnorm = sqrt(tot[0]);
    c->baseline = c->rnorm;
    hist_put(c, hist, 0, c->rnorm);
    crit_check(c, 0, c->rnorm);
    c->done = c->stopped;
    bicg_cycle_start(c, tot[1], tot[0]);
}

// p = r + beta (p - omega v); y = M p     (BicgstabStep1, steps.py:348-378)
template <typename T>
__global__ void __launch_bounds__(KRY_BLOCK)
bicg_step1_kernel(RowBlocks rb, const T* __restrict__ r, T* __restrict__ p, const T* __restrict__ v,
                  T* __restrict__ y, const KrylovCtl* c) {
    if (c->done) return;
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const T beta = (T)c->beta, omega = (T)c->omega;
    for (int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < rb.count(); b += nw) {
        int64_t r0;
        int bs;
        rb.range(b, r0, bs);
        T pv = T(0);
        if (lane < bs) {
            const int64_t i = r0 + lane;
            pv = r[i] + beta * (p[i] - omega * v[i]);
            p[i] = pv;
        }
        if (rb.J.nblocks) {
            const T yv = jacobi_row<T>(rb.J, b, bs, lane, pv);
            if (lane < bs) y[r0 + lane] = yv;
        }
    }
}

// gamma = rt.v; breakdown if gamma == 0 and rho != 0; alpha = rho / gamma
template <typename T>
__global__ void __launch_bounds__(KRY_BLOCK)
bicg_gamma_kernel(int64_t n, const T* __restrict__ rt, const T* __restrict__ v, KrylovCtl* c, double* part) {
    if (c->done) return;
    double s = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        s += (double)rt[i] * (double)v[i];
    double vv[1] = {s}, tot[1];
    if (!grid_reduce<1>(vv, part, &c->ticket[1], tot)) return;
    bicg_gamma_ctl(c, tot);
}

// s = r - alpha v; z = M s; it++; mid check on ||s||   (BicgstabStep2)
template <typename T>
__global__ void __launch_bounds__(KRY_BLOCK)
bicg_step2_kernel(RowBlocks rb, const T* __restrict__ r, const T* __restrict__ v, T* __restrict__ s,
                  T* __restrict__ z, KrylovCtl* c, double* part, double* hist) {
    if (c->done) return;
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const T alpha = (T)c->alpha;
    double ss = 0;
    for (int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < rb.count(); b += nw) {
        int64_t r0;
        int bs;
        rb.range(b, r0, bs);
        T sv = T(0);
        if (lane < bs) {
            const int64_t i = r0 + lane;
            sv = r[i] - alpha * v[i];
            s[i] = sv;
        }
        if (rb.J.nblocks) {
            const T zv = jacobi_row<T>(rb.J, b, bs, lane, sv);
            if (lane < bs) z[r0 + lane] = zv;
        }
        ss += (double)sv * (double)sv;
    }
    double vv[1] = {ss}, tot[1];
    if (!grid_reduce<1>(vv, part, &c->ticket[2], tot)) return;
    c->it += 1;
    c->snorm = sqrt(tot[0]);
    hist_put(c, hist, c->it, c->snorm);
    crit_check(c, c->it, c->snorm);
    if (c->stopped) {
        // converged on ||s||: commit the pending half step (krylov.py:248-253)
        c->mid_final = c->needs_residual;
        c->done = 1;
    }
}

// ts = t.s, tt = t.t; breakdown if tt == 0 and ts != 0; omega = ts / tt
template <typename T>
__global__ void __launch_bounds__(KRY_BLOCK)
bicg_tst_kernel(int64_t n, const T* __restrict__ t, const T* __restrict__ s, KrylovCtl* c, double* part) {
    if (c->done) return;
    double a = 0, bb = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double tv = t[i];
        a += tv * (double)s[i];
        bb += tv * tv;
    }
    double vv[2] = {a, bb}, tot[2];
    if (!grid_reduce<2>(vv, part, &c->ticket[1], tot)) return;
    bicg_tst_ctl(c, tot);
}

// x += alpha y + omega z; r = s - omega t; it++; top check; next cycle start
// (BicgstabStep3); or, after a mid-check stop, x += alpha y (BicgstabFinalize)
template <typename T>
__global__ void __launch_bounds__(KRY_BLOCK)
bicg_step3_kernel(int64_t n, T* __restrict__ x, int64_t xs, T* __restrict__ r, const T* __restrict__ s,
                  const T* __restrict__ t, const T* __restrict__ y, const T* __restrict__ z,
                  const T* __restrict__ rt, KrylovCtl* c, double* part, double* hist) {
    const int mid = c->mid_final;
    if (c->done && !mid) return;
    const T alpha = (T)c->alpha, omega = (T)c->omega;
    double rr = 0, rtr = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (mid) {
            x[i * xs] = x[i * xs] + alpha * y[i];
            continue;
        }
        const T upd = alpha * y[i] + omega * z[i];
        x[i * xs] = x[i * xs] + upd;
        const T rv = s[i] - omega * t[i];
        r[i] = rv;
        rr += (double)rv * (double)rv;
        rtr += (double)rt[i] * (double)rv;
    }
    double vv[2] = {rr, rtr}, tot[2];
    if (!grid_reduce<2>(vv, part, &c->ticket[2], tot)) return;
    if (mid) {
        c->mid_final = 0;
        return;
    }
    c->rho_prev = c->rho;
    c->it += 1;
    c->rnorm = sqrt(tot[0]);
    hist_put(c, hist, c->it, c->rnorm);
    crit_check(c, c->it, c->rnorm);
    c->done = c->stopped;
    bicg_cycle_start(c, tot[1], tot[0]);
}

// Persistent cooperative FCG for small unpreconditioned Csr systems (z = r):
// CgStep1, SpMV + sigma (cg_sigma_ctl), FcgStep2 (t = r_new - r_old, rho =
// r.z, rho_t = t.z, ||r||, check, beta = rho_t / rho_prev) in one launch,
// with the block-local control copies of the cooperative BiCGSTAB below.
// ---------------------------------------------------------------------------
// Tiny systems (n <= 4 rows, the paper's 1x1 overhead benchmark): the whole
// CG / BiCGSTAB solve in ONE thread with the matrix and every vector in
// registers (the row count a template constant) and the control block in a
// local copy -- the cooperative kernels' statements one for one (same
// products, same fused multiply-adds, dots accumulated in fp64 in row order),
// without a single memory round trip per iteration. The vectors and the
// control block are written back at the end.
// ---------------------------------------------------------------------------
constexpr int TINY_ROWS = 4;

template <typename T, int N>
struct TinyCsr {
    int rp[N + 1];
    int ci[N * N];
    T av[N * N];
    __device__ void load(const int* rpg, const int* cig, const T* avg) {
#pragma unroll
        for (int i = 0; i <= N; ++i) rp[i] = rpg[i];
        for (int k = 0; k < rp[N]; ++k) {
            ci[k] = cig[k];
            av[k] = avg[k];
        }
    }
    // out_i = sum_k av[k] * u[ci[k]], left to right (coop_row_dot)
    __device__ void apply(const T (&u)[N], T (&out)[N]) const {
#pragma unroll
        for (int i = 0; i < N; ++i) {
            T acc = 0;
            for (int k = rp[i]; k < rp[i + 1]; ++k) {
                T uk = u[0];
#pragma unroll
                for (int j = 1; j < N; ++j)
                    if (ci[k] == j) uk = u[j];
                acc += av[k] * uk;
            }
            out[i] = acc;
        }
    }
};

template <typename T, int N>
__global__ void __launch_bounds__(32)
cg_tiny_kernel(const int* __restrict__ rp, const int* __restrict__ ci, const T* __restrict__ avg, T* x_g, T* r_g,
               T* p_g, KrylovCtl* c, double* hist) {
    if (threadIdx.x != 0) return;
    TinyCsr<T, N> A;
    A.load(rp, ci, avg);
    KrylovCtl s = *c;
    T x[N], r[N], pin[N], pout[N], q[N];
#pragma unroll
    for (int i = 0; i < N; ++i) x[i] = x_g[i], r[i] = r_g[i], pin[i] = p_g[i];
    double rho = s.rho, beta = s.beta;
    int it = s.it;
    bool done = s.done;
    while (!done) {
        const T tb = (T)beta;
        T pg[N];
#pragma unroll
        for (int j = 0; j < N; ++j) pg[j] = fma_t(tb, pin[j], r[j]);  // p recomputed as in the SpMV of cg_coop
        A.apply(pg, q);
        double sg = 0;
#pragma unroll
        for (int i = 0; i < N; ++i) {
            pout[i] = pg[i];
            sg += (double)pg[i] * (double)q[i];
        }
        const double sigma = sg;
        if (sigma <= 0.0 && rho != 0.0) {  // breakdown (krylov.py:64-70)
            s.sigma = sigma;
            s.breakdown = BD_CG_SIGMA;
            s.breakdown_it = it + 1;
            s.done = 1;
            break;
        }
        const double alpha = safe_div(rho, sigma);
        const T ta = (T)alpha;
        double rr = 0;
#pragma unroll
        for (int i = 0; i < N; ++i) {
            x[i] = x[i] + ta * pout[i];
            r[i] = r[i] - ta * q[i];
            rr += (double)r[i] * (double)r[i];
        }
        const double rho_prev = rho;
        rho = rr;
        it += 1;
        const double nrm = sqrt(rho);
        bool stop = false;
        int sid = 0;
        for (int i = 0; i < s.n_crit && !stop; ++i)
            if (crit_fires(&s, i, it, nrm)) stop = true, sid = i + 1;
        beta = safe_div(rho, rho_prev);
        s.it = it;
        s.rho_prev = rho_prev;
        s.rho = rho;
        s.rnorm = nrm;
        s.sigma = sigma;
        s.alpha = alpha;
        s.beta = beta;
        hist_put(&s, hist, it, nrm);
        if (stop) {
            s.stopped = 1;
            s.stopping_id = sid;
            s.finalized = 1;
            s.done = 1;
        }
        done = stop;
#pragma unroll
        for (int i = 0; i < N; ++i) pin[i] = pout[i];
    }
#pragma unroll
    for (int i = 0; i < N; ++i) x_g[i] = x[i], r_g[i] = r[i], p_g[i] = pin[i];
    *c = s;
}

template <typename T, int N>
__global__ void __launch_bounds__(32)
bicg_tiny_kernel(const int* __restrict__ rp, const int* __restrict__ ci, const T* __restrict__ avg, T* x_g, T* r_g,
                 const T* __restrict__ rt_g, T* p_g, T* v_g, T* s_g, T* t_g, KrylovCtl* c, double* hist) {
    if (threadIdx.x != 0) return;
    TinyCsr<T, N> A;
    A.load(rp, ci, avg);
    KrylovCtl sc = *c;
    T x[N], r[N], rt[N], p[N], v[N], sv[N], t[N];
#pragma unroll
    for (int i = 0; i < N; ++i)
        x[i] = x_g[i], r[i] = r_g[i], rt[i] = rt_g[i], p[i] = p_g[i], v[i] = v_g[i], sv[i] = s_g[i], t[i] = t_g[i];
    while (!sc.done) {
        {   // p = r + beta (p - omega v)   (BicgstabStep1)
            const T beta = (T)sc.beta, omega = (T)sc.omega;
#pragma unroll
            for (int i = 0; i < N; ++i) p[i] = r[i] + beta * (p[i] - omega * v[i]);
        }
        A.apply(p, v);  // v = A p; gamma = rt.v
        double g = 0;
#pragma unroll
        for (int i = 0; i < N; ++i) g += (double)rt[i] * (double)v[i];
        {
            const double tot[1] = {g};
            bicg_gamma_ctl(&sc, tot);
        }
        if (sc.done) break;
        const T alpha = (T)sc.alpha;
        double ss = 0;
#pragma unroll
        for (int i = 0; i < N; ++i) {  // s = r - alpha v   (BicgstabStep2)
            sv[i] = r[i] - alpha * v[i];
            ss += (double)sv[i] * (double)sv[i];
        }
        sc.it += 1;
        sc.snorm = sqrt(ss);
        hist_put(&sc, hist, sc.it, sc.snorm);
        crit_check(&sc, sc.it, sc.snorm);
        if (sc.stopped) {  // converged on ||s||: x += alpha y   (BicgstabFinalize)
            if (sc.needs_residual) {
#pragma unroll
                for (int i = 0; i < N; ++i) x[i] = x[i] + alpha * p[i];
            }
            sc.done = 1;
            break;
        }
        A.apply(sv, t);  // t = A s; ts = t.s, tt = t.t
        double a = 0, bb = 0;
#pragma unroll
        for (int i = 0; i < N; ++i) {
            const double tv = t[i];
            a += tv * (double)sv[i];
            bb += tv * tv;
        }
        {
            const double tot[2] = {a, bb};
            bicg_tst_ctl(&sc, tot);
        }
        if (sc.done) break;
        const T omega = (T)sc.omega;
        double rr = 0, rtr = 0;
#pragma unroll
        for (int i = 0; i < N; ++i) {  // x += alpha y + omega z; r = s - omega t   (BicgstabStep3)
            const T upd = alpha * p[i] + omega * sv[i];
            x[i] = x[i] + upd;
            r[i] = sv[i] - omega * t[i];
            rr += (double)r[i] * (double)r[i];
            rtr += (double)rt[i] * (double)r[i];
        }
        sc.rho_prev = sc.rho;
        sc.it += 1;
        sc.rnorm = sqrt(rr);
        hist_put(&sc, hist, sc.it, sc.rnorm);
        crit_check(&sc, sc.it, sc.rnorm);
        sc.done = sc.stopped;
        bicg_cycle_start(&sc, rtr, rr);
    }
    sc.mid_final = 0;
#pragma unroll
    for (int i = 0; i < N; ++i) x_g[i] = x[i], r_g[i] = r[i], p_g[i] = p[i], v_g[i] = v[i], s_g[i] = sv[i], t_g[i] = t[i];
    *c = sc;
}

template <typename T>
__global__ void __launch_bounds__(KRY_BLOCK)
fcg_coop_kernel(int64_t n, const int* __restrict__ rp, const int* __restrict__ ci, const T* __restrict__ av,
                T* __restrict__ x, T* r, T* p, T* q, T* t, KrylovCtl* c, double* part, double* hist);

// Persistent cooperative BiCGSTAB for small unpreconditioned Csr systems:
// the whole solve in one launch (y = p, z = s). Every block keeps a copy of
// the control block in shared memory and runs the same control functions on
// the same all-reduced totals (bicg_gamma_ctl, bicg_tst_ctl, the mid and top
// checks, bicg_cycle_start), so every block takes the same decisions; block
// 0 writes the state back. Vector updates are the step kernels' expressions
// (steps.py:348-480); the reductions alternate between two partial-sum
// regions so a region is rewritten only after every block has read it.
template <typename T>
__device__ __forceinline__ void coop_row_dot(int64_t i, const int* __restrict__ rp, const int* __restrict__ ci,
                                             const T* __restrict__ av, const T* u, T& out) {
    T acc = 0;
    for (int k = rp[i]; k < rp[i + 1]; ++k) acc += av[k] * u[ci[k]];
    out = acc;
}

template <typename T>
__global__ void __launch_bounds__(KRY_BLOCK)
bicg_coop_kernel(int64_t n, const int* __restrict__ rp, const int* __restrict__ ci, const T* __restrict__ av,
                 T* __restrict__ x, T* r, const T* __restrict__ rt, T* p, T* v, T* s, T* t, KrylovCtl* c,
                 double* part, double* hist) {
    unsigned* const ctr = &c->ticket[3];
    unsigned target = 0;
    __shared__ KrylovCtl sc;
    __shared__ double sh[KRY_BLOCK / 32];
    __shared__ double sh_tot[2];
    const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t gs = (int64_t)gridDim.x * blockDim.x;
    double* const hb = blockIdx.x == 0 ? hist : nullptr;
    double* const part0 = part;
    double* const part1 = part + 2 * KRY_MAX_GRID;
    if (threadIdx.x == 0) sc = *c;
    __syncthreads();
    while (!sc.done) {
        {   // p = r + beta (p - omega v)   (BicgstabStep1)
            const T beta = (T)sc.beta, omega = (T)sc.omega;
            for (int64_t i = gt; i < n; i += gs) p[i] = r[i] + beta * (p[i] - omega * v[i]);
        }
        coop_barrier(ctr, target);
        {   // v = A p; gamma = rt.v
            double g = 0;
            for (int64_t i = gt; i < n; i += gs) {
                T vi;
                coop_row_dot(i, rp, ci, av, p, vi);
                v[i] = vi;
                g += (double)rt[i] * (double)vi;
            }
            double vv[1] = {g}, tot[1];
            coop_exchange<1>(vv, tot, part0, ctr, target, sh, sh_tot);
            if (threadIdx.x == 0) bicg_gamma_ctl(&sc, tot);
            __syncthreads();
            if (sc.done) break;
        }
        {   // s = r - alpha v; it++; mid check on ||s||   (BicgstabStep2)
            const T alpha = (T)sc.alpha;
            double ss = 0;
            for (int64_t i = gt; i < n; i += gs) {
                const T sv = r[i] - alpha * v[i];
                s[i] = sv;
                ss += (double)sv * (double)sv;
            }
            double vv[1] = {ss}, tot[1];
            coop_exchange<1>(vv, tot, part1, ctr, target, sh, sh_tot);
            if (threadIdx.x == 0) {
                sc.it += 1;
                sc.snorm = sqrt(tot[0]);
                hist_put(&sc, hb, sc.it, sc.snorm);
                crit_check(&sc, sc.it, sc.snorm);
                if (sc.stopped) {
                    sc.mid_final = sc.needs_residual;
                    sc.done = 1;
                }
            }
            __syncthreads();
            if (sc.done) {  // converged on ||s||: x += alpha y   (BicgstabFinalize)
                if (sc.mid_final)
                    for (int64_t i = gt; i < n; i += gs) x[i] = x[i] + alpha * p[i];
                __syncthreads();
                if (threadIdx.x == 0) sc.mid_final = 0;
                break;
            }
        }
        {   // t = A s; ts = t.s, tt = t.t
            double a = 0, bb = 0;
            for (int64_t i = gt; i < n; i += gs) {
                T ti;
                coop_row_dot(i, rp, ci, av, s, ti);
                t[i] = ti;
                const double tv = ti;
                a += tv * (double)s[i];
                bb += tv * tv;
            }
            double vv[2] = {a, bb}, tot[2];
            coop_exchange<2>(vv, tot, part0, ctr, target, sh, sh_tot);
            if (threadIdx.x == 0) bicg_tst_ctl(&sc, tot);
            __syncthreads();
            if (sc.done) break;
        }
        {   // x += alpha y + omega z; r = s - omega t; it++; check; next rho   (BicgstabStep3)
            const T alpha = (T)sc.alpha, omega = (T)sc.omega;
            double rr = 0, rtr = 0;
            for (int64_t i = gt; i < n; i += gs) {
                const T upd = alpha * p[i] + omega * s[i];
                x[i] = x[i] + upd;
                const T rv = s[i] - omega * t[i];
                r[i] = rv;
                rr += (double)rv * (double)rv;
                rtr += (double)rt[i] * (double)rv;
            }
            double vv[2] = {rr, rtr}, tot[2];
            coop_exchange<2>(vv, tot, part1, ctr, target, sh, sh_tot);
            if (threadIdx.x == 0) {
                sc.rho_prev = sc.rho;
                sc.it += 1;
                sc.rnorm = sqrt(tot[0]);
                hist_put(&sc, hb, sc.it, sc.rnorm);
                crit_check(&sc, sc.it, sc.rnorm);
                sc.done = sc.stopped;
                bicg_cycle_start(&sc, tot[1], tot[0]);
            }
            __syncthreads();
        }
    }
    coop_exit(ctr, target, c, &sc);
}

template <typename T>
__global__ void __launch_bounds__(KRY_BLOCK)
fcg_coop_kernel(int64_t n, const int* __restrict__ rp, const int* __restrict__ ci, const T* __restrict__ av,
                T* __restrict__ x, T* r, T* p, T* q, T* t, KrylovCtl* c, double* part, double* hist) {
    unsigned* const ctr = &c->ticket[3];
    unsigned target = 0;
    __shared__ KrylovCtl sc;
    __shared__ double sh[KRY_BLOCK / 32];
    __shared__ double sh_tot[4];
    const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t gs = (int64_t)gridDim.x * blockDim.x;
    double* const hb = blockIdx.x == 0 ? hist : nullptr;
    double* const part_s = part;                 // sigma: 1 value per block
    double* const part_2 = part + KRY_MAX_GRID;  // step 2: 3 values per block
    if (threadIdx.x == 0) sc = *c;
    __syncthreads();
    while (!sc.done) {
        {   // p = z + beta p   (CgStep1, z = r)
            const T beta = (T)sc.beta;
            for (int64_t i = gt; i < n; i += gs) p[i] = r[i] + beta * p[i];
        }
        coop_barrier(ctr, target);
        {   // q = A p; sigma = p.q
            double sg = 0;
            for (int64_t i = gt; i < n; i += gs) {
                T qi;
                coop_row_dot(i, rp, ci, av, p, qi);
                q[i] = qi;
                sg += (double)p[i] * (double)qi;
            }
            double vv[1] = {sg}, tot[1];
            coop_exchange<1>(vv, tot, part_s, ctr, target, sh, sh_tot);
            if (threadIdx.x == 0) cg_sigma_ctl(&sc, tot);
            __syncthreads();
            if (sc.done) break;
        }
        {   // FcgStep2
            const T alpha = (T)sc.alpha;
            double rz = 0, tz = 0, rr = 0;
            for (int64_t i = gt; i < n; i += gs) {
                x[i] = x[i] + mul_rn(alpha, p[i]);
                const T ro = r[i];
                const T rv = ro - mul_rn(alpha, q[i]);
                const T tv = rv - ro;
                t[i] = tv;
                r[i] = rv;
                rz += (double)rv * (double)rv;
                tz += (double)tv * (double)rv;
                rr += (double)rv * (double)rv;
            }
            double vv[3] = {rz, tz, rr}, tot[3];
            coop_exchange<3>(vv, tot, part_2, ctr, target, sh, sh_tot);
            if (threadIdx.x == 0) {
                sc.rho_prev = sc.rho;
                sc.rho = tot[0];
                sc.rho_t = tot[1];
                sc.it += 1;
                sc.rnorm = sqrt(tot[2]);
                hist_put(&sc, hb, sc.it, sc.rnorm);
                crit_check(&sc, sc.it, sc.rnorm);
                sc.done = sc.stopped;
                sc.beta = safe_div(sc.rho_t, sc.rho_prev);
            }
            __syncthreads();
        }
    }
    coop_exit(ctr, target, c, &sc);
}

// ===========================================================================
// CGS (src/solvers/krylov.py:128-187; steps.py:246-345). Initialisation is
// BiCGSTAB's (rt = b, workspace zeroed, rho = rt.r, beta = rho / 1); the
// first SpMV carries gamma = rt.v_hat (BiCGSTAB's gamma control: breakdown,
// alpha = rho / gamma); the mid check sees the unchanged ||r||; step 3 ends
// in the top-of-loop check followed by the next rho = rt.r.
// ===========================================================================
__device__ inline void cgs_cycle_start(KrylovCtl* c, double rho_new, double rr) {
    if (c->done) return;
    if (rho_new == 0.0 && rr != 0.0) {  // krylov.py:155-158
        c->breakdown = BD_RHO;
        c->breakdown_it = c->it + 1;
        c->done = 1;
        return;
    }
    c->rho = rho_new;
    c->beta = safe_div(c->rho, c->rho_prev);
}

// u = r + beta q; p = u + beta (q + beta p); ph = M p      (CgsStep1)
template <typename T>
__global__ void __launch_bounds__(KRY_BLOCK)
cgs_step1_kernel(RowBlocks rb, const T* __restrict__ r, const T* __restrict__ q, T* __restrict__ u, T* __restrict__ p,
                 T* __restrict__ ph, const KrylovCtl* c) {
    if (c->done) return;
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const T beta = (T)c->beta;
    for (int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < rb.count(); b += nw) {
        int64_t r0;
        int bs;
        rb.range(b, r0, bs);
        T pv = T(0);
        if (lane < bs) {
            const int64_t i = r0 + lane;
            const T qv = q[i];
            const T uv = r[i] + mul_rn(beta, qv);
            u[i] = uv;
            pv = uv + mul_rn(beta, qv + mul_rn(beta, p[i]));
            p[i] = pv;
        }
        if (rb.J.nblocks) {
            const T yv = jacobi_row<T>(rb.J, b, bs, lane, pv);
            if (lane < bs) ph[r0 + lane] = yv;
        }
    }
}

// q = u - alpha v_hat; w = u + q; uh = M w      (CgsStep2)
template <typename T>
__global__ void __launch_bounds__(KRY_BLOCK)
cgs_step2_kernel(RowBlocks rb, const T* __restrict__ u, const T* __restrict__ vh, T* __restrict__ q, T* __restrict__ w,
                 T* __restrict__ uh, const KrylovCtl* c) {
    if (c->done) return;
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const T alpha = (T)c->alpha;
    for (int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < rb.count(); b += nw) {
        int64_t r0;
        int bs;
        rb.range(b, r0, bs);
        T wv = T(0);
        if (lane < bs) {
            const int64_t i = r0 + lane;
            const T uv = u[i];
            const T qv = uv - mul_rn(alpha, vh[i]);
            q[i] = qv;
            wv = uv + qv;
            w[i] = wv;
        }
        if (rb.J.nblocks) {
            const T yv = jacobi_row<T>(rb.J, b, bs, lane, wv);
            if (lane < bs) uh[r0 + lane] = yv;
        }
    }
}

// mid check: it++, criteria on the unchanged ||r|| (krylov.py:171-176)
__global__ void cgs_mid_kernel(KrylovCtl* c, double* hist) {
    if (threadIdx.x != 0 || blockIdx.x != 0 || c->done) return;
    c->it += 1;
    hist_put(c, hist, c->it, c->rnorm);
    crit_check(c, c->it, c->rnorm);
    c->done = c->stopped;
}

// r -= alpha t; x += alpha uh; it++; top check; next rho = rt.r  (CgsStep3)
template <typename T>
__global__ void __launch_bounds__(KRY_BLOCK)
cgs_step3_kernel(int64_t n, T* __restrict__ x, int64_t xs, T* __restrict__ r, const T* __restrict__ t,
                 const T* __restrict__ uh, const T* __restrict__ rt, KrylovCtl* c, double* part, double* hist) {
    if (c->done) return;
    const T alpha = (T)c->alpha;
    double rr = 0, rtr = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const T rv = r[i] - mul_rn(alpha, t[i]);
        r[i] = rv;
        x[i * xs] = x[i * xs] + mul_rn(alpha, uh[i]);
        rr += (double)rv * (double)rv;
        rtr += (double)rt[i] * (double)rv;
    }
    double vv[2] = {rr, rtr}, tot[2];
    if (!grid_reduce<2>(vv, part, &c->ticket[2], tot)) return;
    c->rho_prev = c->rho;
    c->it += 1;
    c->rnorm = sqrt(tot[0]);
    hist_put(c, hist, c->it, c->rnorm);
    crit_check(c, c->it, c->rnorm);
    c->done = c->stopped;
    cgs_cycle_start(c, tot[1], tot[0]);
}

// Persistent cooperative CGS for small unpreconditioned Csr systems (ph = p,
// uh = w): CgsStep1, SpMV + gamma, CgsStep2, the mid check, SpMV,
// CgsStep3 and the next rho in one launch (block-local control copies as
// in the cooperative BiCGSTAB); four grid barriers per cycle.
template <typename T>
__global__ void __launch_bounds__(KRY_BLOCK)
cgs_coop_kernel(int64_t n, const int* __restrict__ rp, const int* __restrict__ ci, const T* __restrict__ av,
                T* __restrict__ x, T* r, const T* __restrict__ rt, T* p, T* q, T* u, T* vh, T* w, T* t, KrylovCtl* c,
                double* part, double* hist) {
    unsigned* const ctr = &c->ticket[3];
    unsigned target = 0;
    __shared__ KrylovCtl sc;
    __shared__ double sh[KRY_BLOCK / 32];
    __shared__ double sh_tot[2];
    const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t gs = (int64_t)gridDim.x * blockDim.x;
    double* const hb = blockIdx.x == 0 ? hist : nullptr;
    double* const part0 = part;
    double* const part1 = part + 2 * KRY_MAX_GRID;
    if (threadIdx.x == 0) sc = *c;
    __syncthreads();
    while (!sc.done) {
        {   // u = r + beta q; p = u + beta (q + beta p)   (CgsStep1)
            const T beta = (T)sc.beta;
            for (int64_t i = gt; i < n; i += gs) {
                const T qv = q[i];
                const T uv = r[i] + mul_rn(beta, qv);
                u[i] = uv;
                p[i] = uv + mul_rn(beta, qv + mul_rn(beta, p[i]));
            }
        }
        coop_barrier(ctr, target);
        {   // v_hat = A p; gamma = rt.v_hat
            double g = 0;
            for (int64_t i = gt; i < n; i += gs) {
                T vi;
                coop_row_dot(i, rp, ci, av, p, vi);
                vh[i] = vi;
                g += (double)rt[i] * (double)vi;
            }
            double vv[1] = {g}, tot[1];
            coop_exchange<1>(vv, tot, part0, ctr, target, sh, sh_tot);
            if (threadIdx.x == 0) bicg_gamma_ctl(&sc, tot);
            __syncthreads();
            if (sc.done) break;
        }
        const T alpha = (T)sc.alpha;
        // q = u - alpha v_hat; w = u + q   (CgsStep2)
        for (int64_t i = gt; i < n; i += gs) {
            const T uv = u[i];
            const T qv = uv - mul_rn(alpha, vh[i]);
            q[i] = qv;
            w[i] = uv + qv;
        }
        // every thread has read sc (done, alpha) before thread 0 updates it:
        // compute-sanitizer racecheck flagged the unguarded update (round 2)
        __syncthreads();
        if (threadIdx.x == 0) {  // mid check on the unchanged ||r|| (krylov.py:171-176)
            sc.it += 1;
            hist_put(&sc, hb, sc.it, sc.rnorm);
            crit_check(&sc, sc.it, sc.rnorm);
            sc.done = sc.stopped;
        }
        __syncthreads();
        if (sc.done) break;
        coop_barrier(ctr, target);
        {   // t = A w; r -= alpha t; x += alpha w; it++; check; next rho   (CgsStep3)
            double rr = 0, rtr = 0;
            for (int64_t i = gt; i < n; i += gs) {
                T ti;
                coop_row_dot(i, rp, ci, av, w, ti);
                t[i] = ti;
                const T rv = r[i] - mul_rn(alpha, ti);
                r[i] = rv;
                x[i] = x[i] + mul_rn(alpha, w[i]);
                rr += (double)rv * (double)rv;
                rtr += (double)rt[i] * (double)rv;
            }
            double vv[2] = {rr, rtr}, tot[2];
            coop_exchange<2>(vv, tot, part1, ctr, target, sh, sh_tot);
            if (threadIdx.x == 0) {
                sc.rho_prev = sc.rho;
                sc.it += 1;
                sc.rnorm = sqrt(tot[0]);
                hist_put(&sc, hb, sc.it, sc.rnorm);
                crit_check(&sc, sc.it, sc.rnorm);
                sc.done = sc.stopped;
                cgs_cycle_start(&sc, tot[1], tot[0]);
            }
            __syncthreads();
        }
    }
    coop_exit(ctr, target, c, &sc);
}

// ===========================================================================
// GMRES(k), right preconditioned, m = 1.
// gm layout: H[(k+1) x k] row-major | cs[k] | sn[k] | gamma[k+1] | y[k]
// ===========================================================================
struct GmresView {
    double* H;
    double* cs;
    double* sn;
    double* g;
    double* y;
    int k;
    __device__ GmresView(double* gm, int kk) : k(kk) {
        H = gm;
        cs = H + (size_t)(kk + 1) * kk;
        sn = cs + kk;
        g = sn + kk;
        y = g + kk + 1;
    }
};

// reset_segment (gmres.py:75-86) after r = b - A x; `first` also sets the RNR
// baseline and runs the top-of-loop check
template <typename T>
__global__ void __launch_bounds__(KRY_BLOCK)
gmres_reset_kernel(int64_t n, const T* __restrict__ r, KrylovCtl* c, double* part, double* gm, double* hist,
                   int first) {
    if (!first && (c->stopped || c->done)) return;
    double s = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        s += (double)r[i] * (double)r[i];
    double vv[1] = {s}, tot[1];
    if (!grid_reduce<1>(vv, part, &c->ticket[0], tot)) return;
    GmresView G(gm, c->kdim);
    const double beta = sqrt(tot[0]);
    for (int i = 0; i <= G.k; ++i) G.g[i] = 0.0;
    for (int i = 0; i < G.k; ++i) G.cs[i] = G.sn[i] = 0.0;
    G.g[0] = beta;
    c->rnorm = beta;  // res_est
    c->jpos = 0;
    c->committed = 0;
    if (first) {
        c->it = 0;
        c->baseline = beta;
        if (beta == 0.0) {  // exact zero residual: declared converged (gmres.py:210-212)
            c->stopped = 1;
            c->stopping_id = EXACT_CONVERGENCE_ID;
            c->finalized = 1;
            c->rnorm = 0.0;
            c->done = 1;
            return;
        }
    }
    hist_put(c, hist, c->it, c->rnorm);
    crit_check(c, c->it, c->rnorm);
}

// v0 = r / beta (0 if beta == 0)
template <typename T>
__global__ void gmres_scale_v0_kernel(int64_t n, const T* __restrict__ r, T* __restrict__ V, const KrylovCtl* c) {
    if (c->stopped || c->done) return;
    const double beta = c->rnorm;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        V[i] = beta == 0.0 ? T(0) : (T)((double)r[i] / beta);
}

// h_{0,j-1} = v_0 . w
template <typename T>
__global__ void __launch_bounds__(KRY_BLOCK)
gmres_dot0_kernel(int64_t n, int j, const T* __restrict__ V, const T* __restrict__ w, KrylovCtl* c, double* part,
                  double* gm) {
    if (c->stopped || c->done) return;
    double s = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        s += (double)V[i] * (double)w[i];
    double vv[1] = {s}, tot[1];
    if (!grid_reduce<1>(vv, part, &c->ticket[1], tot)) return;
    GmresView G(gm, c->kdim);
    G.H[0 * G.k + (j - 1)] = tot[0];
}

// end of Arnoldi step j: h_{j+1,j} = ||w|| (ww = w.w), the Givens update of
// column j-1, the new residual estimate and the check (gmres.py:88-129)
__device__ inline void gmres_givens_ctl(KrylovCtl* c, GmresView& G, int j, double ww, double* hist) {
    const int col = j - 1;
    const double hj = sqrt(ww);
    c->hnorm = hj;
    G.H[j * G.k + col] = hj;
    for (int q = 0; q < j - 1; ++q) {
        const double h1 = G.H[q * G.k + col], h2 = G.H[(q + 1) * G.k + col];
        G.H[q * G.k + col] = G.cs[q] * h1 + G.sn[q] * h2;
        G.H[(q + 1) * G.k + col] = -G.sn[q] * h1 + G.cs[q] * h2;
    }
    const double h1 = G.H[col * G.k + col], h2 = G.H[j * G.k + col];
    const double den = hypot(h1, h2);
    const double cc = den != 0.0 ? h1 / den : 1.0, sn = den != 0.0 ? h2 / den : 0.0;
    G.cs[col] = cc;
    G.sn[col] = sn;
    G.H[col * G.k + col] = den;
    G.H[j * G.k + col] = 0.0;
    const double gv = G.g[col];
    G.g[col] = cc * gv;
    G.g[j] = -sn * gv;
    c->rnorm = fabs(G.g[j]);
    c->jpos = j;
    c->it += 1;
    if (hj == 0.0) {  // happy breakdown: declared exact (gmres.py:245-248, :262-268)
        c->stopped = 1;
        c->stopping_id = EXACT_CONVERGENCE_ID;
        c->finalized = 1;
        c->rnorm = 0.0;
        return;
    }
    if (j < G.k) {  // at j == k the restart recomputes the residual before the check
        hist_put(c, hist, c->it, c->rnorm);
        crit_check(c, c->it, c->rnorm);
    }
}

// gmres_givens_ctl on a staged copy: L.H / L.cs / L.sn point at shared memory
// (the new column of H with stride 1, the previous rotations); the new
// rotation and the g updates go straight to the workspace G
__device__ inline void gmres_givens_ctl_col(KrylovCtl* c, GmresView& L, GmresView& G, int j, double ww, double* hist) {
    const int col = j - 1;
    const double hj = sqrt(ww);
    c->hnorm = hj;
    L.H[j * L.k + col] = hj;
    for (int q = 0; q < j - 1; ++q) {
        const double h1 = L.H[q * L.k + col], h2 = L.H[(q + 1) * L.k + col];
        L.H[q * L.k + col] = L.cs[q] * h1 + L.sn[q] * h2;
        L.H[(q + 1) * L.k + col] = -L.sn[q] * h1 + L.cs[q] * h2;
    }
    const double h1 = L.H[col * L.k + col], h2 = L.H[j * L.k + col];
    const double den = hypot(h1, h2);
    const double cc = den != 0.0 ? h1 / den : 1.0, sn = den != 0.0 ? h2 / den : 0.0;
    G.cs[col] = cc;
    G.sn[col] = sn;
    L.H[col * L.k + col] = den;
    L.H[j * L.k + col] = 0.0;
    const double gv = G.g[col];
    G.g[col] = cc * gv;
    G.g[j] = -sn * gv;
    c->rnorm = fabs(G.g[j]);
    c->jpos = j;
    c->it += 1;
    if (hj == 0.0) {  // happy breakdown: declared exact (gmres.py:245-248, :262-268)
        c->stopped = 1;
        c->stopping_id = EXACT_CONVERGENCE_ID;
        c->finalized = 1;
        c->rnorm = 0.0;
        return;
    }
    if (j < G.k) {
        hist_put(c, hist, c->it, c->rnorm);
        crit_check(c, c->it, c->rnorm);
    }
}

// MGS step i of Arnoldi step j: w -= h_i v_i, then h_{i+1} = v_{i+1}.w, or,
// for i = j-1, ||w||, the Givens update and the next check (gmres.py:88-129)
template <typename T>
__global__ void __launch_bounds__(KRY_BLOCK)
gmres_mgs_kernel(int64_t n, int j, int i, const T* __restrict__ V, T* __restrict__ w, KrylovCtl* c, double* part,
                 double* gm, double* hist) {
    if (c->stopped || c->done) return;
    GmresView G(gm, c->kdim);
    const T h = (T)G.H[i * G.k + (j - 1)];
    const T* vi = V + (int64_t)i * n;
    const bool last = (i == j - 1);
    const T* vn = last ? w : V + (int64_t)(i + 1) * n;
    double s = 0;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        const T wv = w[r] - h * vi[r];
        w[r] = wv;
        s += (double)(last ? wv : vn[r]) * (double)wv;
    }
    double vv[1] = {s}, tot[1];
    if (!grid_reduce<1>(vv, part, &c->ticket[2], tot)) return;
    if (!last) {
        G.H[(i + 1) * G.k + (j - 1)] = tot[0];
        return;
    }
    gmres_givens_ctl(c, G, j, tot[0], hist);
}

// Small systems (one block covers every row): the whole MGS of Arnoldi step
// j -- h_0 = v_0.w, then for every i: w -= h_i v_i and the next product, the
// Givens update and check, and v_j = w / h -- in ONE single-block launch
// with block barriers instead of j + 2 grid-wide launches (the reference's
// MGS order, gmres.py:88-129, is kept: every h_i uses the updated w).
constexpr int GMRES_SMALL_RPT = 8;  // rows per thread
constexpr int GMRES_SMALL_ROWS = KRY_BLOCK * GMRES_SMALL_RPT;
constexpr int GMRES_SMALL_MAXK = 256;
constexpr int GMRES_SMEM_BYTES = 32 * 1024;  // on-chip basis for tiny systems  // Givens column staged in shared memory up to this restart length

template <typename T, int NT>
__device__ void gmres_arnoldi_small_body(int64_t n, int j, T* __restrict__ V, T* __restrict__ w, KrylovCtl* c,
                                         double* gm, double* hist) {
    constexpr int R = GMRES_SMALL_RPT;
    __shared__ double sh[NT / 32 > 0 ? NT / 32 : 1];
    __shared__ double bc;
    if (((volatile KrylovCtl*)c)->stopped || ((volatile KrylovCtl*)c)->done) return;
    GmresView G(gm, c->kdim);
    auto reduce = [&](double v) {  // block sum broadcast to every thread
        if (NT == 32) return warp_sum(v);  // one warp: no barriers at all
        const double t = block_sum(v, sh);
        if (threadIdx.x == 0) bc = t;
        __syncthreads();
        const double r = bc;
        __syncthreads();
        return r;
    };
    auto load = [&](const T* src, T (&dst)[R]) {
#pragma unroll
        for (int q = 0; q < R; ++q) {
            const int64_t r = threadIdx.x + (int64_t)q * NT;
            dst[q] = r < n ? src[r] : T(0);
        }
    };
    // w and the basis rows live in registers; the next basis row is loaded
    // one pass ahead so its latency overlaps the current pass's reduction
    T wr[R], vi[R], vn[R];
    load(w, wr);
    load(V, vi);
    if (j > 1) load(V + n, vn);
    double s = 0;
#pragma unroll
    for (int q = 0; q < R; ++q) s += (double)vi[q] * (double)wr[q];
    double h = reduce(s);
    if (threadIdx.x == 0) G.H[0 * G.k + (j - 1)] = h;
    for (int i = 0; i < j; ++i) {
        const T th = (T)h;
        const bool last = (i == j - 1);
        T vnn[R];
        if (i + 2 < j) load(V + (int64_t)(i + 2) * n, vnn);
        s = 0;
#pragma unroll
        for (int q = 0; q < R; ++q) {
            const T wv = wr[q] - th * vi[q];
            wr[q] = wv;
            s += (double)(last ? wv : vn[q]) * (double)wv;
        }
        h = reduce(s);
        if (!last) {
            if (threadIdx.x == 0) G.H[(i + 1) * G.k + (j - 1)] = h;
#pragma unroll
            for (int q = 0; q < R; ++q) {
                vi[q] = vn[q];
                vn[q] = vnn[q];
            }
        } else if (j <= GMRES_SMALL_MAXK) {
            // the Givens sweep over the new column runs out of shared memory:
            // stage the column and the rotations (parallel loads), rotate in
            // one thread, write back (a global-memory sweep is a chain of
            // dependent L2 round trips, ~0.5 us per rotation)
            __shared__ double colb[GMRES_SMALL_MAXK + 1], csb[GMRES_SMALL_MAXK], snb[GMRES_SMALL_MAXK];
            const int col = j - 1;
            __syncthreads();
            for (int q = threadIdx.x; q < j; q += NT) colb[q] = G.H[q * G.k + col];
            for (int q = threadIdx.x; q < j - 1; q += NT) {
                csb[q] = G.cs[q];
                snb[q] = G.sn[q];
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                GmresView L = G;
                L.H = colb - col;  // column view: L.H[q * L.k + col] = colb[q] with L.k = 1
                L.k = 1;
                L.cs = csb;
                L.sn = snb;
                gmres_givens_ctl_col(c, L, G, j, h, hist);
            }
            __syncthreads();
            for (int q = threadIdx.x; q <= j; q += NT) G.H[q * G.k + col] = colb[q];
        } else if (threadIdx.x == 0) {
            gmres_givens_ctl(c, G, j, h, hist);
        }
    }
#pragma unroll
    for (int q = 0; q < R; ++q) {
        const int64_t r = threadIdx.x + (int64_t)q * NT;
        if (r < n) w[r] = wr[q];
    }
    __syncthreads();
    // v_j = w / h_{j,j-1}   (gmres_normalize)
    if (((volatile KrylovCtl*)c)->done) return;
    if (((volatile KrylovCtl*)c)->stopped && ((volatile KrylovCtl*)c)->jpos != j) return;
    const double hj = ((volatile KrylovCtl*)c)->hnorm;
    T* vj = V + (int64_t)j * n;
#pragma unroll
    for (int q = 0; q < R; ++q) {
        const int64_t r = threadIdx.x + (int64_t)q * NT;
        if (r < n) vj[r] = hj == 0.0 ? T(0) : (T)((double)wr[q] / hj);
    }
}

template <typename T>
__global__ void __launch_bounds__(KRY_BLOCK)
gmres_arnoldi_small_kernel(int64_t n, int j, T* __restrict__ V, T* __restrict__ w, KrylovCtl* c, double* gm,
                           double* hist) {
    gmres_arnoldi_small_body<T, KRY_BLOCK>(n, j, V, w, c, gm, hist);
}

// A whole Arnoldi cycle of an unpreconditioned small system in one
// single-block launch: for j = 1..k (until a check stops it) w = A v_{j-1}
// (rows summed left to right), then the single-block Arnoldi step above.
template <typename T, int NT>
__global__ void __launch_bounds__(NT)
gmres_cycle_small_kernel(int64_t n, const int* __restrict__ rp, const int* __restrict__ ci, const T* __restrict__ av,
                         T* __restrict__ V, T* __restrict__ w, KrylovCtl* c, double* gm, double* hist);

// v_j = w / h_{j,j-1} (0 on happy breakdown)
template <typename T>
__global__ void gmres_normalize_kernel(int64_t n, int j, T* __restrict__ V, const T* __restrict__ w, const KrylovCtl* c) {
    if (c->done) return;
    if (c->stopped && c->jpos != j) return;
    const double hj = c->hnorm;
    T* vj = V + (int64_t)j * n;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
        vj[r] = hj == 0.0 ? T(0) : (T)((double)w[r] / hj);
}

template <typename T, int NT>
__global__ void __launch_bounds__(NT)
gmres_cycle_small_kernel(int64_t n, const int* __restrict__ rp, const int* __restrict__ ci, const T* __restrict__ av,
                         T* __restrict__ Vg, T* __restrict__ wg, KrylovCtl* c, double* gm, double* hist) {
    // tiny systems (the basis fits in shared memory, `dynamic` bytes): the
    // cycle runs on an on-chip copy of V and w, written back at the end
    extern __shared__ __align__(16) unsigned char gsm[];
    const int k = c->kdim;
    const bool onchip = (size_t)(k + 2) * n * sizeof(T) <= GMRES_SMEM_BYTES;
    T* V = onchip ? reinterpret_cast<T*>(gsm) : Vg;
    T* w = onchip ? V + (size_t)(k + 1) * n : wg;
    if (onchip) {
        for (int64_t r = threadIdx.x; r < n; r += NT) V[r] = Vg[r];  // v_0 from gmres_scale_v0
        __syncthreads();
    }
    int jdone = 0;
    for (int j = 1; j <= k; ++j) {
        if (((volatile KrylovCtl*)c)->stopped || ((volatile KrylovCtl*)c)->done) break;
        const T* src = V + (int64_t)(j - 1) * n;
        for (int64_t r = threadIdx.x; r < n; r += NT) {
            T acc = 0;
            for (int q = rp[r]; q < rp[r + 1]; ++q) acc += av[q] * src[ci[q]];
            w[r] = acc;
        }
        __syncthreads();
        gmres_arnoldi_small_body<T, NT>(n, j, V, w, c, gm, hist);
        __syncthreads();
        jdone = j;
    }
    if (onchip) {  // the basis rows written this cycle (gmres_combine reads them)
        for (int64_t e = n + threadIdx.x; e < (int64_t)(jdone + 1) * n; e += NT) Vg[e] = V[e];
        for (int64_t r = threadIdx.x; r < n; r += NT) wg[r] = w[r];
    }
}

// Tiny systems (n <= GMRES_TINY_ROWS, the paper's 1x1 overhead benchmark):
// a whole Arnoldi cycle AND its back-solve in one launch. Thread 0 runs the
// cycle -- no cross-lane reduction is worth its shuffles when a dot has at
// most four terms (the row count is a template constant: every row loop
// unrolls) -- with the basis, the rotations, gamma and the Hessenberg matrix
// in shared memory and the control block in a local copy; then the warp
// back-solves the rotated triangle column by column from shared memory (row
// i's y_i by its owner lane, broadcast, the other rows' partial sums updated
// in parallel) instead of a separate kernel paying an L2 round trip per row.
// Same arithmetic as the single-block kernel (dots accumulated in fp64 in row
// order; MGS, Givens and the checks of gmres_givens_ctl in the reference's
// order, gmres.py:88-129); the back-solve sums h[i, i+1:jc] @ y in
// descending column order (the reference's NumPy dot order is unspecified).
constexpr int GMRES_TINY_ROWS = 4;
constexpr int GMRES_TINY_MAXK = 128;

__host__ __device__ inline size_t gmres_tiny_smem(int k, int64_t n, size_t tb) {
    return ((size_t)(k + 1) * n * tb + 15) / 16 * 16 + ((size_t)(k + 1) * k + 4 * k + 3) * sizeof(double);
}  // V | cs, sn (k) | g, y (k + 1) | H ((k + 1) x k)

template <typename T, int N>
__global__ void __launch_bounds__(32)
gmres_solve_tiny_kernel(const int* __restrict__ rp, const int* __restrict__ ci, const T* __restrict__ av,
                        T* __restrict__ xg, const T* __restrict__ bg, T* __restrict__ Vg, T* __restrict__ wg,
                        KrylovCtl* c, double* gm, double* hist) {
    extern __shared__ __align__(16) unsigned char gsm[];
    __shared__ int sh_jc, sh_solve, sh_bd;
    constexpr int64_t n = N;  // rows, a compile-time constant: every row loop unrolls
    const int k = c->kdim;
    const int lane = threadIdx.x;
    GmresView G(gm, k);
    T* V = reinterpret_cast<T*>(gsm);
    double* cs = reinterpret_cast<double*>(gsm + ((size_t)(k + 1) * n * sizeof(T) + 15) / 16 * 16);
    double* sn = cs + k;
    double* g = sn + k;
    double* ys = g + k + 1;
    double* H = ys + k + 1;  // (k + 1) x k, row-major like the workspace
    KrylovCtl s;
    T w[N], x[N], bv[N];
    if (lane == 0) {
        s = *c;
#pragma unroll
        for (int64_t r = 0; r < n; ++r) {
            V[r] = Vg[r];  // v_0 from gmres_scale_v0
            x[r] = xg[r];
            bv[r] = bg[r];
        }
        for (int i = 0; i <= k; ++i) g[i] = G.g[i];
    }
    while (true) {
        // ---- one Arnoldi cycle (thread 0) ----
        if (lane == 0) {
            int jdone = 0;
            for (int j = 1; j <= k; ++j) {
                if (s.stopped || s.done) break;
                const T* src = V + (int64_t)(j - 1) * n;
#pragma unroll
                for (int64_t r = 0; r < n; ++r) {
                    T acc = 0;
                    for (int q = rp[r]; q < rp[r + 1]; ++q) acc += av[q] * src[ci[q]];
                    w[r] = acc;
                }
                // modified Gram-Schmidt: h_i from the current w, then w -= h_i v_i
                double* __restrict__ hcol = ys;  // scratch for the new column (ys is free during the cycle)
                // the basis row of step i + 1 is loaded while step i runs (the
                // loads are off the MGS dependency chain)
                T vnext[N];
#pragma unroll
                for (int64_t r = 0; r < n; ++r) vnext[r] = V[r];
                for (int i = 0; i < j; ++i) {
                    T vi[N];
#pragma unroll
                    for (int64_t r = 0; r < n; ++r) vi[r] = vnext[r];
                    if (i + 1 < j) {
#pragma unroll
                        for (int64_t r = 0; r < n; ++r) vnext[r] = V[(int64_t)(i + 1) * n + r];
                    }
                    double h = 0;
#pragma unroll
                    for (int64_t r = 0; r < n; ++r) h += (double)vi[r] * (double)w[r];
                    hcol[i] = h;
                    const T th = (T)h;
#pragma unroll
                    for (int64_t r = 0; r < n; ++r) w[r] = w[r] - th * vi[r];
                }
                double ww = 0;
#pragma unroll
                for (int64_t r = 0; r < n; ++r) ww += (double)w[r] * (double)w[r];
                // Givens update of column j-1 (gmres_givens_ctl): the running
                // entry stays in a register, each finished entry goes to H
                const int cl = j - 1;
                const double hj = sqrt(ww);
                s.hnorm = hj;
                double run = hcol[0];
                double h2n = j > 1 ? hcol[1] : 0.0, csn = cs[0], snn = sn[0];  // prefetched one rotation ahead
                for (int q = 0; q < j - 1; ++q) {
                    const double h2 = h2n, cq = csn, sq = snn;
                    if (q + 2 < j) {
                        h2n = hcol[q + 2];
                        csn = cs[q + 1];
                        snn = sn[q + 1];
                    }
                    H[q * k + cl] = cq * run + sq * h2;
                    run = -sq * run + cq * h2;
                }
                const double h1 = run, h2 = hj;
                const double den = hypot(h1, h2);
                const double cc = den != 0.0 ? h1 / den : 1.0, sv = den != 0.0 ? h2 / den : 0.0;
                cs[cl] = cc;
                sn[cl] = sv;
                H[cl * k + cl] = den;
                H[j * k + cl] = 0.0;
                const double gv = g[cl];
                g[cl] = cc * gv;
                g[j] = -sv * gv;
                s.rnorm = fabs(g[j]);
                s.jpos = j;
                s.it += 1;
                jdone = j;
                if (hj == 0.0) {  // happy breakdown: declared exact (gmres.py:245-248, :262-268)
                    s.stopped = 1;
                    s.stopping_id = EXACT_CONVERGENCE_ID;
                    s.finalized = 1;
                    s.rnorm = 0.0;
                } else if (j < k) {
                    hist_put(&s, hist, s.it, s.rnorm);
                    crit_check(&s, s.it, s.rnorm);
                }
                if (!s.stopped || s.jpos == j) {  // v_j = w / h_{j,j-1}
                    T* vj = V + (int64_t)j * n;
#pragma unroll
                    for (int64_t r = 0; r < n; ++r) vj[r] = hj == 0.0 ? T(0) : (T)((double)w[r] / hj);
                }
            }
            (void)jdone;
            // the cycle ends in a commit when stopped or at j == k (gmres_backsolve_kernel's rule)
            const int jc = s.jpos;
            const bool solve = !s.done && (s.stopped || jc == k);
            sh_jc = jc;
            sh_solve = solve;
            sh_bd = 0;
        }
        __syncwarp();
        // ---- back-solve of the rotated triangle, column by column (warp) ----
        if (sh_solve) {
            const int jc = sh_jc;
            double acc[GMRES_TINY_MAXK / 32];
#pragma unroll
            for (int m = 0; m < GMRES_TINY_MAXK / 32; ++m) acc[m] = 0.0;
            for (int i = jc - 1; i >= 0; --i) {
                const double d = H[i * k + i];
                if (d == 0.0) {  // singular rotated triangle (gmres.py:157-167)
                    if (lane == 0) sh_bd = 1;
                    break;
                }
                double mine = 0.0;
#pragma unroll
                for (int m = 0; m < GMRES_TINY_MAXK / 32; ++m)
                    if (m == (i >> 5)) mine = acc[m];
                const double yi = __shfl_sync(0xffffffffu, (g[i] - mine) / d, i & 31);
                if (lane == (i & 31)) ys[i] = yi;
#pragma unroll
                for (int m = 0; m < GMRES_TINY_MAXK / 32; ++m) {
                    const int r = lane + 32 * m;
                    if (r < i) acc[m] += H[r * k + i] * yi;
                }
            }
        }
        __syncwarp();
        // ---- commit, restart (thread 0): gmres_combine, gmres_after_commit,
        //      the true residual, gmres_reset and gmres_scale_v0 ----
        int fin = 0;
        if (lane == 0) {
            if (sh_bd) {
                s.breakdown = BD_HESSENBERG;
                s.breakdown_it = s.it;
                s.done = 1;
            } else if (sh_solve) {
                const int jc = sh_jc;
#pragma unroll
                for (int64_t r = 0; r < n; ++r) {  // x += V y
                    T u = T(0);
                    for (int q = 0; q < jc; ++q) u += (T)ys[q] * V[(int64_t)q * n + r];
                    x[r] += u;
                }
                if (s.stopped) s.done = 1;
            } else if (s.stopped) {
                s.done = 1;
            }
            if (!s.done) {
#pragma unroll
                for (int64_t r = 0; r < n; ++r) {  // r = b - A x (the fused residual: -acc + b)
                    T acc = 0;
                    for (int q = rp[r]; q < rp[r + 1]; ++q) acc += av[q] * x[ci[q]];
                    w[r] = -acc + bv[r];
                }
                double rr = 0;
#pragma unroll
                for (int64_t r = 0; r < n; ++r) rr += (double)w[r] * (double)w[r];
                const double beta = sqrt(rr);
                for (int i = 0; i <= k; ++i) g[i] = 0.0;
                for (int i = 0; i < k; ++i) cs[i] = sn[i] = 0.0;
                g[0] = beta;
                s.rnorm = beta;
                s.jpos = 0;
                s.committed = 0;
                hist_put(&s, hist, s.it, s.rnorm);
                crit_check(&s, s.it, s.rnorm);
                if (!s.stopped) {
#pragma unroll
                    for (int64_t r = 0; r < n; ++r) V[r] = beta == 0.0 ? T(0) : (T)((double)w[r] / beta);
                }
            }
            fin = s.done;
        }
        fin = __shfl_sync(0xffffffffu, fin, 0);
        if (fin) break;
    }
    if (lane == 0) {
#pragma unroll
        for (int64_t r = 0; r < n; ++r) xg[r] = x[r];
        for (int i = 0; i <= k; ++i) G.g[i] = g[i];
        s.committed = 0;
        *c = s;
    }
}

// back-solve of the rotated triangular system at jc = jpos (gmres.py:157-167)
// One warp: row i's dot with y[i+1:jc] (the reference's h[i, i+1:jc] @ y)
// is spread over the lanes and shuffle-summed -- a single thread's serial
// sweep is jc^2/2 dependent global loads (~340 us per GMRES(100) cycle).
// The triangle is first staged in shared memory with coalesced loads when it
// fits (jc <= GMRES_BS_STAGE): the sweep's dependent steps then read shared
// memory instead of paying an L2 round trip each (GMRES(100): 64 -> ~10 us).
constexpr int GMRES_BS_STAGE = 128;

__global__ void gmres_backsolve_kernel(KrylovCtl* c, double* gm) {
    extern __shared__ double bs_h[];  // GMRES_BS_STAGE^2 (+ GMRES_BS_STAGE for y) doubles
    if (blockIdx.x != 0 || threadIdx.x >= 32) return;
    const int lane = threadIdx.x;
    if (c->done || c->committed) return;
    GmresView G(gm, c->kdim);
    const int jc = c->jpos;
    const bool restart = !c->stopped && jc == G.k;
    if (!(c->stopped || restart)) return;
    const bool staged = jc <= GMRES_BS_STAGE;
    double* ys = bs_h + GMRES_BS_STAGE * GMRES_BS_STAGE;  // y on chip while solving
    if (staged) {
        for (int i = 0; i < jc; ++i)
            for (int q = i + lane; q < jc; q += 32) bs_h[i * GMRES_BS_STAGE + q] = G.H[i * G.k + q];
        __syncwarp();
    }
    for (int i = jc - 1; i >= 0; --i) {
        if (staged) {
            const double d = bs_h[i * GMRES_BS_STAGE + i];
            if (d == 0.0) {
                if (lane == 0) {
                    c->breakdown = BD_HESSENBERG;
                    c->breakdown_it = c->it;
                    c->done = 1;
                }
                return;
            }
            double acc = 0.0;
            for (int q = i + 1 + lane; q < jc; q += 32) acc += bs_h[i * GMRES_BS_STAGE + q] * ys[q];
            acc = warp_sum(acc);
            if (lane == 0) {
                const double yi = (G.g[i] - acc) / d;
                ys[i] = yi;
                G.y[i] = yi;
            }
            __syncwarp();
            continue;
        }
        const double d = G.H[i * G.k + i];
        if (d == 0.0) {
            if (lane == 0) {
                c->breakdown = BD_HESSENBERG;
                c->breakdown_it = c->it;
                c->done = 1;
            }
            return;
        }
        double acc = 0.0;
        for (int q = i + 1 + lane; q < jc; q += 32) acc += G.H[i * G.k + q] * ((volatile double*)G.y)[q];
        acc = warp_sum(acc);
        if (lane == 0) G.y[i] = (G.g[i] - acc) / d;
        __syncwarp();
    }
    if (lane == 0) c->committed = 1;  // combine pending
}

// x += M (V y): u = sum_i y_i v_i row-wise, then the block-Jacobi of u
template <typename T>
__global__ void __launch_bounds__(KRY_BLOCK)
gmres_combine_kernel(RowBlocks rb, const T* __restrict__ V, T* __restrict__ x, int64_t xs, KrylovCtl* c,
                     const double* gm) {
    if (c->done || !c->committed) return;
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int jc = c->jpos;
    const double* y = gm + (size_t)(c->kdim + 1) * c->kdim + 3 * (size_t)c->kdim + 1;
    for (int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < rb.count(); b += nw) {
        int64_t r0;
        int bs;
        rb.range(b, r0, bs);
        T u = T(0);
        if (lane < bs)
            for (int q = 0; q < jc; ++q) u += (T)y[q] * V[(int64_t)q * rb.n + r0 + lane];
        if (rb.J.nblocks) u = jacobi_row<T>(rb.J, b, bs, lane, u);
        if (lane < bs) x[(r0 + lane) * xs] += u;
    }
}

// after the commit: a stopped solve is finished; a restart keeps going
__global__ void gmres_after_commit_kernel(KrylovCtl* c) {
    if (threadIdx.x != 0 || blockIdx.x != 0 || c->done) return;
    if (c->committed) {
        c->committed = 0;
        if (c->stopped) c->done = 1;
    } else if (c->stopped) {
        c->done = 1;  // stopped with nothing to commit (jc = 0)
    }
}

}  // namespace b200sp

// ===========================================================================
// C ABI
// ===========================================================================
using namespace b200sp;

static RowBlocks make_rb(int64_t n, int64_t nb, const int32_t* starts, const int64_t* offs, const uint8_t* prec,
                         const void* storage) {
    return RowBlocks{n, JacobiView{nb, starts, (const long long*)offs, prec, (const unsigned char*)storage}};
}

namespace b200sp {

// ===========================================================================
// Csr SpMV with the solver's next reduction fused into its epilogue:
//   q = A p and
//   PH_SIGMA (CG):        sigma = p.q                -> cg_sigma_ctl
//   PH_GAMMA (BiCGSTAB):  gamma = rt.q  (u = rt)      -> bicg_gamma_ctl
//   PH_TST   (BiCGSTAB):  ts = q.s, tt = q.q (u = s)  -> bicg_tst_ctl
// Rows as in the classical SpMV (sub-warp per row, L1-allocating matrix
// loads, spmv.cu); the owner lane of a row multiplies the fresh q_i by p_i /
// u_i, so the separate dot kernel's re-read of p and q (2n values per
// iteration, ~9% of a 7-point CG iteration) disappears. Same ticket / block
// order determinism as every other reduction here.
// ===========================================================================
// PH_SIGMA_ACC (distributed CG, ghost block): q += A_ghost p_ghost and
// sigma = u.q with u = the owned p (the SpMV input is the ghost vector)
// (Round 1's phase 5 -- CgStep1 folded into the SpMV, p recomputed for every
// gathered column -- measured no faster than the separate step and was
// removed; the cooperative small-system CG keeps that idea on chip.)
enum FusedPhase : int { PH_SIGMA = 1, PH_GAMMA = 2, PH_TST = 3, PH_SIGMA_ACC = 4 };

// 8 CTAs per SM (<= 32 registers): the unbounded build took 40 registers at
// sub-warp 1 (6 CTAs per SM) and ran slower than SpMV + separate dot
// MODE (U = 1 only; both keep the loop's entry order, so the same sums):
// 1 = entries in predicated blocks of 4 per lane (all loads of a block in
// flight, no dependent remainder loop); 2 = thread per row reading aligned
// (index, value) pairs in blocks of 2 (needs 16-byte aligned arrays and an
// even entry count) -- the SpMV kernel's variants (spmv.cu csr_classical)
template <typename T> struct KVec2;
template <> struct KVec2<double> { using type = double2; };
template <> struct KVec2<float> { using type = float2; };

template <typename T, int SW, int PH, int MODE = 0>
__global__ void __launch_bounds__(KRY_BLOCK, SW <= 4 ? 8 : 4)
csr_spmv_dot_kernel(int64_t n, const int* __restrict__ rp, const int* __restrict__ ci, const T* __restrict__ av,
                    const T* __restrict__ p, T* __restrict__ q, const T* __restrict__ u, KrylovCtl* c,
                    double* part) {
    if (c->done) return;
    constexpr int U = SW >= 32 ? 4 : (SW >= 8 ? 2 : 1);
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & (SW - 1);
    const int64_t nsw = (int64_t)gridDim.x * blockDim.x / SW;
    double d0 = 0, d1 = 0;
    const int64_t wfirst = (tid / 32) * (32 / SW) * U;
    for (int64_t row0 = (tid / SW) * U, w0 = wfirst; w0 < n; row0 += nsw * U, w0 += nsw * U) {
        int st[U], len[U];
        int nxt = row0 < n ? __ldg(rp + row0) : 0;
        int maxlen = 0;
#pragma unroll
        for (int k = 0; k < U; ++k) {
            st[k] = nxt;
            nxt = (row0 + k < n) ? __ldg(rp + row0 + k + 1) : nxt;
            len[k] = nxt - st[k];
            maxlen = max(maxlen, len[k]);
        }
        T acc[U];
#pragma unroll
        for (int k = 0; k < U; ++k) acc[k] = 0;
        if (MODE == 2 && U == 1 && SW == 1) {
            const int s0 = st[0], e0 = st[0] + len[0];
#pragma unroll 1
            for (int k0 = s0 & ~1; k0 < e0; k0 += 4) {
                int2 cc[2];
                typename KVec2<T>::type vv[2];
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    const int k = k0 + 2 * j;
                    if (k < e0) {
                        cc[j] = __ldg(reinterpret_cast<const int2*>(ci + k));
                        vv[j] = __ldg(reinterpret_cast<const typename KVec2<T>::type*>(av + k));
                    } else {
                        cc[j] = make_int2(-1, -1);
                    }
                }
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    const int k = k0 + 2 * j;
                    if (k >= s0 && cc[j].x >= 0) acc[0] += vv[j].x * __ldg(p + cc[j].x);
                    if (k + 1 < e0 && cc[j].y >= 0) acc[0] += vv[j].y * __ldg(p + cc[j].y);
                }
            }
        } else if (MODE >= 1 && U == 1) {
#pragma unroll 1
            for (int e0 = lane; e0 < maxlen; e0 += 4 * SW) {
                int cc[4];
                T vv[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int e = e0 + j * SW;
                    const bool ok = e < len[0];
                    cc[j] = ok ? __ldg(ci + st[0] + e) : -1;
                    vv[j] = ok ? __ldg(av + st[0] + e) : T(0);
                }
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (cc[j] >= 0) acc[0] += vv[j] * __ldg(p + cc[j]);
            }
        } else
        for (int e = lane; e < maxlen; e += SW) {
            int cc[U];
            T vv[U];
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const bool ok = e < len[k];
                cc[k] = ok ? __ldg(ci + st[k] + e) : -1;
                vv[k] = ok ? __ldg(av + st[k] + e) : T(0);
            }
#pragma unroll
            for (int k = 0; k < U; ++k)
                if (cc[k] >= 0) acc[k] += vv[k] * __ldg(p + cc[k]);
        }
#pragma unroll
        for (int k = 0; k < U; ++k) acc[k] = subwarp_sum<SW>(acc[k]);
#pragma unroll
        for (int k = 0; k < U; ++k) {  // row k written by lane k % SW (U may exceed SW)
            const int64_t row = row0 + k;
            if (k % SW == lane && row < n) {
                T mine = acc[k];
                if (PH == PH_SIGMA_ACC) {
                    mine += q[row];
                    d0 += (double)__ldg(u + row) * (double)mine;
                }
                q[row] = mine;
                if (PH == PH_SIGMA) d0 += (double)__ldg(p + row) * (double)mine;
                if (PH == PH_GAMMA) d0 += (double)__ldg(u + row) * (double)mine;
                if (PH == PH_TST) {
                    d0 += (double)mine * (double)__ldg(u + row);
                    d1 += (double)mine * (double)mine;
                }
            }
        }
    }
    if (PH == PH_TST) {
        double v[2] = {d0, d1}, tot[2];
        if (!grid_reduce<2>(v, part, &c->ticket[1], tot)) return;
        bicg_tst_ctl(c, tot);
    } else {
        double v[1] = {d0}, tot[1];
        if (!grid_reduce<1>(v, part, &c->ticket[1], tot)) return;
        if (PH == PH_SIGMA || PH == PH_SIGMA_ACC) {
            if (c->dist) {
                c->red[0] = tot[0];
                return;
            }
            cg_sigma_ctl(c, tot);
        } else {
            bicg_gamma_ctl(c, tot);
        }
    }
}

template <typename T, int SW, int MODE>
static void launch_spmv_dot_m(int64_t n, const int* rp, const int* ci, const T* av, const T* p, T* q, const T* u,
                              int phase, KrylovCtl* c, double* part, cudaStream_t st) {
    constexpr int U = SW >= 32 ? 4 : (SW >= 8 ? 2 : 1);
    const int grid = kry_grid(ceil_div(n, U) * SW, KRY_BLOCK);
    if (phase == PH_SIGMA) csr_spmv_dot_kernel<T, SW, PH_SIGMA, MODE><<<grid, KRY_BLOCK, 0, st>>>(n, rp, ci, av, p, q, u, c, part);
    else if (phase == PH_GAMMA) csr_spmv_dot_kernel<T, SW, PH_GAMMA, MODE><<<grid, KRY_BLOCK, 0, st>>>(n, rp, ci, av, p, q, u, c, part);
    else if (phase == PH_SIGMA_ACC) csr_spmv_dot_kernel<T, SW, PH_SIGMA_ACC, MODE><<<grid, KRY_BLOCK, 0, st>>>(n, rp, ci, av, p, q, u, c, part);
    else csr_spmv_dot_kernel<T, SW, PH_TST, MODE><<<grid, KRY_BLOCK, 0, st>>>(n, rp, ci, av, p, q, u, c, part);
}
template <typename T, int SW>
static void launch_spmv_dot(int64_t n, const int* rp, const int* ci, const T* av, const T* p, T* q, const T* u,
                            int phase, KrylovCtl* c, double* part, bool even_nnz, cudaStream_t st) {
    // knob "spmv_dot_mode": 0 = loop, 1 = 4-entry blocks, 2 = pairs (thread per row)
    const bool pairs = SW == 1 && even_nnz && ((reinterpret_cast<uintptr_t>(ci) | reinterpret_cast<uintptr_t>(av)) & 15) == 0;
    int mode = tuning("spmv_dot_mode", pairs ? 2 : 1);
    if (mode == 2 && !pairs) mode = 1;
    if (SW >= 8) mode = 0;  // U > 1: the loop form
    if (mode == 2) launch_spmv_dot_m<T, SW, 2>(n, rp, ci, av, p, q, u, phase, c, part, st);
    else if (mode == 1) launch_spmv_dot_m<T, SW, 1>(n, rp, ci, av, p, q, u, phase, c, part, st);
    else launch_spmv_dot_m<T, SW, 0>(n, rp, ci, av, p, q, u, phase, c, part, st);
}

template <typename T>
static int csr_spmv_dot(int64_t n, const int* rp, const int* ci, const T* av, const T* p, T* q, const T* u,
                        int phase, int subwarp, void* ctl, double* part, void* stream) {
    B200SP_REQUIRE(phase >= PH_SIGMA && phase <= PH_SIGMA_ACC, B200SP_EINVAL, "csr_spmv_dot: phase must be 1..4");
    B200SP_REQUIRE(phase == PH_SIGMA || u, B200SP_EINVAL, "csr_spmv_dot: phase %d needs the second vector", phase);
    if (n == 0) return B200SP_OK;
    cudaStream_t st = as_stream(stream);
    KrylovCtl* c = (KrylovCtl*)ctl;
    const bool ev = (subwarp & B200SP_SUBWARP_EVEN_NNZ) != 0;
    subwarp &= ~B200SP_SUBWARP_EVEN_NNZ;
    switch (subwarp) {
        case 1: launch_spmv_dot<T, 1>(n, rp, ci, av, p, q, u, phase, c, part, ev, st); break;
        case 2: launch_spmv_dot<T, 2>(n, rp, ci, av, p, q, u, phase, c, part, ev, st); break;
        case 4: launch_spmv_dot<T, 4>(n, rp, ci, av, p, q, u, phase, c, part, ev, st); break;
        case 8: launch_spmv_dot<T, 8>(n, rp, ci, av, p, q, u, phase, c, part, ev, st); break;
        case 16: launch_spmv_dot<T, 16>(n, rp, ci, av, p, q, u, phase, c, part, ev, st); break;
        case 32: launch_spmv_dot<T, 32>(n, rp, ci, av, p, q, u, phase, c, part, ev, st); break;
        default: set_error("csr_spmv_dot: subwarp must be a power of two <= 32 (got %d)", subwarp); return B200SP_EINVAL;
    }
    count_launch();
    return check_launch("csr_spmv_dot");
}

}  // namespace b200sp

#define KRY_LAUNCH(kernel, units, per_block, ...)                                                     \
    do {                                                                                              \
        kernel<<<kry_grid((units), (per_block)), KRY_BLOCK, 0, as_stream(stream)>>>(__VA_ARGS__);     \
        count_launch();                                                                               \
        return check_launch(#kernel);                                                                 \
    } while (0)

#define JAC_ARGS int64_t jnb, const int32_t *jstarts, const int64_t *joffs, const uint8_t *jprec, const void *jstore
#define RB(n) make_rb((n), jnb, jstarts, joffs, jprec, jstore)
#define RB_UNITS(n) (jnb ? jnb * 32 : ((n) + 31) / 32 * 32)

__global__ void krylov_start_clock_kernel(KrylovCtl* c) { c->t_start = global_ns(); }

extern "C" {

int64_t b200sp_krylov_ctl_bytes(void) { return (int64_t)sizeof(KrylovCtl); }
int64_t b200sp_krylov_part_elems(void) { return (int64_t)(KRY_NRED + 2) * KRY_MAX_GRID; }  // + flagged slots

int b200sp_krylov_ctl_init(void* ctl, int32_t n_crit, const int32_t* crit_type, const double* crit_param,
                           int32_t needs_residual, int32_t hist_cap, int32_t kdim, void* stream) {
    B200SP_REQUIRE(n_crit >= 0 && n_crit <= KRY_MAX_CRIT, B200SP_EINVAL, "krylov: at most %d criteria", KRY_MAX_CRIT);
    KrylovCtl h;
    memset(&h, 0, sizeof(h));
    h.n_crit = n_crit;
    for (int i = 0; i < n_crit; ++i) {
        h.crit_type[i] = crit_type[i];
        h.crit_param[i] = crit_param[i];
    }
    h.needs_residual = needs_residual;
    h.hist_cap = hist_cap;
    h.kdim = kdim;
    B200SP_CHECK_CUDA(cudaMemcpyAsync(ctl, &h, sizeof(h), cudaMemcpyHostToDevice, as_stream(stream)));
    krylov_start_clock_kernel<<<1, 1, 0, as_stream(stream)>>>((KrylovCtl*)ctl);  // TimeLimit origin
    count_launch();
    B200SP_CHECK_CUDA(cudaStreamSynchronize(as_stream(stream)));  // &h is a stack buffer
    return check_launch("krylov_ctl_init");
}

// status: ints [it, stopped, stopping_id, finalized, done, breakdown, breakdown_it, jpos]
//         doubles [baseline, rnorm, rho, alpha, omega, snorm, hnorm, sigma]
int b200sp_krylov_status(const void* ctl, int32_t* out_i, double* out_d, void* stream) {
    KrylovCtl h;
    B200SP_CHECK_CUDA(cudaMemcpyAsync(&h, ctl, sizeof(h), cudaMemcpyDeviceToHost, as_stream(stream)));
    B200SP_CHECK_CUDA(cudaStreamSynchronize(as_stream(stream)));
    const int iv[8] = {h.it, h.stopped, h.stopping_id, h.finalized, h.done, h.breakdown, h.breakdown_it, h.jpos};
    const double dv[8] = {h.baseline, h.rnorm, h.rho, h.alpha, h.omega, h.snorm, h.hnorm, h.sigma};
    memcpy(out_i, iv, sizeof(iv));
    memcpy(out_d, dv, sizeof(dv));
    return B200SP_OK;
}

// host-side stop (TimeLimit): mark stopped with the given id
__global__ void krylov_force_stop_kernel(KrylovCtl* c, int id, int gmres) {
    if (c->stopped || c->done) return;
    c->stopped = 1;
    c->stopping_id = id;
    c->finalized = 1;
    if (!gmres) c->done = 1;
}
int b200sp_krylov_force_stop(void* ctl, int32_t stopping_id, int32_t gmres, void* stream) {
    krylov_force_stop_kernel<<<1, 1, 0, as_stream(stream)>>>((KrylovCtl*)ctl, stopping_id, gmres);
    count_launch();
    return check_launch("krylov_force_stop");
}

const int32_t* b200sp_krylov_guard(const void* ctl, int32_t which) {
    const KrylovCtl* c = (const KrylovCtl*)ctl;
    return which == 1 ? &c->stopped : &c->done;
}

#define KRYLOV_T(T, SUF)                                                                                          \
    int b200sp_cg_init_##SUF(int64_t n, const T* r, T* z, T* p, JAC_ARGS, void* ctl, double* part, double* hist,  \
                             void* stream) {                                                                      \
        KRY_LAUNCH(cg_init_kernel<T>, RB_UNITS(n), KRY_BLOCK, RB(n), r, z, p, (KrylovCtl*)ctl, part, hist);       \
    }                                                                                                             \
    int b200sp_cg_step1_##SUF(int64_t n, T* p, const T* z, const void* ctl, void* stream) {                        \
        KRY_LAUNCH(cg_step1_kernel<T>, n, KRY_BLOCK, n, p, z, (const KrylovCtl*)ctl);                             \
    }                                                                                                             \
    int b200sp_cg_sigma_##SUF(int64_t n, const T* p, const T* q, void* ctl, double* part, void* stream) {          \
        KRY_LAUNCH(cg_sigma_kernel<T>, n, KRY_BLOCK, n, p, q, (KrylovCtl*)ctl, part);                             \
    }                                                                                                             \
    int b200sp_fcg_step2_##SUF(int64_t n, T* x, int64_t xs, T* r, const T* p, const T* q, T* t, T* z, JAC_ARGS,    \
                               void* ctl, double* part, double* hist, void* stream) {                             \
        KRY_LAUNCH(fcg_step2_kernel<T>, RB_UNITS(n), KRY_BLOCK, RB(n), x, xs, r, p, q, t, z, (KrylovCtl*)ctl, part, \
                   hist);                                                                                         \
    }                                                                                                             \
    int b200sp_cg_step2_##SUF(int64_t n, T* x, int64_t xs, T* r, const T* p, const T* q, T* z, JAC_ARGS,           \
                              void* ctl, double* part, double* hist, void* stream) {                              \
        KRY_LAUNCH(cg_step2_kernel<T>, RB_UNITS(n), KRY_BLOCK, RB(n), x, xs, r, p, q, z, (KrylovCtl*)ctl, part,   \
                   hist);                                                                                         \
    }                                                                                                             \
    int b200sp_bicgstab_init_##SUF(int64_t n, const T* b, int64_t bs, const T* r, T* rt, T* p, T* v, T* s, T* t,   \
                                   T* y, T* z, void* ctl, double* part, double* hist, void* stream) {             \
        KRY_LAUNCH(bicg_init_kernel<T>, n, KRY_BLOCK, n, b, bs, r, rt, p, v, s, t, y, z, (KrylovCtl*)ctl, part,   \
                   hist);                                                                                         \
    }                                                                                                             \
    int b200sp_bicgstab_step1_##SUF(int64_t n, const T* r, T* p, const T* v, T* y, JAC_ARGS, const void* ctl,     \
                                    void* stream) {                                                               \
        KRY_LAUNCH(bicg_step1_kernel<T>, RB_UNITS(n), KRY_BLOCK, RB(n), r, p, v, y, (const KrylovCtl*)ctl);       \
    }                                                                                                             \
    int b200sp_bicgstab_gamma_##SUF(int64_t n, const T* rt, const T* v, void* ctl, double* part, void* stream) {  \
        KRY_LAUNCH(bicg_gamma_kernel<T>, n, KRY_BLOCK, n, rt, v, (KrylovCtl*)ctl, part);                          \
    }                                                                                                             \
    int b200sp_bicgstab_step2_##SUF(int64_t n, const T* r, const T* v, T* s, T* z, JAC_ARGS, void* ctl,           \
                                    double* part, double* hist, void* stream) {                                   \
        KRY_LAUNCH(bicg_step2_kernel<T>, RB_UNITS(n), KRY_BLOCK, RB(n), r, v, s, z, (KrylovCtl*)ctl, part, hist); \
    }                                                                                                             \
    int b200sp_bicgstab_tst_##SUF(int64_t n, const T* t, const T* s, void* ctl, double* part, void* stream) {     \
        KRY_LAUNCH(bicg_tst_kernel<T>, n, KRY_BLOCK, n, t, s, (KrylovCtl*)ctl, part);                             \
    }                                                                                                             \
    int b200sp_bicgstab_step3_##SUF(int64_t n, T* x, int64_t xs, T* r, const T* s, const T* t, const T* y,        \
                                    const T* z, const T* rt, void* ctl, double* part, double* hist,               \
                                    void* stream) {                                                               \
        KRY_LAUNCH(bicg_step3_kernel<T>, n, KRY_BLOCK, n, x, xs, r, s, t, y, z, rt, (KrylovCtl*)ctl, part, hist); \
    }                                                                                                             \
    int b200sp_cgs_step1_##SUF(int64_t n, const T* r, const T* q, T* u, T* p, T* ph, JAC_ARGS, const void* ctl,   \
                               void* stream) {                                                                    \
        KRY_LAUNCH(cgs_step1_kernel<T>, RB_UNITS(n), KRY_BLOCK, RB(n), r, q, u, p, ph, (const KrylovCtl*)ctl);     \
    }                                                                                                             \
    int b200sp_cgs_step2_##SUF(int64_t n, const T* u, const T* vh, T* q, T* w, T* uh, JAC_ARGS, const void* ctl,  \
                               void* stream) {                                                                    \
        KRY_LAUNCH(cgs_step2_kernel<T>, RB_UNITS(n), KRY_BLOCK, RB(n), u, vh, q, w, uh, (const KrylovCtl*)ctl);    \
    }                                                                                                             \
    int b200sp_cgs_step3_##SUF(int64_t n, T* x, int64_t xs, T* r, const T* t, const T* uh, const T* rt, void* ctl, \
                               double* part, double* hist, void* stream) {                                        \
        KRY_LAUNCH(cgs_step3_kernel<T>, n, KRY_BLOCK, n, x, xs, r, t, uh, rt, (KrylovCtl*)ctl, part, hist);        \
    }                                                                                                             \
    int b200sp_gmres_reset_##SUF(int64_t n, const T* r, void* ctl, double* part, double* gm, double* hist,        \
                                 int32_t first, void* stream) {                                                   \
        KRY_LAUNCH(gmres_reset_kernel<T>, n, KRY_BLOCK, n, r, (KrylovCtl*)ctl, part, gm, hist, first);            \
    }                                                                                                             \
    int b200sp_gmres_scale_v0_##SUF(int64_t n, const T* r, T* V, const void* ctl, void* stream) {                 \
        KRY_LAUNCH(gmres_scale_v0_kernel<T>, n, KRY_BLOCK, n, r, V, (const KrylovCtl*)ctl);                       \
    }                                                                                                             \
    int b200sp_gmres_dot0_##SUF(int64_t n, int32_t j, const T* V, const T* w, void* ctl, double* part, double* gm, \
                                void* stream) {                                                                   \
        KRY_LAUNCH(gmres_dot0_kernel<T>, n, KRY_BLOCK, n, j, V, w, (KrylovCtl*)ctl, part, gm);                    \
    }                                                                                                             \
    int b200sp_gmres_mgs_##SUF(int64_t n, int32_t j, int32_t i, const T* V, T* w, void* ctl, double* part,        \
                               double* gm, double* hist, void* stream) {                                          \
        KRY_LAUNCH(gmres_mgs_kernel<T>, n, KRY_BLOCK, n, j, i, V, w, (KrylovCtl*)ctl, part, gm, hist);            \
    }                                                                                                             \
    int b200sp_gmres_arnoldi_small_##SUF(int64_t n, int32_t j, T* V, T* w, void* ctl, double* gm, double* hist, \
                                         void* stream) {                                                          \
        B200SP_REQUIRE(n <= GMRES_SMALL_ROWS, B200SP_EINVAL, "gmres_arnoldi_small: n must be <= %d",             \
                       GMRES_SMALL_ROWS);                                                                         \
        gmres_arnoldi_small_kernel<T><<<1, KRY_BLOCK, 0, as_stream(stream)>>>(n, j, V, w, (KrylovCtl*)ctl, gm, hist); \
        count_launch();                                                                                           \
        return check_launch("gmres_arnoldi_small");                                                               \
    }                                                                                                             \
    int b200sp_gmres_cycle_small_##SUF(int64_t n, const int32_t* rp, const int32_t* ci, const T* v, T* V, T* w,  \
                                       void* ctl, double* gm, double* hist, void* stream) {                      \
        B200SP_REQUIRE(n <= GMRES_SMALL_ROWS, B200SP_EINVAL, "gmres_cycle_small: n must be <= %d",               \
                       GMRES_SMALL_ROWS);                                                                         \
        if (n <= 32 * GMRES_SMALL_RPT) /* one warp: reductions without block barriers */                        \
            gmres_cycle_small_kernel<T, 32><<<1, 32, GMRES_SMEM_BYTES, as_stream(stream)>>>(n, rp, ci, v, V, w,  \
                                                                                           (KrylovCtl*)ctl, gm, hist); \
        else                                                                                                      \
            gmres_cycle_small_kernel<T, KRY_BLOCK><<<1, KRY_BLOCK, GMRES_SMEM_BYTES, as_stream(stream)>>>(         \
                n, rp, ci, v, V, w, (KrylovCtl*)ctl, gm, hist);                                                   \
        count_launch();                                                                                           \
        return check_launch("gmres_cycle_small");                                                                 \
    }                                                                                                             \
    int b200sp_gmres_solve_tiny_##SUF(int64_t n, const int32_t* rp, const int32_t* ci, const T* v, T* x,        \
                                      const T* b, T* V, T* w, void* ctl, double* gm, double* hist, int32_t k,    \
                                      void* stream) {                                                             \
        B200SP_REQUIRE(n >= 1 && n <= GMRES_TINY_ROWS && k >= 1 && k <= GMRES_TINY_MAXK, B200SP_EINVAL,          \
                       "gmres_solve_tiny: n must be 1..%d and k 1..%d", GMRES_TINY_ROWS, GMRES_TINY_MAXK);       \
        const size_t sm = gmres_tiny_smem(k, n, sizeof(T));                                                      \
        auto kern = n == 1 ? gmres_solve_tiny_kernel<T, 1> : n == 2 ? gmres_solve_tiny_kernel<T, 2>               \
                  : n == 3 ? gmres_solve_tiny_kernel<T, 3> : gmres_solve_tiny_kernel<T, 4>;                        \
        B200SP_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));      \
        kern<<<1, 32, sm, as_stream(stream)>>>(rp, ci, v, x, b, V, w, (KrylovCtl*)ctl, gm, hist);                \
        count_launch();                                                                                           \
        return check_launch("gmres_solve_tiny");                                                                  \
    }                                                                                                             \
    int b200sp_gmres_normalize_##SUF(int64_t n, int32_t j, T* V, const T* w, const void* ctl, void* stream) {     \
        KRY_LAUNCH(gmres_normalize_kernel<T>, n, KRY_BLOCK, n, j, V, w, (const KrylovCtl*)ctl);                   \
    }                                                                                                             \
    int b200sp_gmres_combine_##SUF(int64_t n, const T* V, T* x, int64_t xs, JAC_ARGS, void* ctl, const double* gm, \
                                   void* stream) {                                                                \
        KRY_LAUNCH(gmres_combine_kernel<T>, RB_UNITS(n), KRY_BLOCK, RB(n), V, x, xs, (KrylovCtl*)ctl, gm);        \
    }

KRYLOV_T(double, f64)
KRYLOV_T(float, f32)

int32_t b200sp_gmres_small_rows(void) { return GMRES_SMALL_ROWS; }

int b200sp_gmres_backsolve(void* ctl, double* gm, void* stream) {
    constexpr int smem = (GMRES_BS_STAGE * GMRES_BS_STAGE + GMRES_BS_STAGE) * (int)sizeof(double);
    static bool attr = false;
    if (!attr) {
        B200SP_CHECK_CUDA(cudaFuncSetAttribute(gmres_backsolve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        attr = true;
    }
    gmres_backsolve_kernel<<<1, 32, smem, as_stream(stream)>>>((KrylovCtl*)ctl, gm);
    count_launch();
    return check_launch("gmres_backsolve");
}
int b200sp_gmres_after_commit(void* ctl, void* stream) {
    gmres_after_commit_kernel<<<1, 32, 0, as_stream(stream)>>>((KrylovCtl*)ctl);
    count_launch();
    return check_launch("gmres_after_commit");
}
int64_t b200sp_gmres_workspace_elems(int32_t k) { return (int64_t)(k + 1) * k + 3 * (int64_t)k + 1 + k; }

}  // extern "C"

namespace b200sp {

template <typename T, int N>
__global__ void __launch_bounds__(32)
fcg_tiny_kernel(const int* __restrict__ rp, const int* __restrict__ ci, const T* __restrict__ avg, T* x_g, T* r_g,
                T* p_g, T* q_g, T* t_g, KrylovCtl* c, double* hist) {
    if (threadIdx.x != 0) return;
    TinyCsr<T, N> A;
    A.load(rp, ci, avg);
    KrylovCtl sc = *c;
    T x[N], r[N], p[N], q[N], t[N];
#pragma unroll
    for (int i = 0; i < N; ++i) x[i] = x_g[i], r[i] = r_g[i], p[i] = p_g[i], q[i] = q_g[i], t[i] = t_g[i];
    while (!sc.done) {
        const T beta = (T)sc.beta;
#pragma unroll
        for (int i = 0; i < N; ++i) p[i] = r[i] + beta * p[i];  // CgStep1 (z = r)
        A.apply(p, q);
        double sg = 0;
#pragma unroll
        for (int i = 0; i < N; ++i) sg += (double)p[i] * (double)q[i];
        {
            const double tot[1] = {sg};
            cg_sigma_ctl(&sc, tot);
        }
        if (sc.done) break;
        const T alpha = (T)sc.alpha;
        double rz = 0, tz = 0, rr = 0;
#pragma unroll
        for (int i = 0; i < N; ++i) {  // FcgStep2
            x[i] = x[i] + mul_rn(alpha, p[i]);
            const T ro = r[i];
            const T rv = ro - mul_rn(alpha, q[i]);
            const T tv = rv - ro;
            t[i] = tv;
            r[i] = rv;
            rz += (double)rv * (double)rv;
            tz += (double)tv * (double)rv;
            rr += (double)rv * (double)rv;
        }
        sc.rho_prev = sc.rho;
        sc.rho = rz;
        sc.rho_t = tz;
        sc.it += 1;
        sc.rnorm = sqrt(rr);
        hist_put(&sc, hist, sc.it, sc.rnorm);
        crit_check(&sc, sc.it, sc.rnorm);
        sc.done = sc.stopped;
        sc.beta = safe_div(sc.rho_t, sc.rho_prev);
    }
#pragma unroll
    for (int i = 0; i < N; ++i) x_g[i] = x[i], r_g[i] = r[i], p_g[i] = p[i], q_g[i] = q[i], t_g[i] = t[i];
    *c = sc;
}

template <typename T, int N>
__global__ void __launch_bounds__(32)
cgs_tiny_kernel(const int* __restrict__ rp, const int* __restrict__ ci, const T* __restrict__ avg, T* x_g, T* r_g,
                const T* __restrict__ rt_g, T* p_g, T* q_g, T* u_g, T* vh_g, T* w_g, T* t_g, KrylovCtl* c,
                double* hist) {
    if (threadIdx.x != 0) return;
    TinyCsr<T, N> A;
    A.load(rp, ci, avg);
    KrylovCtl sc = *c;
    T x[N], r[N], rt[N], p[N], q[N], u[N], vh[N], w[N], t[N];
#pragma unroll
    for (int i = 0; i < N; ++i)
        x[i] = x_g[i], r[i] = r_g[i], rt[i] = rt_g[i], p[i] = p_g[i], q[i] = q_g[i], u[i] = u_g[i], vh[i] = vh_g[i],
        w[i] = w_g[i], t[i] = t_g[i];
    while (!sc.done) {
        {   // u = r + beta q; p = u + beta (q + beta p)   (CgsStep1)
            const T beta = (T)sc.beta;
#pragma unroll
            for (int i = 0; i < N; ++i) {
                const T qv = q[i];
                const T uv = r[i] + mul_rn(beta, qv);
                u[i] = uv;
                p[i] = uv + mul_rn(beta, qv + mul_rn(beta, p[i]));
            }
        }
        A.apply(p, vh);  // v_hat = A p; gamma = rt.v_hat
        double g = 0;
#pragma unroll
        for (int i = 0; i < N; ++i) g += (double)rt[i] * (double)vh[i];
        {
            const double tot[1] = {g};
            bicg_gamma_ctl(&sc, tot);
        }
        if (sc.done) break;
        const T alpha = (T)sc.alpha;
#pragma unroll
        for (int i = 0; i < N; ++i) {  // q = u - alpha v_hat; w = u + q   (CgsStep2)
            const T uv = u[i];
            const T qv = uv - mul_rn(alpha, vh[i]);
            q[i] = qv;
            w[i] = uv + qv;
        }
        sc.it += 1;  // mid check on the unchanged ||r|| (krylov.py:171-176)
        hist_put(&sc, hist, sc.it, sc.rnorm);
        crit_check(&sc, sc.it, sc.rnorm);
        sc.done = sc.stopped;
        if (sc.done) break;
        A.apply(w, t);  // t = A w; r -= alpha t; x += alpha w   (CgsStep3)
        double rr = 0, rtr = 0;
#pragma unroll
        for (int i = 0; i < N; ++i) {
            const T rv = r[i] - mul_rn(alpha, t[i]);
            r[i] = rv;
            x[i] = x[i] + mul_rn(alpha, w[i]);
            rr += (double)rv * (double)rv;
            rtr += (double)rt[i] * (double)rv;
        }
        sc.rho_prev = sc.rho;
        sc.it += 1;
        sc.rnorm = sqrt(rr);
        hist_put(&sc, hist, sc.it, sc.rnorm);
        crit_check(&sc, sc.it, sc.rnorm);
        sc.done = sc.stopped;
        cgs_cycle_start(&sc, rtr, rr);
    }
#pragma unroll
    for (int i = 0; i < N; ++i)
        x_g[i] = x[i], r_g[i] = r[i], p_g[i] = p[i], q_g[i] = q[i], u_g[i] = u[i], vh_g[i] = vh[i], w_g[i] = w[i],
        t_g[i] = t[i];
    *c = sc;
}

}  // namespace b200sp

// tiny systems (n <= 32 rows): the one-block cooperative solve runs as ONE
// warp -- its block reductions and barriers then never leave the warp
static unsigned coop_threads(int64_t n) { return n <= 32 && tuning("coop_tiny_warp", 1) ? 32u : (unsigned)KRY_BLOCK; }

template <typename T>
static int cg_coop(int64_t n, const int32_t* rp, const int32_t* ci, const T* v, T* x, T* r, T* p, T* p2, T* q, void* ctl,
                   double* part, double* hist, void* stream) {
    if (n >= 1 && n <= TINY_ROWS && tuning("coop_tiny", 1)) {  // one thread, registers only
        KrylovCtl* c = (KrylovCtl*)ctl;
        auto k = n == 1 ? cg_tiny_kernel<T, 1> : n == 2 ? cg_tiny_kernel<T, 2> : n == 3 ? cg_tiny_kernel<T, 3>
                                                                                      : cg_tiny_kernel<T, 4>;
        k<<<1, 32, 0, as_stream(stream)>>>(rp, ci, v, x, r, p, c, hist);
        count_launch();
        return check_launch("cg_tiny");
    }
    int dev = 0, sms = 0, per_sm = 0;
    B200SP_CHECK_CUDA(cudaGetDevice(&dev));
    B200SP_CHECK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    B200SP_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cg_coop_kernel<T>, KRY_BLOCK, 0));
    int64_t grid = (int64_t)sms * per_sm;
    if (grid > KRY_MAX_GRID) grid = KRY_MAX_GRID;
    const int64_t need = ceil_div(n, KRY_BLOCK);
    if (grid > need) grid = need;
    const int cap = tuning("coop_blocks", 0);  // sweep knob: fewer blocks = cheaper grid barriers
    const unsigned threads = coop_threads(n);
    if (cap > 0 && grid > cap) grid = cap;
    if (grid < 1) grid = 1;
    KrylovCtl* c = (KrylovCtl*)ctl;
    void* args[] = {&n, (void*)&rp, (void*)&ci, (void*)&v, &x, &r, &p, &p2, &q, &c, &part, &hist};
    // the register-resident kernel when a thread owns at most 2 rows of a
    // co-resident grid of CG_RES_BLOCK-thread CTAs (larger CTAs: fewer
    // partials to exchange per barrier)
    const void* fn = (const void*)cg_coop_kernel<T>;
    const int res_bs = tuning("coop_res_block", 512);
    if (n > 32 && tuning("coop_resident", 1) && (res_bs == 256 || res_bs == 512 || res_bs == 1024)) {
        for (int rpt = 1; rpt <= 2 && fn == (const void*)cg_coop_kernel<T>; ++rpt) {
            const void* res =
                res_bs == 256 ? (rpt == 1 ? (const void*)cg_coop_res_kernel<T, 1, 8, 256> : (const void*)cg_coop_res_kernel<T, 2, 8, 256>)
                : res_bs == 512 ? (rpt == 1 ? (const void*)cg_coop_res_kernel<T, 1, 8, 512> : (const void*)cg_coop_res_kernel<T, 2, 8, 512>)
                                : (rpt == 1 ? (const void*)cg_coop_res_kernel<T, 1, 8, 1024> : (const void*)cg_coop_res_kernel<T, 2, 8, 1024>);
            int per_sm_res = 0;
            B200SP_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_res, res, res_bs, 0));
            int64_t g = ceil_div(n, (int64_t)res_bs * rpt);
            if (cap > 0 && g > cap) continue;
            if (g <= (int64_t)per_sm_res * sms && g <= KRY_MAX_GRID) {
                fn = res;
                grid = g;
            }
        }
    }
    const unsigned nthr = fn == (const void*)cg_coop_kernel<T> ? threads : (unsigned)res_bs;
    int nofence = tuning("coop_nofence", 1);
    void* args_res[] = {&n, (void*)&rp, (void*)&ci, (void*)&v, &x, &r, &p, &p2, &q, &c, &part, &hist, &nofence};
    B200SP_CHECK_CUDA(cudaLaunchCooperativeKernel(fn, dim3((unsigned)grid), dim3(nthr),
                                                  fn == (const void*)cg_coop_kernel<T> ? args : args_res, 0,
                                                  as_stream(stream)));
    count_launch();
    return B200SP_OK;
}

template <typename T>
static int bicg_coop(int64_t n, const int32_t* rp, const int32_t* ci, const T* v, T* x, T* r, const T* rt, T* p,
                     T* vv, T* s, T* t, void* ctl, double* part, double* hist, void* stream) {
    if (n >= 1 && n <= TINY_ROWS && tuning("coop_tiny", 1)) {  // one thread, registers only
        KrylovCtl* c = (KrylovCtl*)ctl;
        auto k = n == 1 ? bicg_tiny_kernel<T, 1> : n == 2 ? bicg_tiny_kernel<T, 2>
               : n == 3 ? bicg_tiny_kernel<T, 3> : bicg_tiny_kernel<T, 4>;
        k<<<1, 32, 0, as_stream(stream)>>>(rp, ci, v, x, r, rt, p, vv, s, t, c, hist);
        count_launch();
        return check_launch("bicgstab_tiny");
    }
    int dev = 0, sms = 0, per_sm = 0;
    B200SP_CHECK_CUDA(cudaGetDevice(&dev));
    B200SP_CHECK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    B200SP_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bicg_coop_kernel<T>, KRY_BLOCK, 0));
    int64_t grid = (int64_t)sms * per_sm;
    if (grid > KRY_MAX_GRID) grid = KRY_MAX_GRID;
    const int64_t need = ceil_div(n, KRY_BLOCK);
    if (grid > need) grid = need;
    const int cap = tuning("coop_blocks", 0);
    const unsigned threads = coop_threads(n);
    if (cap > 0 && grid > cap) grid = cap;
    if (grid < 1) grid = 1;
    KrylovCtl* c = (KrylovCtl*)ctl;
    void* args[] = {&n, (void*)&rp, (void*)&ci, (void*)&v, &x, &r, (void*)&rt, &p, &vv, &s, &t, &c, &part, &hist};
    B200SP_CHECK_CUDA(cudaLaunchCooperativeKernel((const void*)bicg_coop_kernel<T>, dim3((unsigned)grid),
                                                  dim3(threads), args, 0, as_stream(stream)));
    count_launch();
    return B200SP_OK;
}

template <typename T>
static int fcg_coop(int64_t n, const int32_t* rp, const int32_t* ci, const T* v, T* x, T* r, T* p, T* q, T* t,
                    void* ctl, double* part, double* hist, void* stream) {
    if (n >= 1 && n <= TINY_ROWS && tuning("coop_tiny", 1)) {  // one thread, registers only
        KrylovCtl* c = (KrylovCtl*)ctl;
        auto k = n == 1 ? fcg_tiny_kernel<T, 1> : n == 2 ? fcg_tiny_kernel<T, 2>
               : n == 3 ? fcg_tiny_kernel<T, 3> : fcg_tiny_kernel<T, 4>;
        k<<<1, 32, 0, as_stream(stream)>>>(rp, ci, v, x, r, p, q, t, c, hist);
        count_launch();
        return check_launch("fcg_tiny");
    }
    int dev = 0, sms = 0, per_sm = 0;
    B200SP_CHECK_CUDA(cudaGetDevice(&dev));
    B200SP_CHECK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    B200SP_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fcg_coop_kernel<T>, KRY_BLOCK, 0));
    int64_t grid = (int64_t)sms * per_sm;
    if (grid > KRY_MAX_GRID) grid = KRY_MAX_GRID;
    const int64_t need = ceil_div(n, KRY_BLOCK);
    if (grid > need) grid = need;
    const int cap = tuning("coop_blocks", 0);
    const unsigned threads = coop_threads(n);
    if (cap > 0 && grid > cap) grid = cap;
    if (grid < 1) grid = 1;
    KrylovCtl* c = (KrylovCtl*)ctl;
    void* args[] = {&n, (void*)&rp, (void*)&ci, (void*)&v, &x, &r, &p, &q, &t, &c, &part, &hist};
    B200SP_CHECK_CUDA(cudaLaunchCooperativeKernel((const void*)fcg_coop_kernel<T>, dim3((unsigned)grid),
                                                  dim3(threads), args, 0, as_stream(stream)));
    count_launch();
    return B200SP_OK;
}

template <typename T>
static int cgs_coop(int64_t n, const int32_t* rp, const int32_t* ci, const T* v, T* x, T* r, const T* rt, T* p, T* q,
                    T* u, T* vh, T* w, T* t, void* ctl, double* part, double* hist, void* stream) {
    if (n >= 1 && n <= TINY_ROWS && tuning("coop_tiny", 1)) {  // one thread, registers only
        KrylovCtl* c = (KrylovCtl*)ctl;
        auto k = n == 1 ? cgs_tiny_kernel<T, 1> : n == 2 ? cgs_tiny_kernel<T, 2>
               : n == 3 ? cgs_tiny_kernel<T, 3> : cgs_tiny_kernel<T, 4>;
        k<<<1, 32, 0, as_stream(stream)>>>(rp, ci, v, x, r, rt, p, q, u, vh, w, t, c, hist);
        count_launch();
        return check_launch("cgs_tiny");
    }
    int dev = 0, sms = 0, per_sm = 0;
    B200SP_CHECK_CUDA(cudaGetDevice(&dev));
    B200SP_CHECK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    B200SP_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cgs_coop_kernel<T>, KRY_BLOCK, 0));
    int64_t grid = (int64_t)sms * per_sm;
    if (grid > KRY_MAX_GRID) grid = KRY_MAX_GRID;
    const int64_t need = ceil_div(n, KRY_BLOCK);
    if (grid > need) grid = need;
    const int cap = tuning("coop_blocks", 0);
    const unsigned threads = coop_threads(n);
    if (cap > 0 && grid > cap) grid = cap;
    if (grid < 1) grid = 1;
    KrylovCtl* c = (KrylovCtl*)ctl;
    void* args[] = {&n, (void*)&rp, (void*)&ci, (void*)&v, &x, &r, (void*)&rt, &p, &q, &u, &vh, &w, &t, &c, &part, &hist};
    B200SP_CHECK_CUDA(cudaLaunchCooperativeKernel((const void*)cgs_coop_kernel<T>, dim3((unsigned)grid),
                                                  dim3(threads), args, 0, as_stream(stream)));
    count_launch();
    return B200SP_OK;
}

extern "C" {
int b200sp_cg_coop_f64(int64_t n, const int32_t* rp, const int32_t* ci, const double* v, double* x, double* r,
                       double* p, double* p2, double* q, void* ctl, double* part, double* hist, void* stream) {
    return cg_coop<double>(n, rp, ci, v, x, r, p, p2, q, ctl, part, hist, stream);
}
int b200sp_cg_coop_f32(int64_t n, const int32_t* rp, const int32_t* ci, const float* v, float* x, float* r,
                       float* p, float* p2, float* q, void* ctl, double* part, double* hist, void* stream) {
    return cg_coop<float>(n, rp, ci, v, x, r, p, p2, q, ctl, part, hist, stream);
}

int b200sp_csr_spmv_dot_f64(int64_t n, const int32_t* rp, const int32_t* ci, const double* v, const double* p,
                            double* q, const double* u, int32_t phase, int32_t subwarp, void* ctl, double* part,
                            void* stream) {
    return csr_spmv_dot<double>(n, rp, ci, v, p, q, u, phase, subwarp, ctl, part, stream);
}
int b200sp_csr_spmv_dot_f32(int64_t n, const int32_t* rp, const int32_t* ci, const float* v, const float* p,
                            float* q, const float* u, int32_t phase, int32_t subwarp, void* ctl, double* part,
                            void* stream) {
    return csr_spmv_dot<float>(n, rp, ci, v, p, q, u, phase, subwarp, ctl, part, stream);
}

int b200sp_cgs_coop_f64(int64_t n, const int32_t* rp, const int32_t* ci, const double* v, double* x, double* r,
                        const double* rt, double* p, double* q, double* u, double* vh, double* w, double* t, void* ctl,
                        double* part, double* hist, void* stream) {
    return cgs_coop<double>(n, rp, ci, v, x, r, rt, p, q, u, vh, w, t, ctl, part, hist, stream);
}
int b200sp_cgs_coop_f32(int64_t n, const int32_t* rp, const int32_t* ci, const float* v, float* x, float* r,
                        const float* rt, float* p, float* q, float* u, float* vh, float* w, float* t, void* ctl,
                        double* part, double* hist, void* stream) {
    return cgs_coop<float>(n, rp, ci, v, x, r, rt, p, q, u, vh, w, t, ctl, part, hist, stream);
}

int b200sp_fcg_coop_f64(int64_t n, const int32_t* rp, const int32_t* ci, const double* v, double* x, double* r,
                        double* p, double* q, double* t, void* ctl, double* part, double* hist, void* stream) {
    return fcg_coop<double>(n, rp, ci, v, x, r, p, q, t, ctl, part, hist, stream);
}
int b200sp_fcg_coop_f32(int64_t n, const int32_t* rp, const int32_t* ci, const float* v, float* x, float* r,
                        float* p, float* q, float* t, void* ctl, double* part, double* hist, void* stream) {
    return fcg_coop<float>(n, rp, ci, v, x, r, p, q, t, ctl, part, hist, stream);
}

int b200sp_bicgstab_coop_f64(int64_t n, const int32_t* rp, const int32_t* ci, const double* v, double* x,
                             double* r, const double* rt, double* p, double* vv, double* s, double* t, void* ctl,
                             double* part, double* hist, void* stream) {
    return bicg_coop<double>(n, rp, ci, v, x, r, rt, p, vv, s, t, ctl, part, hist, stream);
}
int b200sp_bicgstab_coop_f32(int64_t n, const int32_t* rp, const int32_t* ci, const float* v, float* x, float* r,
                             const float* rt, float* p, float* vv, float* s, float* t, void* ctl, double* part,
                             double* hist, void* stream) {
    return bicg_coop<float>(n, rp, ci, v, x, r, rt, p, vv, s, t, ctl, part, hist, stream);
}

int b200sp_cgs_mid(void* ctl, double* hist, void* stream) {
    cgs_mid_kernel<<<1, 32, 0, as_stream(stream)>>>((KrylovCtl*)ctl, hist);
    count_launch();
    return check_launch("cgs_mid");
}

int b200sp_fcg_init_ctl(void* ctl, void* stream) {
    fcg_init_ctl_kernel<<<1, 32, 0, as_stream(stream)>>>((KrylovCtl*)ctl);
    count_launch();
    return check_launch("fcg_init_ctl");
}

int b200sp_cg_finish(void* ctl, double* hist, int32_t phase, void* stream) {
    cg_finish_kernel<<<1, 32, 0, as_stream(stream)>>>((KrylovCtl*)ctl, hist, phase);
    count_launch();
    return check_launch("cg_finish");
}

}  // extern "C"
