// Device-side generators for the benchmark systems (Csr, canonical order).
//
// The reference assembles its test systems with Python loops into host
// MatrixData (src/problems.py:11-45); at C2/C5 sizes (56M / 938M entries) that
// is a 1.3-22.5 GB host detour, so the systems are generated in place on the
// device. oracle/problems.py restates every generator in NumPy and the CPU
// tests pin it against the reference's own five_point_poisson /
// convection_diffusion (tests/golden).
//
// Stencils (grid index idx = (i*g + j)*g + k, Dirichlet truncation; the 3-D
// kinds take nz planes along i -- nz = g is the cube, nz = N g the weak-scaled
// slab stack of the multi-GPU benchmark):
//   kind 0: 2-D 5-point,  g x g,   centre 4, neighbours -1  (== five_point_poisson)
//   kind 1: 3-D 7-point,  g^3,     centre 6, neighbours -1
//   kind 2: 3-D 27-point, g^3,     centre 26, neighbours -1
//   kind 3: 3-D 7-point convection-diffusion, centre 6, neighbour at offset
//           s = -1 / +1 along any axis: -1 - c / -1 + c (3-D extension of
//           convection_diffusion, src/problems.py:42-45)
// Power law: row length L_i = max{k : u_i <= t_k} with thresholds
//   t_k = (c/k)^1.5 supplied by the host (so host and device agree bitwise),
//   u_i = 1 - U(hash(seed, 0, i)); columns stratified: entry k of row i lies in
//   [floor(k n / L), floor((k+1) n / L)), offset by a hash; values U(-1, 1).
#include "common.cuh"

namespace b200sp {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
// hash(seed, a, b) -- restated in oracle/problems.py::_hash
__device__ __forceinline__ uint64_t hash3(uint64_t seed, uint64_t a, uint64_t b) {
    return mix64(mix64(mix64(seed) ^ (a * 0xD1B54A32D192ED03ull)) + b);
}
__device__ __forceinline__ double unit(uint64_t h) { return (double)(h >> 11) * 0x1.0p-53; }

struct Stencil {
    int kind;
    int64_t g;
    int64_t nz;  // planes along the slowest axis i (3-D kinds; nz = g is the cube)
    double conv;
    int64_t row0;
};

__device__ __forceinline__ int stencil_len(const Stencil& s, int64_t row) {
    if (s.kind == 0) {
        const int64_t i = row / s.g, j = row % s.g;
        return 1 + (i > 0) + (i < s.g - 1) + (j > 0) + (j < s.g - 1);
    }
    const int64_t g = s.g;
    const int64_t i = row / (g * g), j = (row / g) % g, k = row % g;
    if (s.kind == 2) {
        const int ni = 1 + (i > 0) + (i < s.nz - 1), nj = 1 + (j > 0) + (j < g - 1), nk = 1 + (k > 0) + (k < g - 1);
        return ni * nj * nk;
    }
    return 1 + (i > 0) + (i < s.nz - 1) + (j > 0) + (j < g - 1) + (k > 0) + (k < g - 1);
}

// n = rows generated, starting at global row s.row0 (row-partitioned solves
// generate only their own rows, with global column indices)
__global__ void stencil_lengths_kernel(Stencil s, int64_t n, int* __restrict__ len) {
    for (int64_t lr = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; lr < n; lr += (int64_t)gridDim.x * blockDim.x)
        len[lr] = stencil_len(s, s.row0 + lr);
}

template <typename T>
__global__ void stencil_fill_kernel(Stencil s, int64_t n, const int* __restrict__ rp, int* __restrict__ ci,
                                    T* __restrict__ v) {
    for (int64_t lr = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; lr < n; lr += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = s.row0 + lr;
        int64_t o = rp[lr];
        const int64_t g = s.g;
        if (s.kind == 0) {
            const int64_t i = r / g, j = r % g;
            // canonical column order: (i-1,j) (i,j-1) (i,j) (i,j+1) (i+1,j)
            if (i > 0) { ci[o] = (int)(r - g); v[o] = T(-1); ++o; }
            if (j > 0) { ci[o] = (int)(r - 1); v[o] = T(-1); ++o; }
            ci[o] = (int)r; v[o] = T(4); ++o;
            if (j < g - 1) { ci[o] = (int)(r + 1); v[o] = T(-1); ++o; }
            if (i < g - 1) { ci[o] = (int)(r + g); v[o] = T(-1); ++o; }
            continue;
        }
        const int64_t i = r / (g * g), j = (r / g) % g, k = r % g;
        if (s.kind == 2) {
            for (int di = -1; di <= 1; ++di) {
                if (i + di < 0 || i + di >= s.nz) continue;
                for (int dj = -1; dj <= 1; ++dj) {
                    if (j + dj < 0 || j + dj >= g) continue;
                    for (int dk = -1; dk <= 1; ++dk) {
                        if (k + dk < 0 || k + dk >= g) continue;
                        const bool centre = di == 0 && dj == 0 && dk == 0;
                        ci[o] = (int)(r + (di * g + dj) * g + dk);
                        v[o] = centre ? T(26) : T(-1);
                        ++o;
                    }
                }
            }
            continue;
        }
        // 7-point, canonical order: -g^2, -g, -1, centre, +1, +g, +g^2
        const double lo = s.kind == 3 ? -1.0 - s.conv : -1.0;  // offset s = -1
        const double hi = s.kind == 3 ? -1.0 + s.conv : -1.0;  // offset s = +1
        if (i > 0) { ci[o] = (int)(r - g * g); v[o] = T(lo); ++o; }
        if (j > 0) { ci[o] = (int)(r - g); v[o] = T(lo); ++o; }
        if (k > 0) { ci[o] = (int)(r - 1); v[o] = T(lo); ++o; }
        ci[o] = (int)r; v[o] = T(6); ++o;
        if (k < g - 1) { ci[o] = (int)(r + 1); v[o] = T(hi); ++o; }
        if (j < g - 1) { ci[o] = (int)(r + g); v[o] = T(hi); ++o; }
        if (i < s.nz - 1) { ci[o] = (int)(r + g * g); v[o] = T(hi); ++o; }
    }
}

// thresholds t[0..max_len-1] = t_1..t_max, non-increasing
__global__ void powerlaw_lengths_kernel(int64_t n, uint64_t seed, const double* __restrict__ t, int max_len,
                                        int* __restrict__ len) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        const double u = 1.0 - unit(hash3(seed, 0, (uint64_t)r));
        // count of k with t_k >= u (t non-increasing)
        int lo = 0, hi = max_len;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (t[mid] >= u) lo = mid + 1;
            else hi = mid;
        }
        int L = lo < 1 ? 1 : lo;
        if (L > n) L = (int)n;
        len[r] = L;
    }
}

template <typename T>
__global__ void powerlaw_fill_kernel(int64_t n, uint64_t seed, const int* __restrict__ rp, int* __restrict__ ci,
                                     T* __restrict__ v) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = rp[r];
        const int64_t L = rp[r + 1] - s;
        for (int64_t k = 0; k < L; ++k) {
            const int64_t lo = k * n / L, hi = (k + 1) * n / L;
            const uint64_t h = hash3(seed, (uint64_t)r + 1, (uint64_t)k);
            ci[s + k] = (int)(lo + (int64_t)(h % (uint64_t)(hi - lo)));
            v[s + k] = T(2.0 * unit(mix64(h ^ 0x5851F42D4C957F2Dull)) - 1.0);
        }
    }
}

}  // namespace b200sp

using namespace b200sp;

extern "C" {

int b200sp_stencil_lengths(int32_t kind, int64_t g, int64_t nz, int64_t row0, int64_t n, int32_t* len, void* stream) {
    B200SP_REQUIRE(kind >= 0 && kind <= 3, B200SP_EINVAL, "stencil: unknown kind %d", kind);
    B200SP_REQUIRE(nz >= 1, B200SP_EINVAL, "stencil: nz must be positive");
    if (n == 0) return B200SP_OK;
    stencil_lengths_kernel<<<grid_for(n, 256, 8), 256, 0, as_stream(stream)>>>(Stencil{kind, g, nz, 0.0, row0}, n, len);
    count_launch();
    return check_launch("stencil_lengths");
}

int b200sp_stencil_fill_f64(int32_t kind, int64_t g, int64_t nz, double conv, int64_t row0, int64_t n, const int32_t* rp,
                            int32_t* ci, double* v, void* stream) {
    if (n == 0) return B200SP_OK;
    stencil_fill_kernel<double><<<grid_for(n, 256, 8), 256, 0, as_stream(stream)>>>(Stencil{kind, g, nz, conv, row0}, n, rp, ci, v);
    count_launch();
    return check_launch("stencil_fill");
}
int b200sp_stencil_fill_f32(int32_t kind, int64_t g, int64_t nz, double conv, int64_t row0, int64_t n, const int32_t* rp,
                            int32_t* ci, float* v, void* stream) {
    if (n == 0) return B200SP_OK;
    stencil_fill_kernel<float><<<grid_for(n, 256, 8), 256, 0, as_stream(stream)>>>(Stencil{kind, g, nz, conv, row0}, n, rp, ci, v);
    count_launch();
    return check_launch("stencil_fill");
}

int b200sp_powerlaw_lengths(int64_t n, uint64_t seed, const double* thresholds, int32_t max_len, int32_t* len,
                            void* stream) {
    if (n == 0) return B200SP_OK;
    powerlaw_lengths_kernel<<<grid_for(n, 256, 8), 256, 0, as_stream(stream)>>>(n, seed, thresholds, max_len, len);
    count_launch();
    return check_launch("powerlaw_lengths");
}

int b200sp_powerlaw_fill_f64(int64_t n, uint64_t seed, const int32_t* rp, int32_t* ci, double* v, void* stream) {
    if (n == 0) return B200SP_OK;
    powerlaw_fill_kernel<double><<<grid_for(n, 256, 8), 256, 0, as_stream(stream)>>>(n, seed, rp, ci, v);
    count_launch();
    return check_launch("powerlaw_fill");
}
int b200sp_powerlaw_fill_f32(int64_t n, uint64_t seed, const int32_t* rp, int32_t* ci, float* v, void* stream) {
    if (n == 0) return B200SP_OK;
    powerlaw_fill_kernel<float><<<grid_for(n, 256, 8), 256, 0, as_stream(stream)>>>(n, seed, rp, ci, v);
    count_launch();
    return check_launch("powerlaw_fill");
}

}  // extern "C"
