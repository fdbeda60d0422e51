// aux.cu -- device workload generator and the exact GPU verifier.
//
//  * 27-point stencil rows (BASELINE configs 2 and 5), position-keyed values;
//    bit-identical twin of paper_2307_14774_b200/workloads.py:stencil27_rows.
//  * power-law rows (config 3) and FEM-like 3x3-block rows (config 4): integer
//    stratified column sampling, so every row range is regenerated exactly by
//    the host twins workloads.py:powerlaw_rows / fem_rows.
//  * csr_exact: csr_reference (kernels.py:233-250) on the GPU -- products in
//    the matrix precision, summed in double-double (~106 bits) per row, so
//    verify_against_oracle (kernels.py:269-317) runs at full BASELINE sizes.
#include <cub/cub.cuh>

#include "common.cuh"

namespace spc5 {
int scan_inclusive_i64(const int64_t *in, int64_t *out, int64_t n, cudaStream_t st);

namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

uint64_t mix64_host(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ int axis_count(int64_t c, int64_t n) {
    return 1 + (c > 0) + (c < n - 1);
}

// n x n x nz grid (nz = n: the cube of configs 2 and 5; nz = n * ranks: the
// weak-scaling box whose z-slabs are the ranks' shards)
__global__ void stencil_count_kernel(int64_t n, int64_t nz, int64_t lo, int64_t rows,
                                     int64_t *counts) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= rows) return;
    const int64_t i = lo + t;
    const int64_t z = i / (n * n), y = (i / n) % n, x = i % n;
    counts[t] = (int64_t)axis_count(z, nz) * axis_count(y, n) * axis_count(x, n);
}

template <typename T>
__global__ void stencil_fill_kernel(int64_t n, int64_t nz, int64_t lo, int64_t rows,
                                    uint64_t seedmix,
                                    double diag, const int64_t *__restrict__ row_ptr,
                                    int32_t *__restrict__ col, T *__restrict__ val) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= rows) return;
    const int64_t i = lo + t;
    const int64_t z = i / (n * n), y = (i / n) % n, x = i % n;
    int64_t k = row_ptr[t];
    for (int dz = -1; dz <= 1; ++dz) {
        if (z + dz < 0 || z + dz >= nz) continue;
        for (int dy = -1; dy <= 1; ++dy) {
            if (y + dy < 0 || y + dy >= n) continue;
            for (int dx = -1; dx <= 1; ++dx) {
                if (x + dx < 0 || x + dx >= n) continue;
                const int64_t j = i + dz * n * n + dy * n + dx;
                double v;
                if (j == i) {
                    v = diag;
                } else {
                    const uint64_t key = ((uint64_t)i << 32) ^ (uint64_t)j ^ seedmix;
                    const double u = (double)(mix64(key) >> 11) * 0x1.0p-53;
                    v = 2.0 * u - 1.0;
                }
                col[k] = (int32_t)j;
                val[k] = (T)v;
                ++k;
            }
        }
    }
}

// ---- config 3: power-law rows ---------------------------------------------
// row i: len = table[hash >> (64 - bits)] (lognormal quantiles, host-made);
// k_loc = (4 len + 2) / 5 columns stratified over the window i +- 4096 and
// k_uni = len - k_loc stratified over [0, n); the two sorted picks are merged
// and duplicates dropped.
constexpr int64_t kPlWindow = 4096;
__device__ __forceinline__ uint64_t pl_key(uint64_t seedmix, int64_t i, int64_t s, int tag) {
    return mix64(seedmix ^ ((uint64_t)i << 24) ^ ((uint64_t)s << 2) ^ (uint64_t)tag);
}
struct PlRow {
    int64_t lo_w, W, k_loc, k_uni, n, i;
    uint64_t seedmix;
    __device__ int64_t loc(int64_t s) const {
        const int64_t a = lo_w + s * W / k_loc, b = lo_w + (s + 1) * W / k_loc;
        return a + (int64_t)(pl_key(seedmix, i, s, 1) % (uint64_t)(b - a));
    }
    __device__ int64_t uni(int64_t s) const {
        const int64_t a = s * n / k_uni, b = (s + 1) * n / k_uni;
        return a + (int64_t)(pl_key(seedmix, i, s, 2) % (uint64_t)(b - a));
    }
};
__device__ PlRow pl_row(int64_t n, int64_t i, uint64_t seedmix, const int32_t *table, int bits) {
    PlRow r;
    r.n = n;
    r.i = i;
    r.seedmix = seedmix;
    const int64_t len = table[pl_key(seedmix, i, 0, 0) >> (64 - bits)];
    r.lo_w = max((int64_t)0, i - kPlWindow);
    const int64_t hi_w = min(n - 1, i + kPlWindow);
    r.W = hi_w - r.lo_w + 1;
    r.k_loc = min((4 * len + 2) / 5, r.W);
    r.k_uni = min(len - r.k_loc, n);
    return r;
}
// merge the two sorted pick sequences; emit(col) per distinct column
template <typename F>
__device__ void pl_merge(const PlRow &r, F emit) {
    int64_t a = 0, b = 0, last = -1;
    int64_t ca = r.k_loc ? r.loc(0) : INT64_MAX, cb = r.k_uni ? r.uni(0) : INT64_MAX;
    while (a < r.k_loc || b < r.k_uni) {
        int64_t c;
        if (ca <= cb) {
            c = ca;
            ++a;
            ca = a < r.k_loc ? r.loc(a) : INT64_MAX;
        } else {
            c = cb;
            ++b;
            cb = b < r.k_uni ? r.uni(b) : INT64_MAX;
        }
        if (c != last) {
            emit(c);
            last = c;
        }
    }
}
__global__ void powerlaw_count_kernel(int64_t n, int64_t lo, int64_t rows, uint64_t seedmix,
                                      const int32_t *__restrict__ table, int bits,
                                      int64_t *counts) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= rows) return;
    const PlRow r = pl_row(n, lo + t, seedmix, table, bits);
    int64_t c = 0;
    pl_merge(r, [&](int64_t) { ++c; });
    counts[t] = c;
}
template <typename T>
__global__ void powerlaw_fill_kernel(int64_t n, int64_t lo, int64_t rows, uint64_t seedmix,
                                     uint64_t valmix, const int32_t *__restrict__ table, int bits,
                                     const int64_t *__restrict__ row_ptr, int32_t *__restrict__ col,
                                     T *__restrict__ val) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= rows) return;
    const int64_t i = lo + t;
    const PlRow r = pl_row(n, i, seedmix, table, bits);
    int64_t k = row_ptr[t];
    pl_merge(r, [&](int64_t j) {
        const uint64_t key = ((uint64_t)i << 32) ^ (uint64_t)j ^ valmix;
        const double u = (double)(mix64(key) >> 11) * 0x1.0p-53;
        col[k] = (int32_t)j;
        val[k] = (T)(2.0 * u - 1.0);
        ++k;
    });
}

// ---- config 4: FEM-like rows ----------------------------------------------
// node q couples to itself and 26 nodes stratified over q +- 2048 (self
// excluded); row 3q+d holds the dense 3x3 blocks of those 27 nodes, values
// N(0,1) approximated by sqrt(3) * (u1 + u2 + u3 + u4 - 2) (Irwin-Hall 4).
constexpr int64_t kFemWindow = 2048;
constexpr int kFemNbr = 26;
__device__ __forceinline__ int64_t fem_nbr(int64_t nodes, int64_t q, int s, uint64_t seedmix) {
    const int64_t lo_w = max((int64_t)0, q - kFemWindow);
    const int64_t W = min(nodes - 1, q + kFemWindow) - lo_w;  // positions without q
    const int64_t a = s * W / kFemNbr, b = (s + 1) * W / kFemNbr;
    const int64_t p = lo_w + a + (int64_t)(pl_key(seedmix, q, s, 3) % (uint64_t)(b - a));
    return p >= q ? p + 1 : p;
}
__global__ void fem_count_kernel(int64_t lo, int64_t rows, int64_t *counts) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < rows) counts[t] = 3 * (kFemNbr + 1);
}
template <typename T>
__global__ void fem_fill_kernel(int64_t nodes, int64_t lo, int64_t rows, uint64_t seedmix,
                                uint64_t valmix, const int64_t *__restrict__ row_ptr,
                                int32_t *__restrict__ col, T *__restrict__ val) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= rows) return;
    const int64_t i = lo + t, q = i / 3;
    int64_t k = row_ptr[t];
    auto emit_node = [&](int64_t j) {
        for (int d = 0; d < 3; ++d) {
            const int64_t c = 3 * j + d;
            uint64_t h = mix64(((uint64_t)i << 32) ^ (uint64_t)c ^ valmix);
            double acc = 0.0;
            for (int m = 0; m < 4; ++m) {
                acc += (double)(h >> 11) * 0x1.0p-53;
                h = mix64(h + 0x9E3779B97F4A7C15ull);
            }
            col[k] = (int32_t)c;
            val[k] = (T)((acc - 2.0) * 1.7320508075688772);
            ++k;
        }
    };
    bool self_done = false;
    for (int s = 0; s < kFemNbr; ++s) {
        const int64_t nb = fem_nbr(nodes, q, s, seedmix);
        if (!self_done && q < nb) {
            emit_node(q);
            self_done = true;
        }
        emit_node(nb);
    }
    if (!self_done) emit_node(q);
}

__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }

struct DD {
    double hi, lo;
};

__device__ __forceinline__ DD dd_add(DD a, double b) {
    const double s = a.hi + b;
    const double bb = s - a.hi;
    const double err = (a.hi - (s - bb)) + (b - bb);
    const double lo = a.lo + err;
    const double hi = s + lo;
    return DD{hi, lo - (hi - s)};
}

__device__ __forceinline__ DD dd_add(DD a, DD b) {
    DD s = dd_add(a, b.hi);
    return dd_add(s, b.lo);
}

template <typename T>
__global__ void csr_exact_kernel(int64_t num_rows, const int64_t *__restrict__ rp,
                                 const int32_t *__restrict__ ci, const T *__restrict__ v,
                                 const T *__restrict__ x, double *y, double *a) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = warp; i < num_rows; i += nwarps) {
        DD s{0.0, 0.0}, sa{0.0, 0.0};
        for (int64_t k = rp[i] + lane; k < rp[i + 1]; k += 32) {
            const T p = mul_rn(v[k], x[ci[k]]);  // rounded product, never contracted
            s = dd_add(s, (double)p);
            sa = dd_add(sa, (double)(p < T(0) ? -p : p));
        }
#pragma unroll
        for (int d = 16; d >= 1; d >>= 1) {
            DD o{__shfl_xor_sync(0xffffffffu, s.hi, d), __shfl_xor_sync(0xffffffffu, s.lo, d)};
            DD oa{__shfl_xor_sync(0xffffffffu, sa.hi, d), __shfl_xor_sync(0xffffffffu, sa.lo, d)};
            s = dd_add(s, o);
            sa = dd_add(sa, oa);
        }
        if (lane == 0) {
            y[i] = s.hi + s.lo;
            a[i] = sa.hi + sa.lo;
        }
    }
}

}  // namespace

int gen_stencil27_rowptr(int64_t n, int64_t nz, int64_t lo, int64_t hi, int64_t *rp,
                         cudaStream_t st) {
    if (n < 1 || nz < 1 || lo < 0 || hi < lo || hi > n * n * nz || n * n * nz > (1ll << 31))
        return fail(SPC5_EINVAL, "stencil27: bad n / nz / row range");
    const int64_t rows = hi - lo;
    SPC5_CUDA(cudaMemsetAsync(rp, 0, sizeof(int64_t), st));
    if (!rows) return SPC5_OK;
    int64_t *counts = nullptr;
    SPC5_TRY(dev_alloc(&counts, (size_t)rows));
    stencil_count_kernel<<<(unsigned)cdiv(rows, 256), 256, 0, st>>>(n, nz, lo, rows, counts);
    SPC5_CUDA(cudaGetLastError());
    SPC5_TRY(scan_inclusive_i64(counts, rp + 1, rows, st));
    SPC5_CUDA(cudaStreamSynchronize(st));
    dev_free(counts);
    return SPC5_OK;
}

int gen_stencil27_fill(int64_t n, int64_t nz, int64_t lo, int64_t hi, int precision,
                       uint64_t seed, double diag, const int64_t *rp, int32_t *ci, void *v,
                       cudaStream_t st) {
    const int64_t rows = hi - lo;
    if (rows <= 0) return SPC5_OK;
    const uint64_t seedmix = mix64_host(seed + 0x9E3779B97F4A7C15ull);
    const unsigned grid = (unsigned)cdiv(rows, 256);
    if (precision == SPC5_F64)
        stencil_fill_kernel<double><<<grid, 256, 0, st>>>(n, nz, lo, rows, seedmix, diag, rp, ci,
                                                          static_cast<double *>(v));
    else
        stencil_fill_kernel<float><<<grid, 256, 0, st>>>(n, nz, lo, rows, seedmix, diag, rp, ci,
                                                         static_cast<float *>(v));
    SPC5_CUDA(cudaGetLastError());
    return SPC5_OK;
}

// ---- config 3/4 host entry points ------------------------------------------
namespace {
int gen_rowptr_from_counts(int64_t rows, int64_t *counts, int64_t *rp, cudaStream_t st) {
    SPC5_TRY(scan_inclusive_i64(counts, rp + 1, rows, st));
    SPC5_CUDA(cudaStreamSynchronize(st));
    dev_free(counts);
    return SPC5_OK;
}
}  // namespace

int gen_powerlaw_rowptr(int64_t n, int64_t lo, int64_t hi, uint64_t seed, const int32_t *table,
                        int bits, int64_t *rp, cudaStream_t st) {
    if (n < 1 || n > INT32_MAX || lo < 0 || hi < lo || hi > n || bits < 1 || bits > 24)
        return fail(SPC5_EINVAL, "powerlaw: bad n / row range / table");
    const int64_t rows = hi - lo;
    SPC5_CUDA(cudaMemsetAsync(rp, 0, sizeof(int64_t), st));
    if (!rows) return SPC5_OK;
    int64_t *counts = nullptr;
    SPC5_TRY(dev_alloc(&counts, (size_t)rows));
    powerlaw_count_kernel<<<(unsigned)cdiv(rows, 256), 256, 0, st>>>(
        n, lo, rows, mix64_host(seed + 0x9E3779B97F4A7C15ull) ^ 0x5bd1e995ull, table, bits,
        counts);
    SPC5_CUDA(cudaGetLastError());
    return gen_rowptr_from_counts(rows, counts, rp, st);
}

int gen_powerlaw_fill(int64_t n, int64_t lo, int64_t hi, int precision, uint64_t seed,
                      const int32_t *table, int bits, const int64_t *rp, int32_t *ci, void *v,
                      cudaStream_t st) {
    const int64_t rows = hi - lo;
    if (rows <= 0) return SPC5_OK;
    const uint64_t seedmix = mix64_host(seed + 0x9E3779B97F4A7C15ull) ^ 0x5bd1e995ull;
    const uint64_t valmix = mix64_host(seed + 0x9E3779B97F4A7C15ull);
    const unsigned grid = (unsigned)cdiv(rows, 128);
    if (precision == SPC5_F64)
        powerlaw_fill_kernel<double><<<grid, 128, 0, st>>>(n, lo, rows, seedmix, valmix, table,
                                                           bits, rp, ci, static_cast<double *>(v));
    else
        powerlaw_fill_kernel<float><<<grid, 128, 0, st>>>(n, lo, rows, seedmix, valmix, table,
                                                          bits, rp, ci, static_cast<float *>(v));
    SPC5_CUDA(cudaGetLastError());
    return SPC5_OK;
}

int gen_fem_rowptr(int64_t nodes, int64_t lo, int64_t hi, int64_t *rp, cudaStream_t st) {
    if (nodes < 2 * kFemWindow || 3 * nodes > INT32_MAX || lo < 0 || hi < lo || hi > 3 * nodes)
        return fail(SPC5_EINVAL, "fem: bad node count / row range");
    const int64_t rows = hi - lo;
    SPC5_CUDA(cudaMemsetAsync(rp, 0, sizeof(int64_t), st));
    if (!rows) return SPC5_OK;
    int64_t *counts = nullptr;
    SPC5_TRY(dev_alloc(&counts, (size_t)rows));
    fem_count_kernel<<<(unsigned)cdiv(rows, 256), 256, 0, st>>>(lo, rows, counts);
    SPC5_CUDA(cudaGetLastError());
    return gen_rowptr_from_counts(rows, counts, rp, st);
}

int gen_fem_fill(int64_t nodes, int64_t lo, int64_t hi, int precision, uint64_t seed,
                 const int64_t *rp, int32_t *ci, void *v, cudaStream_t st) {
    const int64_t rows = hi - lo;
    if (rows <= 0) return SPC5_OK;
    const uint64_t seedmix = mix64_host(seed + 0x9E3779B97F4A7C15ull) ^ 0x5bd1e995ull;
    const uint64_t valmix = mix64_host(seed + 0x9E3779B97F4A7C15ull);
    const unsigned grid = (unsigned)cdiv(rows, 128);
    if (precision == SPC5_F64)
        fem_fill_kernel<double><<<grid, 128, 0, st>>>(nodes, lo, rows, seedmix, valmix, rp, ci,
                                                      static_cast<double *>(v));
    else
        fem_fill_kernel<float><<<grid, 128, 0, st>>>(nodes, lo, rows, seedmix, valmix, rp, ci,
                                                     static_cast<float *>(v));
    SPC5_CUDA(cudaGetLastError());
    return SPC5_OK;
}

int csr_exact(int64_t num_rows, int precision, const int64_t *rp, const int32_t *ci,
              const void *v, const void *x, double *y, double *a, cudaStream_t st) {
    if (num_rows <= 0) return SPC5_OK;
    const unsigned grid = (unsigned)std::min<int64_t>(cdiv(num_rows, 8), 148 * 64);
    if (precision == SPC5_F64)
        csr_exact_kernel<double><<<grid, 256, 0, st>>>(num_rows, rp, ci,
                                                       static_cast<const double *>(v),
                                                       static_cast<const double *>(x), y, a);
    else
        csr_exact_kernel<float><<<grid, 256, 0, st>>>(num_rows, rp, ci,
                                                      static_cast<const float *>(v),
                                                      static_cast<const float *>(x), y, a);
    SPC5_CUDA(cudaGetLastError());
    return SPC5_OK;
}

}  // namespace spc5
