// aux.cu -- device workload generator and the exact GPU verifier.
//
//  * 27-point stencil rows (BASELINE configs 2 and 5), position-keyed values;
//    bit-identical twin of paper_2307_14774_b200/workloads.py:stencil27_rows.
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

__global__ void stencil_count_kernel(int64_t n, int64_t lo, int64_t rows, int64_t *counts) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= rows) return;
    const int64_t i = lo + t;
    const int64_t z = i / (n * n), y = (i / n) % n, x = i % n;
    counts[t] = (int64_t)axis_count(z, n) * axis_count(y, n) * axis_count(x, n);
}

template <typename T>
__global__ void stencil_fill_kernel(int64_t n, int64_t lo, int64_t rows, uint64_t seedmix,
                                    double diag, const int64_t *__restrict__ row_ptr,
                                    int32_t *__restrict__ col, T *__restrict__ val) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= rows) return;
    const int64_t i = lo + t;
    const int64_t z = i / (n * n), y = (i / n) % n, x = i % n;
    int64_t k = row_ptr[t];
    for (int dz = -1; dz <= 1; ++dz) {
        if (z + dz < 0 || z + dz >= n) continue;
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

int gen_stencil27_rowptr(int64_t n, int64_t lo, int64_t hi, int64_t *rp, cudaStream_t st) {
    if (n < 1 || lo < 0 || hi < lo || hi > n * n * n)
        return fail(SPC5_EINVAL, "stencil27: bad n / row range");
    const int64_t rows = hi - lo;
    SPC5_CUDA(cudaMemsetAsync(rp, 0, sizeof(int64_t), st));
    if (!rows) return SPC5_OK;
    int64_t *counts = nullptr;
    SPC5_TRY(dev_alloc(&counts, (size_t)rows));
    stencil_count_kernel<<<(unsigned)cdiv(rows, 256), 256, 0, st>>>(n, lo, rows, counts);
    SPC5_CUDA(cudaGetLastError());
    SPC5_TRY(scan_inclusive_i64(counts, rp + 1, rows, st));
    SPC5_CUDA(cudaStreamSynchronize(st));
    dev_free(counts);
    return SPC5_OK;
}

int gen_stencil27_fill(int64_t n, int64_t lo, int64_t hi, int precision, uint64_t seed,
                       double diag, const int64_t *rp, int32_t *ci, void *v, cudaStream_t st) {
    const int64_t rows = hi - lo;
    if (rows <= 0) return SPC5_OK;
    const uint64_t seedmix = mix64_host(seed + 0x9E3779B97F4A7C15ull);
    const unsigned grid = (unsigned)cdiv(rows, 256);
    if (precision == SPC5_F64)
        stencil_fill_kernel<double><<<grid, 256, 0, st>>>(n, lo, rows, seedmix, diag, rp, ci,
                                                          static_cast<double *>(v));
    else
        stencil_fill_kernel<float><<<grid, 256, 0, st>>>(n, lo, rows, seedmix, diag, rp, ci,
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
