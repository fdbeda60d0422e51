// convert.cu -- K1: CSR -> SPC5 beta(r,vs) conversion on the GPU, and the
// inverse spc5_to_csr.
//
// Bit-exact contract: csr_to_spc5, /root/reference/pkg/src/spc5/blocks.py:96-143
// (SURVEY.md Appendix A).  The reference builds keys panel<<32|col, takes
// np.unique and walks them with a greedy span (blocks.py:114-123).  Here a
// panel is owned by a group of r lanes (lane rr holds a cursor into row rr of
// the panel); one step of the greedy chain is
//     anchor = min over the group of the next unconsumed column  (shfl_xor)
//     every lane consumes its columns <= anchor + vs - 1, OR-ing 1<<(c-anchor)
// which visits the sorted union U_p in order without materialising it.
// Values are written in slot order (block, row-in-panel, column) with a
// group prefix sum of per-row counts -- the stable argsort of blocks.py:136-137.
// For r = 1 that order is the CSR order, so values are one D2D copy.
#include <cub/cub.cuh>

#include "common.cuh"

namespace spc5 {
namespace {

// ---------------------------------------------------------------- validation
// CsrMatrix contract (mmio.py:84-100 / SPEC.md:35-38): row_ptr non-decreasing
// from 0 to nnz, columns strictly increasing per row and inside [0, num_cols).
__global__ void csr_check_kernel(int64_t num_rows, int64_t num_cols, int64_t nnz,
                                 const int64_t *__restrict__ row_ptr,
                                 const int32_t *__restrict__ col_idx, int *err) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = warp; i < num_rows; i += nwarps) {
        const int64_t s = row_ptr[i], e = row_ptr[i + 1];
        int bad = 0;
        if (i == 0 && s != 0) bad = 1;
        if (i == num_rows - 1 && e != nnz) bad = 1;
        if (e < s || s < 0 || e > nnz) bad = 1;
        if (!bad) {
            for (int64_t k = s + lane; k < e; k += 32) {
                const int32_t c = col_idx[k];
                if (c < 0 || (int64_t)c >= num_cols) bad = 1;
                if (k > s && c <= col_idx[k - 1]) bad = 1;
            }
        }
        if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(err, 1);
    }
}

struct ConvArgs {
    int64_t num_rows, num_panels;
    const int64_t *row_ptr;
    const int32_t *col_idx;
    const void *vin;
    int vs, vsize;
    int64_t *panel_blocks;  // count pass
    const int64_t *rowptr;  // write pass: first block of each panel
    uint32_t *colidx;
    void *masks;
    void *vout;
};

// One group of R lanes per panel; R divides 32 so groups never straddle warps.
template <int R, bool WRITE>
__global__ void __launch_bounds__(256) convert_kernel(ConvArgs a) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const int64_t p = t / R;
    const int rr = (int)(t % R);
    if (p >= a.num_panels) return;  // whole groups leave together
    const unsigned gmask = (R == 1) ? (1u << lane) : (((1u << R) - 1u) << (lane & ~(R - 1)));
    const int64_t row = p * R + rr;
    int64_t cur = 0, end = 0;
    if (row < a.num_rows) {
        cur = a.row_ptr[row];
        end = a.row_ptr[row + 1];
    }
    const int64_t row0 = p * R < a.num_rows ? p * R : a.num_rows;
    int64_t bpos = WRITE ? a.rowptr[p] : 0;
    int64_t vpos = WRITE ? a.row_ptr[row0] : 0;
    int64_t nblk = 0;
    const uint32_t kSent = 0xffffffffu;
    const int span = a.vs - 1;
    for (;;) {
        uint32_t anchor = cur < end ? (uint32_t)__ldg(a.col_idx + cur) : kSent;
#pragma unroll
        for (int d = 1; d < R; d <<= 1) anchor = min(anchor, __shfl_xor_sync(gmask, anchor, d));
        if (anchor == kSent) break;
        const uint32_t limit = anchor + (uint32_t)span;
        uint32_t m = 0;
        const int64_t s = cur;
        while (cur < end) {
            const uint32_t c = (uint32_t)__ldg(a.col_idx + cur);
            if (c > limit) break;
            m |= 1u << (c - anchor);
            ++cur;
        }
        if (WRITE) {
            if (rr == 0) a.colidx[bpos] = anchor;
            if (a.vs <= 8) ((uint8_t *)a.masks)[bpos * R + rr] = (uint8_t)m;
            else ((uint16_t *)a.masks)[bpos * R + rr] = (uint16_t)m;
            if (R > 1) {
                const int n = (int)(cur - s);
                int incl = n;
#pragma unroll
                for (int d = 1; d < R; d <<= 1) {
                    const int v = __shfl_up_sync(gmask, incl, d, R);
                    if (rr >= d) incl += v;
                }
                const int total = __shfl_sync(gmask, incl, R - 1, R);
                const int64_t dst = vpos + incl - n;
                if (a.vsize == 8) {
                    const double *src = (const double *)a.vin + s;
                    double *out = (double *)a.vout + dst;
                    for (int j = 0; j < n; ++j) out[j] = src[j];
                } else {
                    const float *src = (const float *)a.vin + s;
                    float *out = (float *)a.vout + dst;
                    for (int j = 0; j < n; ++j) out[j] = src[j];
                }
                vpos += total;
            }
            ++bpos;
        }
        ++nblk;
    }
    if (!WRITE && rr == 0) a.panel_blocks[p] = nblk;
}

template <bool WRITE>
void launch_convert(int r, const ConvArgs &a, cudaStream_t st) {
    const int64_t threads = a.num_panels * r;
    const unsigned grid = (unsigned)cdiv(threads, 256);
    switch (r) {
        case 1: convert_kernel<1, WRITE><<<grid, 256, 0, st>>>(a); break;
        case 2: convert_kernel<2, WRITE><<<grid, 256, 0, st>>>(a); break;
        case 4: convert_kernel<4, WRITE><<<grid, 256, 0, st>>>(a); break;
        default: convert_kernel<8, WRITE><<<grid, 256, 0, st>>>(a); break;
    }
}

// ---------------------------------------------------------------- to CSR
// blocks.py:146-168: one thread per (panel, row-in-panel) walks the panel's
// blocks; destination = CSR order (blocks ascend, so columns ascend).
__global__ void row_counts_kernel(int64_t num_rows, int64_t num_panels, int r, int vs,
                                  const int64_t *__restrict__ rowptr,
                                  const void *__restrict__ masks, int64_t *counts) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t p = t / r;
    const int rr = (int)(t % r);
    if (p >= num_panels) return;
    const int64_t row = p * r + rr;
    if (row >= num_rows) return;
    int64_t c = 0;
    for (int64_t b = rowptr[p]; b < rowptr[p + 1]; ++b) c += __popc(load_mask(masks, b * r + rr, vs));
    counts[row] = c;
}

__global__ void to_csr_kernel(int64_t num_rows, int64_t num_panels, int r, int vs, int vsize,
                              const int64_t *__restrict__ rowptr,
                              const uint32_t *__restrict__ colidx,
                              const void *__restrict__ masks, const void *__restrict__ vals,
                              const int64_t *__restrict__ voff,
                              const int64_t *__restrict__ row_ptr, int32_t *col_out,
                              void *val_out) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t p = t / r;
    const int rr = (int)(t % r);
    if (p >= num_panels) return;
    const int64_t row = p * r + rr;
    if (row >= num_rows) return;
    int64_t dst = row_ptr[row];
    for (int64_t b = rowptr[p]; b < rowptr[p + 1]; ++b) {
        int64_t src = voff[b];
        for (int q = 0; q < rr; ++q) src += __popc(load_mask(masks, b * r + q, vs));
        uint32_t m = load_mask(masks, b * r + rr, vs);
        const int64_t anchor = colidx[b];
        while (m) {
            const int k = __ffs(m) - 1;
            m &= m - 1;
            col_out[dst] = (int32_t)(anchor + k);
            if (vsize == 8) ((double *)val_out)[dst] = ((const double *)vals)[src];
            else ((float *)val_out)[dst] = ((const float *)vals)[src];
            ++src;
            ++dst;
        }
    }
}

template <typename T>
int inclusive_scan(const T *in, T *out, int64_t n, cudaStream_t st) {
    if (n <= 0) return SPC5_OK;
    size_t bytes = 0;
    SPC5_CUDA(cub::DeviceScan::InclusiveSum(nullptr, bytes, in, out, n, st));
    void *tmp = nullptr;
    SPC5_TRY(dev_alloc(&tmp, bytes));
    cudaError_t e = cub::DeviceScan::InclusiveSum(tmp, bytes, in, out, n, st);
    dev_free(tmp);
    if (e != cudaSuccess) return cuda_fail(e, "cub::DeviceScan::InclusiveSum");
    return SPC5_OK;
}

}  // namespace

int scan_inclusive_i64(const int64_t *in, int64_t *out, int64_t n, cudaStream_t st) {
    return inclusive_scan<int64_t>(in, out, n, st);
}

int convert_csr(Matrix &m, const int64_t *d_row_ptr, const int32_t *d_col_idx,
                const void *d_values, cudaStream_t st) {
    const int64_t np = m.num_panels;
    SPC5_TRY(dev_alloc(&m.rowptr, (size_t)np + 1));
    SPC5_CUDA(cudaMemsetAsync(m.rowptr, 0, sizeof(int64_t) * (np + 1), st));
    if (m.num_rows > 0) {
        int *err = nullptr;
        SPC5_TRY(dev_alloc(&err, 1));
        SPC5_CUDA(cudaMemsetAsync(err, 0, sizeof(int), st));
        const unsigned grid = (unsigned)std::min<int64_t>(cdiv(m.num_rows, 8), 148 * 64);
        csr_check_kernel<<<grid, 256, 0, st>>>(m.num_rows, m.num_cols, m.nnz, d_row_ptr,
                                               d_col_idx, err);
        int h_err = 0;
        SPC5_CUDA(cudaMemcpyAsync(&h_err, err, sizeof(int), cudaMemcpyDeviceToHost, st));
        SPC5_CUDA(cudaStreamSynchronize(st));
        dev_free(err);
        if (h_err)
            return fail(SPC5_EINVAL,
                        "CSR input violates the CsrMatrix contract (row_ptr monotone 0..nnz, "
                        "columns strictly increasing per row and < num_cols)");
    }
    if (m.nnz == 0) {  // blocks.py:102-107
        m.num_blocks = 0;
        SPC5_TRY(dev_alloc(&m.colidx, 1));
        SPC5_TRY(dev_alloc(&m.masks, 1));
        SPC5_TRY(dev_alloc(&m.values, 1));
        return SPC5_OK;
    }
    ConvArgs a{};
    a.num_rows = m.num_rows;
    a.num_panels = np;
    a.row_ptr = d_row_ptr;
    a.col_idx = d_col_idx;
    a.vin = d_values;
    a.vs = m.vs;
    a.vsize = m.value_bytes();
    int64_t *counts = nullptr;
    SPC5_TRY(dev_alloc(&counts, (size_t)np));
    a.panel_blocks = counts;
    struct Events {  // destroyed on every exit path
        cudaEvent_t e[4] = {};
        ~Events() {
            for (auto &x : e)
                if (x) cudaEventDestroy(x);
        }
    } evs;
    cudaEvent_t *ev = evs.e;
    for (int i = 0; i < 4; ++i) SPC5_CUDA(cudaEventCreate(&ev[i]));
    SPC5_CUDA(cudaEventRecord(ev[0], st));
    launch_convert<false>(m.r, a, st);
    SPC5_CUDA(cudaGetLastError());
    SPC5_CUDA(cudaEventRecord(ev[1], st));
    SPC5_TRY(inclusive_scan<int64_t>(counts, m.rowptr + 1, np, st));
    dev_free(counts);
    int64_t nb = 0;
    SPC5_CUDA(cudaMemcpyAsync(&nb, m.rowptr + np, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    SPC5_CUDA(cudaStreamSynchronize(st));
    m.num_blocks = nb;
    SPC5_TRY(dev_alloc(&m.colidx, (size_t)nb));
    SPC5_TRY(dev_alloc(reinterpret_cast<uint8_t **>(&m.masks), (size_t)(nb * m.r * m.mask_bytes())));
    SPC5_TRY(dev_alloc(reinterpret_cast<uint8_t **>(&m.values), (size_t)(m.nnz * m.value_bytes())));
    a.rowptr = m.rowptr;
    a.colidx = m.colidx;
    a.masks = m.masks;
    a.vout = m.values;
    SPC5_CUDA(cudaEventRecord(ev[2], st));
    launch_convert<true>(m.r, a, st);
    SPC5_CUDA(cudaGetLastError());
    if (m.r == 1)  // slot order == CSR order for single-row panels
        SPC5_CUDA(cudaMemcpyAsync(m.values, d_values, (size_t)m.nnz * m.value_bytes(),
                                  cudaMemcpyDeviceToDevice, st));
    SPC5_CUDA(cudaEventRecord(ev[3], st));
    SPC5_CUDA(cudaEventSynchronize(ev[3]));
    cudaEventElapsedTime(&m.k1_count_ms, ev[0], ev[1]);
    cudaEventElapsedTime(&m.k1_fill_ms, ev[2], ev[3]);
    note_launches(m.r == 1 ? 2 : 2);
    return SPC5_OK;
}

int to_csr(const Matrix &m, int64_t *d_row_ptr, int32_t *d_col_idx, void *d_values,
           cudaStream_t st) {
    SPC5_CUDA(cudaMemsetAsync(d_row_ptr, 0, sizeof(int64_t) * (m.num_rows + 1), st));
    if (m.num_blocks == 0) {
        if (m.nnz)
            SPC5_CUDA(cudaMemcpyAsync(d_values, m.values, (size_t)m.nnz * m.value_bytes(),
                                      cudaMemcpyDeviceToDevice, st));
        return SPC5_OK;
    }
    int64_t *counts = nullptr, *voff = nullptr;
    SPC5_TRY(dev_alloc(&counts, (size_t)m.num_rows));
    SPC5_TRY(dev_alloc(&voff, (size_t)m.num_blocks + 1));
    const int64_t threads = m.num_panels * m.r;
    const unsigned grid = (unsigned)cdiv(threads, 256);
    row_counts_kernel<<<grid, 256, 0, st>>>(m.num_rows, m.num_panels, m.r, m.vs, m.rowptr,
                                            m.masks, counts);
    SPC5_CUDA(cudaGetLastError());
    SPC5_TRY(inclusive_scan<int64_t>(counts, d_row_ptr + 1, m.num_rows, st));
    SPC5_TRY(block_value_offsets(m, voff, st));
    to_csr_kernel<<<grid, 256, 0, st>>>(m.num_rows, m.num_panels, m.r, m.vs, m.value_bytes(),
                                        m.rowptr, m.colidx, m.masks, m.values, voff,
                                        d_row_ptr, d_col_idx, d_values);
    SPC5_CUDA(cudaGetLastError());
    SPC5_CUDA(cudaStreamSynchronize(st));
    dev_free(counts);
    dev_free(voff);
    return SPC5_OK;
}

}  // namespace spc5
