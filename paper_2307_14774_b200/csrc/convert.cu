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

#include <algorithm>
#include <mutex>

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

// Count pass.  One group of R lanes per panel (R divides 32, so groups never
// straddle warps) runs the greedy chain and counts the panel's blocks.
template <int R>
__global__ void __launch_bounds__(256) count_kernel(ConvArgs a) {
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
    int64_t nblk = 0;
    const uint32_t kSent = 0xffffffffu;
    const int span = a.vs - 1;
    for (;;) {
        uint32_t anchor = cur < end ? (uint32_t)__ldg(a.col_idx + cur) : kSent;
#pragma unroll
        for (int d = 1; d < R; d <<= 1) anchor = min(anchor, __shfl_xor_sync(gmask, anchor, d));
        if (anchor == kSent) break;
        const uint32_t limit = anchor + (uint32_t)span;
        while (cur < end && (uint32_t)__ldg(a.col_idx + cur) <= limit) ++cur;
        ++nblk;
    }
    if (rr == 0) a.panel_blocks[p] = nblk;
}

// Fill pass with coalesced global traffic.  A CTA of T threads owns T/R
// consecutive panels, so its CSR entries [K0, K1), its blocks [B0, B1) and its
// output values [K0, K1) are contiguous ranges.  Walking the rows straight from
// global memory costs one 32-byte sector transaction per lane and load (rows
// are ~100 bytes apart), which bounds the pass at ~2 TB/s; so
//   A. the CTA loads its column indices into shared memory, consecutive
//      threads on consecutive addresses;
//   B. the lane groups run the greedy chain over the staged columns, write
//      column starts and masks to staged block arrays and overwrite every
//      consumed column index with the value's destination (slot order:
//      block, row-in-panel, column -- the stable argsort of blocks.py:136-137);
//   C. (R > 1) values are read from the CSR array in order, scattered into a
//      staged copy by those destinations and written out in order; for R = 1
//      slot order is CSR order and the values are one device copy.
// A CTA whose ranges exceed the staging capacity (a tail of very long rows)
// walks global memory directly, as the count pass does.
struct StageCaps {
    int entries;  // staged CSR entries (column / destination words; R > 1: + value copy)
    int blocks;   // staged blocks
};

// n (<= vs) values of one block row: four loads in flight, then their stores.
// (A plain out[j] = src[j] loop serialises load -> store -> load: the arrays
// may alias as far as the compiler knows, and every load is an L2 round trip.
// 400^3 beta(2|4|8,8) fill: 24.1 / 15.2 / 16.1 ms with the plain loop -- 9.3 /
// 4.9 / 6.6 ms of it the structure alone, value reads alone +0.4 / +3.3 / +4.6,
// writes alone +4.1 / +3.9 / +3.0 (timing probes) -- and 15.6 / 12.1 / 13.5 ms
// with the loads batched.)
template <typename V>
__device__ __forceinline__ void copy_values(const V *__restrict__ src, V *__restrict__ out, int n) {
    if (n == 1) {  // (most block rows of a power-law matrix)
        out[0] = __ldg(src);
        return;
    }
    for (int j = 0; j < n; j += 4) {
        V v[4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
            if (j + i < n) v[i] = __ldg(src + j + i);
#pragma unroll
        for (int i = 0; i < 4; ++i)
            if (j + i < n) out[j + i] = v[i];
    }
}

template <int R, bool STAGED>
__device__ __forceinline__ void greedy_fill(const ConvArgs &a, int64_t p, int rr, unsigned gmask,
                                            int64_t K0, int64_t B0, uint32_t *s_ci,
                                            uint32_t *s_col, uint8_t *s_mask, int mb) {
    const int64_t row = p * R + rr;
    int64_t cur = 0, end = 0;
    if (row < a.num_rows) {
        cur = a.row_ptr[row];
        end = a.row_ptr[row + 1];
    }
    int64_t bpos = a.rowptr[p];
    int64_t vpos = a.row_ptr[min(p * R, a.num_rows)];
    const uint32_t kSent = 0xffffffffu;
    const int span = a.vs - 1;
    auto col_at = [&](int64_t k) -> uint32_t {
        return STAGED ? s_ci[k - K0] : (uint32_t)__ldg(a.col_idx + k);
    };
    for (;;) {
        uint32_t anchor = cur < end ? col_at(cur) : kSent;
#pragma unroll
        for (int d = 1; d < R; d <<= 1) anchor = min(anchor, __shfl_xor_sync(gmask, anchor, d));
        if (anchor == kSent) break;
        const uint32_t limit = anchor + (uint32_t)span;
        uint32_t m = 0;
        const int64_t s = cur;
        while (cur < end) {
            const uint32_t c = col_at(cur);
            if (c > limit) break;
            m |= 1u << (c - anchor);
            ++cur;
        }
        if (STAGED) {
            if (rr == 0) s_col[bpos - B0] = anchor;
            if (mb == 1) s_mask[(bpos - B0) * R + rr] = (uint8_t)m;
            else reinterpret_cast<uint16_t *>(s_mask)[(bpos - B0) * R + rr] = (uint16_t)m;
        } else {
            if (rr == 0) a.colidx[bpos] = anchor;
            if (mb == 1) static_cast<uint8_t *>(a.masks)[bpos * R + rr] = (uint8_t)m;
            else static_cast<uint16_t *>(a.masks)[bpos * R + rr] = (uint16_t)m;
        }
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
            if (STAGED) {  // destinations replace the consumed columns
                for (int j = 0; j < n; ++j) s_ci[s - K0 + j] = (uint32_t)(dst - K0 + j);
            } else if (a.vsize == 8) {
                copy_values((const double *)a.vin + s, (double *)a.vout + dst, n);
            } else {
                copy_values((const float *)a.vin + s, (float *)a.vout + dst, n);
            }
            vpos += total;
        }
        ++bpos;
    }
}

template <int R>
__global__ void __launch_bounds__(256) fill_staged_kernel(ConvArgs a, StageCaps cap) {
    extern __shared__ __align__(16) uint8_t stage[];
    const int T = (int)blockDim.x, tid = (int)threadIdx.x, lane = tid & 31;
    const int ppc = T / R;  // panels per CTA
    const int64_t P0 = blockIdx.x * (int64_t)ppc;
    const int64_t P1 = min(P0 + ppc, a.num_panels);
    const int64_t B0 = a.rowptr[P0], B1 = a.rowptr[P1];
    const int64_t K0 = a.row_ptr[min(P0 * R, a.num_rows)], K1 = a.row_ptr[min(P1 * R, a.num_rows)];
    const int mb = a.vs <= 8 ? 1 : 2;
    const int64_t nk = K1 - K0, nblk = B1 - B0;
    const bool staged = nk <= cap.entries && nblk <= cap.blocks;  // CTA-uniform
    // layout: value copy (R > 1) | columns / destinations | block column starts | masks
    uint8_t *s_val = stage;
    uint32_t *s_ci = reinterpret_cast<uint32_t *>(stage + (R > 1 ? (size_t)cap.entries * a.vsize : 0));
    uint32_t *s_col = s_ci + cap.entries;
    uint8_t *s_mask = reinterpret_cast<uint8_t *>(s_col + cap.blocks);
    const int64_t p = P0 + tid / R;
    const int rr = tid % R;
    const unsigned gmask = (R == 1) ? (1u << lane) : (((1u << R) - 1u) << (lane & ~(R - 1)));
    if (!staged) {
        if (p < P1) greedy_fill<R, false>(a, p, rr, gmask, K0, B0, s_ci, s_col, s_mask, mb);
        return;
    }
    for (int64_t i = tid; i < nk; i += T) s_ci[i] = (uint32_t)a.col_idx[K0 + i];
    __syncthreads();
    if (p < P1) greedy_fill<R, true>(a, p, rr, gmask, K0, B0, s_ci, s_col, s_mask, mb);
    __syncthreads();
    // coalesced copy-out of the block arrays
    for (int64_t i = tid; i < nblk; i += T) a.colidx[B0 + i] = s_col[i];
    {
        const int64_t nbytes = nblk * R * mb;
        uint8_t *out = static_cast<uint8_t *>(a.masks) + B0 * R * mb;
        // bytes up to the first 4-byte boundary of the output, then words
        const int64_t mis = (int64_t)((4 - (reinterpret_cast<uintptr_t>(out) & 3)) & 3);
        const int head = (int)(mis < nbytes ? mis : nbytes);
        for (int64_t i = tid; i < head; i += T) out[i] = s_mask[i];
        const int64_t nwords = (nbytes - head) / 4;
        uint32_t *ow = reinterpret_cast<uint32_t *>(out + head);
        if (head == 0) {
            const uint32_t *sw = reinterpret_cast<const uint32_t *>(s_mask);
            for (int64_t i = tid; i < nwords; i += T) ow[i] = sw[i];
        } else {  // staged bytes are misaligned relative to the output words
            for (int64_t i = tid; i < nwords; i += T) {
                const uint8_t *b = s_mask + head + i * 4;
                ow[i] = (uint32_t)b[0] | ((uint32_t)b[1] << 8) | ((uint32_t)b[2] << 16) |
                        ((uint32_t)b[3] << 24);
            }
        }
        for (int64_t i = head + nwords * 4 + tid; i < nbytes; i += T) out[i] = s_mask[i];
    }
    if (R > 1) {  // values: in order from CSR, permuted in shared memory, out in order
        if (a.vsize == 8) {
            double *sv = reinterpret_cast<double *>(s_val);
            const double *in = static_cast<const double *>(a.vin) + K0;
            for (int64_t i = tid; i < nk; i += T) sv[s_ci[i]] = in[i];
            __syncthreads();
            double *out = static_cast<double *>(a.vout) + K0;
            for (int64_t i = tid; i < nk; i += T) out[i] = sv[i];
        } else {
            float *sv = reinterpret_cast<float *>(s_val);
            const float *in = static_cast<const float *>(a.vin) + K0;
            for (int64_t i = tid; i < nk; i += T) sv[s_ci[i]] = in[i];
            __syncthreads();
            float *out = static_cast<float *>(a.vout) + K0;
            for (int64_t i = tid; i < nk; i += T) out[i] = sv[i];
        }
    }
}

void launch_count(int r, const ConvArgs &a, cudaStream_t st) {
    const int64_t threads = a.num_panels * r;
    const unsigned grid = (unsigned)cdiv(threads, 256);
    switch (r) {
        case 1: count_kernel<1><<<grid, 256, 0, st>>>(a); break;
        case 2: count_kernel<2><<<grid, 256, 0, st>>>(a); break;
        case 4: count_kernel<4><<<grid, 256, 0, st>>>(a); break;
        default: count_kernel<8><<<grid, 256, 0, st>>>(a); break;
    }
}

// CTA shape of the fill pass: T threads (T/R panels) sized so that the staged
// ranges of an average CTA, plus 25 %, fit ~48 KB (several CTAs per SM).
template <int R>
int launch_fill(const ConvArgs &a, int64_t nnz, int64_t nb, cudaStream_t st) {
    const double rows = (double)std::max<int64_t>(a.num_rows, 1);
    const int mb = a.vs <= 8 ? 1 : 2;
    const double erow = (double)nnz / rows;  // entries per row
    const double ebytes = 4.0 + (R > 1 ? a.vsize : 0);
    const double brow = (double)nb / rows * (4.0 / R + mb);  // staged block bytes per row
    int T = 256;
    while (T > 32 && (erow * ebytes + brow) * T * 1.25 > 48.0 * 1024) T >>= 1;
    StageCaps cap;
    cap.entries = ((int)(erow * T * 1.25) + 128 + 3) / 4 * 4;
    cap.blocks = ((int)((double)nb / rows * T / R * 1.25) + 64 + 3) / 4 * 4;
    size_t smem = (size_t)cap.entries * (size_t)ebytes + (size_t)cap.blocks * (4 + R * mb) + 16;
    // (Staging only the block outputs of R > 1 was slower too: 400^3 fill
    // beta(2|4|8,8) 20.0 / 14.1 / 15.7 vs 15.6 / 12.1 / 13.5 ms direct.)
    // R > 1: the staged path measured slower than the direct walk (400^3 stencil
    // beta(8,8) fill 46 vs 18 ms, FEM beta(8,8) 7.5 vs 1.1 ms: the value
    // permutation through shared memory and CTAs of 64-128 threads cost more
    // than the sector-per-lane loads they replace), so only R = 1 stages
    // (beta(1,8) 9.8 -> 8.9 ms, beta(1,16) 8.4 -> 6.6 ms).
    if (R > 1 || smem > 160 * 1024) {  // (or rows of several KB on average)
        T = 256;
        cap.entries = 0;
        cap.blocks = 0;
        smem = 16;
    }
    static std::once_flag once;
    static cudaError_t attr_err = cudaSuccess;
    std::call_once(once, [] {
        attr_err = cudaFuncSetAttribute(fill_staged_kernel<R>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    });
    if (attr_err != cudaSuccess) return cuda_fail(attr_err, "cudaFuncSetAttribute(fill_staged_kernel)");
    const unsigned grid = (unsigned)cdiv(a.num_panels, T / R);
    fill_staged_kernel<R><<<grid, T, smem, st>>>(a, cap);
    SPC5_CUDA(cudaGetLastError());
    return SPC5_OK;
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
    launch_count(m.r, a, st);
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
    switch (m.r) {
        case 1: SPC5_TRY(launch_fill<1>(a, m.nnz, nb, st)); break;
        case 2: SPC5_TRY(launch_fill<2>(a, m.nnz, nb, st)); break;
        case 4: SPC5_TRY(launch_fill<4>(a, m.nnz, nb, st)); break;
        default: SPC5_TRY(launch_fill<8>(a, m.nnz, nb, st)); break;
    }
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
