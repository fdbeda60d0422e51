// plan.cu -- K3: popcount prefix, structural checks, the SpMV work plan and
// partition_by_nnz, all on the device.
//
//  * mask_popcounts / block_value_offsets (kernels.py:82-96): per-tile
//    popcount sums (kTile blocks) + an exclusive scan; the value offset of any
//    block b is tile_prefix[b / kTile] + a warp popcount over < kTile blocks.
//  * The SpMV plan cuts the block array into chunks (one ring slot each).
//    Chunk starts are panel starts (targets every CB blocks snapped back to
//    the start of the panel holding them) plus, inside panels longer than
//    split_len blocks, the GLOBAL multiples of split_len (the largest power of
//    two whose fullest window fits 6 KB).  Per chunk the plan also writes a
//    metadata blob and a bulk-copy issue record (see blob_fill_kernel).
//  * partition_by_nnz (parallel.py:31-52): boundary_k =
//    searchsorted(cum, total*k/P, 'left') + 1 with cum[p] = nnz up to the end
//    of panel p, clamped to num_panels; one warp binary-searches each target.
//  * validate_spc5 (blocks.py:201-232): same checks, same messages, same order.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <string>
#include <vector>

#include "common.cuh"

namespace spc5 {
int scan_inclusive_i64(const int64_t *in, int64_t *out, int64_t n, cudaStream_t st);

namespace {

__global__ void tile_sums_kernel(int64_t nb, int r, int vs, const void *__restrict__ masks,
                                 int64_t num_tiles, int64_t *tile_sums) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t t = warp; t < num_tiles; t += nwarps) {
        const int64_t lo = t * kTile * r, hi = std::min<int64_t>((t + 1) * kTile, nb) * r;
        int s = 0;
        for (int64_t i = lo + lane; i < hi; i += 32) s += __popc(load_mask(masks, i, vs));
        s = __reduce_add_sync(0xffffffffu, s);
        if (lane == 0) tile_sums[t] = s;
    }
}

// value offset of block b, computed by a full warp
__device__ int64_t warp_value_offset(int64_t b, int r, int vs, const void *masks,
                                     const int64_t *tile_prefix) {
    const int lane = threadIdx.x & 31;
    const int64_t t = b / kTile;
    int s = 0;
    for (int64_t i = t * kTile * r + lane; i < b * r; i += 32) s += __popc(load_mask(masks, i, vs));
    s = __reduce_add_sync(0xffffffffu, s);
    return tile_prefix[t] + s;
}

// first index i in [0, n] with a[i] > key (a non-decreasing)
__device__ __forceinline__ int64_t upper_bound_dev(const int64_t *a, int64_t n, int64_t key) {
    int64_t lo = 0, hi = n + 1;
    while (lo < hi) {
        const int64_t mid = lo + (hi - lo) / 2;
        if (a[mid] <= key) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ int64_t cdiv_dev(int64_t a, int64_t b) { return (a + b - 1) / b; }

// structural checks over panels (thread per panel)
struct CheckOut {
    unsigned long long popc;
    int rowptr_bad;      // non-decreasing / start
    int bits_beyond;     // mask >> vs != 0
    int anchor_missing;  // OR of the block's masks lacks bit 0
    int past_end;        // set bit maps to column >= num_cols
    long long first_unsorted_panel;
};

__global__ void check_kernel(int64_t num_panels, int64_t nb, int64_t num_cols, int r, int vs,
                             const int64_t *__restrict__ rowptr,
                             const uint32_t *__restrict__ colidx,
                             const void *__restrict__ masks, CheckOut *out) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= num_panels) return;
    const int64_t s = rowptr[p], e = rowptr[p + 1];
    if (e < s || s < 0 || e > nb || (p == 0 && s != 0)) {
        atomicOr(&out->rowptr_bad, 1);
        return;
    }
    unsigned long long pc = 0;
    int beyond = 0, anchor = 0, past = 0;
    bool unsorted = false;
    for (int64_t b = s; b < e; ++b) {
        uint32_t orm = 0;
        for (int rr = 0; rr < r; ++rr) {
            const uint32_t m = load_mask(masks, b * r + rr, vs);
            orm |= m;
            pc += __popc(m);
        }
        if (orm >> vs) beyond = 1;
        if (!(orm & 1u)) anchor = 1;
        if (orm && (int64_t)colidx[b] + (31 - __clz(orm)) >= num_cols) past = 1;
        if (b > s && colidx[b] <= colidx[b - 1]) unsorted = true;
    }
    if (pc) atomicAdd(&out->popc, pc);
    if (beyond) atomicOr(&out->bits_beyond, 1);
    if (anchor) atomicOr(&out->anchor_missing, 1);
    if (past) atomicOr(&out->past_end, 1);
    if (unsorted) atomicMin(&out->first_unsorted_panel, (long long)p);
}

// ---- chunk plan ----------------------------------------------------------
// (a) snapped targets
__global__ void targets_kernel(int64_t num_panels, const int64_t *__restrict__ rowptr,
                               int64_t cb, int64_t num_targets, int64_t *cand) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= num_targets) return;
    if (c == 0) {
        cand[0] = 0;
        return;
    }
    const int64_t t = c * cb;
    const int64_t P = upper_bound_dev(rowptr, num_panels, t) - 1;
    cand[c] = rowptr[P];
}

// (a'') exact targets (LBR plans): a chunk at every global multiple of cb
// blocks, whatever the panels (chunk heads inside a panel use the carry slots)
__global__ void targets_exact_kernel(int64_t nb, int64_t base, int64_t cb, int64_t num_targets,
                                     int64_t *cand) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= num_targets) return;
    cand[c] = c == 0 ? 0 : min((base / cb + c) * cb - base, nb - 1);
}

// (a') panel-count targets: a chunk every ppc panels (regular matrices, so
// every lane-per-panel-row step of the chunk is a full warp)
__global__ void targets_panels_kernel(int64_t num_panels, const int64_t *__restrict__ rowptr,
                                      int64_t ppc, int64_t num_targets, int64_t *cand) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= num_targets) return;
    cand[c] = rowptr[min(c * ppc, num_panels)];
}

// (b) forced splits inside giant panels at global multiples of kSplit
__device__ __forceinline__ int64_t split_count(int64_t s, int64_t e, int64_t base,
                                               int64_t kSplit) {
    if (e - s <= kSplit) return 0;
    const int64_t gs = s + base, ge = e + base;
    // multiples g of kSplit with gs < g < ge
    const int64_t first = gs / kSplit + 1, last = (ge - 1) / kSplit;
    return last >= first ? last - first + 1 : 0;
}

__global__ void split_count_kernel(int64_t num_panels, const int64_t *__restrict__ rowptr,
                                   int64_t base, int64_t kSplit, int64_t *counts) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= num_panels) return;
    counts[p] = split_count(rowptr[p], rowptr[p + 1], base, kSplit);
}

__global__ void split_fill_kernel(int64_t num_panels, const int64_t *__restrict__ rowptr,
                                  int64_t base, int64_t kSplit, const int64_t *__restrict__ incl,
                                  int64_t *out) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= num_panels) return;
    const int64_t s = rowptr[p], e = rowptr[p + 1];
    const int64_t n = split_count(s, e, base, kSplit);
    if (!n) return;
    int64_t pos = incl[p] - n;
    const int64_t first = (s + base) / kSplit + 1;
    for (int64_t j = 0; j < n; ++j) out[pos + j] = (first + j) * kSplit - base;
}

__global__ void chunk_desc_kernel(int64_t num_chunks, int64_t num_panels, int r, int vs,
                                  const int64_t *__restrict__ rowptr, const void *__restrict__ masks,
                                  const int64_t *__restrict__ tile_prefix,
                                  const int64_t *__restrict__ chunk_b, int64_t *chunk_v,
                                  int64_t *chunk_p, uint8_t *split_flag) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t c = warp; c < num_chunks; c += nwarps) {
        const int64_t b = chunk_b[c];
        const int64_t v = warp_value_offset(b, r, vs, masks, tile_prefix);
        if (lane == 0) {
            const int64_t P = upper_bound_dev(rowptr, num_panels, b) - 1;
            chunk_v[c] = v;
            chunk_p[c] = P;
            split_flag[c] = rowptr[P] < b ? 1 : 0;
        }
    }
}

__global__ void empty_flag_kernel(int64_t num_panels, const int64_t *__restrict__ rowptr,
                                  uint8_t *flag) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p < num_panels) flag[p] = rowptr[p] == rowptr[p + 1] ? 1 : 0;
}

// ---- ring-slot sizing ------------------------------------------------------
// largest popcount of one block (all r rows)
// most values in one window of sl blocks at global multiples of sl (warp per
// window): bounds the bytes of any piece of a panel cut at those multiples
__global__ void window_values_max_kernel(int64_t nb, int r, int vs, const void *__restrict__ masks,
                                         int64_t base, int64_t sl, unsigned long long *out) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t w0 = base / sl, w1 = (base + nb - 1) / sl;
    int best = 0;
    for (int64_t w = w0 + warp; w <= w1; w += nwarps) {
        const int64_t lo = max(w * sl - base, (int64_t)0), hi = min((w + 1) * sl - base, nb);
        int s = 0;
        for (int64_t b = lo + lane; b < hi; b += 32)
            for (int rr = 0; rr < r; ++rr) s += __popc(load_mask(masks, b * r + rr, vs));
        best = max(best, __reduce_add_sync(0xffffffffu, s));
    }
    if (lane == 0) atomicMax(out, (unsigned long long)best);
}

// max blocks and max values of one chunk (a chunk is one shared-memory slot)
__global__ void chunk_stats_kernel(int64_t nc, const int64_t *__restrict__ chunk_b,
                                   const int64_t *__restrict__ chunk_v,
                                   unsigned long long *out /* [2] */) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= nc) return;
    atomicMax(out, (unsigned long long)(chunk_b[c + 1] - chunk_b[c]));
    atomicMax(out + 1, (unsigned long long)(chunk_v[c + 1] - chunk_v[c]));
}

// is every row mask one contiguous run of bits (or empty)?  Stencils, bands and
// dense sub-blocks are; K2's lane-per-panel-row steps then gather x at
// immediate offsets from the run's top (spmv_kernel.cuh row_slots RUN)
__global__ void runs_kernel(int64_t nmasks, int vs, const void *__restrict__ masks, int *not_runs) {
    int bad = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nmasks;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t m = load_mask(masks, i, vs);
        const uint32_t t = m >> (__ffs(m | 0x80000000u) - 1);  // run shifted down to bit 0
        bad |= (m != 0u && (t & (t + 1u)) != 0u) ? 1 : 0;
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(not_runs, 1);
}

// panel-start bitmap over granules (derived plan data, 1 bit per block)
__global__ void pstart_bits_kernel(int64_t np, const int64_t *__restrict__ rowptr, int off32,
                                   uint32_t *bits) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= np) return;
    const int64_t b = rowptr[p];
    if (b == rowptr[p + 1]) return;  // empty panel: no block starts it
    atomicOr(bits + ((b + off32) >> 5), 1u << ((b + off32) & 31));
}

// per chunk: bit0 = first block is not a panel start, bit1 = empty panels
// inside, bit2 = lane-per-panel-row mode (non-empty panels of similar
// length, >= kLppMinLanes lanes busy), bits3-4 = log2 G: in that mode each
// panel row is split over G lanes (contiguous block ranges, partial sums
// combined by a butterfly), so short chunks still fill the warp; bit5 = in
// that mode, the last panel continues into the next chunk
constexpr int64_t kLppMinLanes = 24;  // panels * r * G
__constant__ int fvr_dense_q = 4;  // FVR instead of LPP below fvr_dense_q/4 values per block row
__global__ void chunk_flags_kernel(int64_t nc, int64_t nb, int64_t np, int r,
                                   const int64_t *__restrict__ chunk_b,
                                   const int64_t *__restrict__ chunk_p,
                                   const int64_t *__restrict__ rowptr,
                                   const int64_t *__restrict__ empty, int64_t ne, int lpr_split,
                                   int lpr_bal_num, int lpr_bal_den, int fvr, int64_t min_lanes,
                                   const int64_t *__restrict__ chunk_v, uint8_t *flags) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= nc) return;
    uint8_t f = rowptr[chunk_p[c]] < chunk_b[c] ? 1 : 0;
    // any empty panel p with chunk_p[c] < p < chunk_p[c+1]?
    const int64_t lo_p = chunk_p[c], hi_p = chunk_p[c + 1];
    int64_t lo = 0, hi = ne;  // first empty panel > lo_p
    while (lo < hi) {
        const int64_t mid = (lo + hi) / 2;
        if (empty[mid] <= lo_p) lo = mid + 1;
        else hi = mid;
    }
    if (lo < ne && empty[lo] < hi_p) f |= 2;
    if (!(f & 2)) {
        // lane-per-panel-row candidate: the chunk's panels, the first possibly
        // started in an earlier chunk (bit0, carry slot) and the last possibly
        // continuing into the next one (bit5)
        const int64_t cb0 = chunk_b[c], cb1 = chunk_b[c + 1];
        const bool ends_clean = hi_p >= np ? cb1 == nb : rowptr[hi_p] == cb1;
        const int64_t npc = hi_p - lo_p + (ends_clean ? 0 : 1);
        // split pieces of long panels run faster in balanced-lane-range mode
        const bool whole = !(f & 1) && ends_clean;
        if ((whole || lpr_split) && lpr_split >= 0 && npc > 0 && npc * r <= 32 * 64) {
            int64_t maxlen = 0;
            for (int64_t p = lo_p; p < lo_p + npc; ++p)
                maxlen = max(maxlen, min(rowptr[p + 1], cb1) - max(rowptr[p], cb0));
            int lg = 0;  // G = 1 << lg lanes per panel row, each with >= 1 block
            while (lg < 3 && npc * r * (2 << lg) <= 32 && maxlen >= (2 << lg)) ++lg;
            if (npc * r * (1 << lg) >= min_lanes && maxlen <= 64 * (1 << lg) &&
                maxlen * npc * lpr_bal_den <= lpr_bal_num * (cb1 - cb0) + 2 * lpr_bal_den * npc)
                f |= 4 | (lg << 3) | (ends_clean ? 0 : 32);
        }
        // flat value-range mode (bit6): fvr 1 (default) for the other
        // chunks without empty panels when r >= 2 (for r = 1 the
        // balanced-lane-range steps are cheaper) and for lane-per-panel
        // chunks that are sparse (fewer than fvr_dense/4 values per block
        // row: lane-per-panel-row lanes would mostly find empty rows); fvr 2:
        // also r = 1; fvr 3: every chunk without empty panels.  Record fields
        // limit a chunk to 4096 blocks and 8192 panels.
        const int64_t nvals = chunk_v[c + 1] - chunk_v[c];
        const bool sparse = nvals * 4 < (int64_t)fvr_dense_q * (cb1 - cb0) * r;
        if (fvr >= 1 && cb1 - cb0 < 4096 && hi_p - lo_p < 8192 &&
            ((f & 4) ? (sparse || fvr >= 3) : (r >= 2 || fvr >= 2)))
            f = (f & 3) | 64 | ((f & 4) ? 0 : 128);  // bit7: was a scan chunk
    }
    flags[c] = f;
}

// Per-chunk metadata blob (what K2 stages first into a ring slot):
//   [0,64)  header: b0, b1, v0, p0, pe (int64), flags, rec offset (int32)
//   [64,..) panel-start words of granules (b0+off32)>>5 .. (b1-1+off32)>>5
//           (scan-mode chunks only)
//   [rec,.) lane-per-panel chunks: for q = 0..npc the record
//           (rowptr[p0+q] - b0) | (values before panel p0+q in the chunk) << 16
__device__ __forceinline__ void blob_shape(int64_t b0, int64_t b1, int64_t npc, int flags,
                                           int off32, int64_t *nwords, int64_t *nrec) {
    const bool lpr = flags & 4;
    *nwords = (!lpr && b1 > b0) ? ((b1 - 1 + off32) >> 5) - ((b0 + off32) >> 5) + 1 : 0;
    // G sub-ranges per panel; scan modes 32 lane records (+ the value count in FVR mode)
    *nrec = lpr ? npc * (1 << ((flags >> 3) & 3)) + 1 : ((flags & 64) ? 33 : 32);
}
__device__ __forceinline__ int64_t a16_dev(int64_t v) { return (v + 15) / 16 * 16; }

__global__ void blob_size_kernel(int64_t nc, const int64_t *__restrict__ chunk_b,
                                 const int64_t *__restrict__ chunk_p,
                                 const uint8_t *__restrict__ flags, int off32, int64_t *size16) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= nc) return;
    int64_t nw, nr;
    blob_shape(chunk_b[c], chunk_b[c + 1], chunk_p[c + 1] - chunk_p[c] + ((flags[c] >> 5) & 1),
               flags[c], off32, &nw, &nr);
    size16[c] = (64 + a16_dev(nw * 4) + a16_dev(nr * 4)) / 16;
}

// warp per chunk: header, panel-start words, panel records
__global__ void blob_fill_kernel(int64_t nc, int r, int vs, int off32,
                                 const int64_t *__restrict__ chunk_b,
                                 const int64_t *__restrict__ chunk_v,
                                 const int64_t *__restrict__ chunk_p,
                                 const uint8_t *__restrict__ flags,
                                 const int64_t *__restrict__ rowptr, const void *__restrict__ masks,
                                 const uint32_t *__restrict__ pstart_bits,
                                 const int64_t *__restrict__ off16_incl, uint8_t *blob) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t c = warp; c < nc; c += nwarps) {
        const int64_t b0 = chunk_b[c], b1 = chunk_b[c + 1], p0 = chunk_p[c], pe = chunk_p[c + 1];
        const int f = flags[c];
        const int64_t npc = pe - p0 + ((f >> 5) & 1);  // lane-per-panel: incl. a tail panel
        int64_t nw, nr;
        blob_shape(b0, b1, npc, f, off32, &nw, &nr);
        uint8_t *bl = blob + (c ? off16_incl[c - 1] : 0) * 16;
        const int rec_off = (int)(64 + a16_dev(nw * 4));
        if (lane == 0) {
            int64_t *h = reinterpret_cast<int64_t *>(bl);
            h[0] = b0;
            h[1] = b1;
            h[2] = chunk_v[c];
            h[3] = p0;
            h[4] = (f & 4) ? p0 + npc : pe;
            reinterpret_cast<int *>(bl)[10] = f;
            reinterpret_cast<int *>(bl)[11] = rec_off;
            h[6] = h[7] = 0;
        }
        uint32_t *words = reinterpret_cast<uint32_t *>(bl + 64);
        const int64_t g0 = (b0 + off32) >> 5;
        for (int64_t i = lane; i < nw; i += 32) words[i] = pstart_bits[g0 + i];
        uint32_t *rec = reinterpret_cast<uint32_t *>(bl + rec_off);
        if (f & 64) {
            // flat value-range chunk: lane l of K2 owns the chunk's values
            // [l*nv/32, (l+1)*nv/32); record = block holding its first value |
            // set bits of that block before it << 12 | panel of that block << 19
            // (relative to b0 / p0); rec[32] = nv
            const int64_t n = b1 - b0;
            const int64_t nv = chunk_v[c + 1] - chunk_v[c];
            const int64_t sl = (lane * n) >> 5, el = ((lane + 1) * n) >> 5;
            int cnt = 0;
            for (int64_t b = sl; b < el; ++b)
                for (int rr = 0; rr < r; ++rr) cnt += __popc(load_mask(masks, (b0 + b) * r + rr, vs));
            int vin = cnt;
            for (int d = 1; d < 32; d <<= 1) {
                const int tv = __shfl_up_sync(0xffffffffu, vin, d);
                if (lane >= d) vin += tv;
            }
            const int j = (int)((lane * nv) >> 5);
            int k = 0;  // the lane whose block range holds value j
            for (int d = 0; d < 32; ++d) k += __shfl_sync(0xffffffffu, vin, d) <= j ? 1 : 0;
            const int excl = __shfl_sync(0xffffffffu, vin - cnt, min(k, 31));
            int64_t b = ((int64_t)min(k, 31) * n) >> 5;
            int run = excl, skip = 0;
            for (; b < n; ++b) {
                int cb = 0;
                for (int rr = 0; rr < r; ++rr) cb += __popc(load_mask(masks, (b0 + b) * r + rr, vs));
                if (run + cb > j) {
                    skip = j - run;
                    break;
                }
                run += cb;
            }
            // panel of block b: panel starts in chunk blocks 1 .. b
            int starts = 0;
            for (int64_t bb = 1; bb <= b; ++bb) {
                const int64_t gb = b0 + bb + off32;
                starts += (int)((pstart_bits[gb >> 5] >> (gb & 31)) & 1u);
            }
            rec[lane] = (uint32_t)b | ((uint32_t)skip << 12) | ((uint32_t)starts << 19);
            if (lane == 0) rec[32] = (uint32_t)nv;
            continue;
        }
        if (!(f & 4)) {
            // scan-mode chunk: lane l of K2 owns blocks [l*n/32, (l+1)*n/32);
            // record = values before its first block | (panel starts in
            // blocks 1 .. its first block) << 16
            const int64_t n = b1 - b0;
            const int64_t sl = (lane * n) >> 5, el = ((lane + 1) * n) >> 5;
            int cnt = 0, starts = 0;
            for (int64_t b = sl; b < el; ++b) {
                for (int rr = 0; rr < r; ++rr) cnt += __popc(load_mask(masks, (b0 + b) * r + rr, vs));
                const int64_t gb = b0 + b + off32;
                starts += b > 0 ? (int)((pstart_bits[gb >> 5] >> (gb & 31)) & 1u) : 0;
            }
            int vin = cnt, pin = starts;
            for (int d = 1; d < 32; d <<= 1) {
                const int tv = __shfl_up_sync(0xffffffffu, vin, d);
                const int tp = __shfl_up_sync(0xffffffffu, pin, d);
                if (lane >= d) {
                    vin += tv;
                    pin += tp;
                }
            }
            // panel of the lane's first block: starts in blocks 1 .. sl
            int first = pin - starts;
            if (sl > 0 && sl < el) {
                const int64_t gb = b0 + sl + off32;
                first += (int)((pstart_bits[gb >> 5] >> (gb & 31)) & 1u);
            }
            rec[lane] = (uint32_t)(vin - cnt) | ((uint32_t)first << 16);
            continue;
        }
        // entry t = q*G + sub: start of sub-range sub of panel p0+q (G contiguous
        // block ranges, ceil(len/G) blocks each), last entry = chunk end
        const int lg = (f >> 3) & 3, G = 1 << lg;
        uint32_t running = 0;
        for (int64_t t0 = 0; t0 < nr; t0 += 32) {
            const int64_t t = t0 + lane;
            auto start = [&](int64_t tt) -> int64_t {  // block offset of entry tt
                if (tt >= nr - 1) return b1 - b0;
                const int64_t q = tt >> lg, sub = tt & (G - 1);
                // panel p0+q's blocks inside the chunk: [max(rowptr, b0), min(rowptr', b1))
                const int64_t ps = min(max(rowptr[p0 + q], b0), b1) - b0;
                const int64_t pe2 = min(rowptr[p0 + q + 1], b1) - b0;
                const int64_t len = pe2 - ps, per = (len + G - 1) >> lg;
                return ps + min(sub * per, len);
            };
            const int64_t s = t < nr ? start(t) : 0;
            int cnt = 0;
            if (t < nr - 1) {
                const int64_t e = start(t + 1);
                for (int64_t b = b0 + s; b < b0 + e; ++b)
                    for (int rr = 0; rr < r; ++rr) cnt += __popc(load_mask(masks, b * r + rr, vs));
            }
            int incl = cnt;
            for (int d = 1; d < 32; d <<= 1) {
                const int tv = __shfl_up_sync(0xffffffffu, incl, d);
                if (lane >= d) incl += tv;
            }
            if (t < nr) rec[t] = (uint32_t)s | ((running + (uint32_t)(incl - cnt)) << 16);
            running += (uint32_t)__shfl_sync(0xffffffffu, incl, 31);
        }
    }
}

// the producer's view of a chunk: source offsets and sizes of its bulk copies
// in 16-byte units (blob, column starts, masks, values) and the byte total
__global__ void issue_rec_kernel(int64_t nc, int lb, int vb, const int64_t *__restrict__ chunk_b,
                                 const int64_t *__restrict__ chunk_v,
                                 const int64_t *__restrict__ off16_incl, uint4 *ir) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= nc) return;
    const int64_t b0 = chunk_b[c], b1 = chunk_b[c + 1], v0 = chunk_v[c], v1 = chunk_v[c + 1];
    const int64_t m0 = c ? off16_incl[c - 1] : 0, mb = off16_incl[c] - m0;
    const int64_t c0 = (b0 * 4) >> 4, cb = ((b1 * 4 + 15) >> 4) - c0;
    const int64_t k0 = (b0 * lb) >> 4, kb = ((b1 * lb + 15) >> 4) - k0;
    const int64_t q0 = (v0 * vb) >> 4, qb = v1 > v0 ? ((v1 * vb + 15) >> 4) - q0 : 0;
    uint4 A, B;
    A.x = (uint32_t)m0;
    A.y = (uint32_t)c0;
    A.z = (uint32_t)k0;
    A.w = (uint32_t)q0;
    B.x = (uint32_t)mb | ((uint32_t)cb << 16);
    B.y = (uint32_t)kb | ((uint32_t)qb << 16);
    B.z = (uint32_t)((mb + cb + kb + qb) * 16);
    B.w = 0;
    ir[2 * c] = A;
    ir[2 * c + 1] = B;
}

// x leading edge of every chunk, for the L2 prefetch K2 issues when it
// queues the chunk's bulk copies: xmax[c] = the end of the columns chunk c
// reads (max over its blocks of colidx + vs, clipped); the new x of chunk c
// is [xmax[c-1], xmax[c]) -- for banded matrices walked in row order that is
// the band's leading edge, first read by this chunk.  Encoded into the issue
// record's last word (B.w): start | sectors << 27 in 32-byte sectors (at most
// 31 sectors, the nearest part of the range; 0 = no prefetch: the range is
// empty, goes backwards, or x is past 4 GB).
__global__ void chunk_xmax_kernel(int64_t nc, const int64_t *__restrict__ chunk_b,
                                  const uint32_t *__restrict__ colidx, int vs, int64_t num_cols,
                                  int64_t *xmax) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t c = warp; c < nc; c += nw) {
        int64_t mx = 0;
        for (int64_t b = chunk_b[c] + lane; b < chunk_b[c + 1]; b += 32)
            mx = max(mx, min((int64_t)colidx[b] + vs, num_cols));
        for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (lane == 0) xmax[c] = mx;
    }
}

__global__ void xedge_kernel(int64_t nc, const int64_t *__restrict__ xmax, int vb, uint4 *ir) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= nc) return;
    const int64_t hi = xmax[c] * vb, lo = c ? xmax[c - 1] * vb : 0;  // bytes
    uint32_t w = 0;
    if (hi > lo && hi <= (int64_t(1) << 32)) {
        const int64_t s1 = hi >> 5;                        // whole sectors inside x only
        const int64_t s0 = max(lo >> 5, s1 - 31);          // at most 31 sectors
        if (s1 > s0) w = (uint32_t)s0 | ((uint32_t)(s1 - s0) << 27);
    }
    ir[2 * c + 1].w = w;
}

// scan chunks of a mostly lane-per-panel plan go back to balanced lane ranges
// (bit7 -> clear bit6): the kernel without the FVR code then runs the plan
__global__ void unfvr_kernel(int64_t nc, uint8_t *flags, unsigned long long *cleared) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c < nc && (flags[c] & 128)) {
        flags[c] &= (uint8_t)~(64 | 128);
        atomicAdd(cleared, 1ull);
    }
}

// largest panel count of a lane-per-panel chunk (sizes the staged records)
__global__ void lpp_panels_kernel(int64_t nc, const int64_t *__restrict__ chunk_p,
                                  const uint8_t *__restrict__ flags, unsigned long long *out,
                                  unsigned long long *num_fvr, unsigned long long *num_lpp) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c < nc && (flags[c] & 64)) atomicAdd(num_fvr, 1ull);
    if (c < nc && (flags[c] & 4)) atomicAdd(num_lpp, 1ull);
    if (c < nc && (flags[c] & 4))
        atomicMax(out, (unsigned long long)((chunk_p[c + 1] - chunk_p[c] + ((flags[c] >> 5) & 1))
                                            << ((flags[c] >> 3) & 3)));
}

__global__ void narrow_kernel(const int64_t *in, int64_t n, int *out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) out[i] = (int)in[i];
}

// ---- partition_by_nnz ----------------------------------------------------
__global__ void partition_kernel(int64_t num_panels, int r, int vs,
                                 const int64_t *__restrict__ rowptr, const void *__restrict__ masks,
                                 const int64_t *__restrict__ tile_prefix, int64_t num_tiles,
                                 int workers, int64_t *bounds) {
    const int lane = threadIdx.x & 31;
    const int k = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) + 1;
    if (k >= workers) return;
    const int64_t total = num_panels ? tile_prefix[num_tiles] : 0;
    const double target = (double)(total * (int64_t)k) / (double)workers;
    int64_t res;
    if (target <= 0) {
        res = 0;
    } else {
        int64_t lo = 0, hi = num_panels;  // searchsorted 'left' over cum[0..num_panels)
        while (lo < hi) {
            const int64_t mid = lo + (hi - lo) / 2;
            const int64_t cum = warp_value_offset(rowptr[mid + 1], r, vs, masks, tile_prefix);
            if ((double)cum < target) lo = mid + 1;
            else hi = mid;
        }
        res = lo + 1;
    }
    if (lane == 0) bounds[k] = res < num_panels ? res : num_panels;
}

struct BlockPopc {
    const void *masks;
    int r, vs;
    __host__ __device__ int64_t operator()(int64_t b) const {
#ifdef __CUDA_ARCH__
        int64_t s = 0;
        for (int rr = 0; rr < r; ++rr) s += __popc(load_mask(masks, b * r + rr, vs));
        return s;
#else
        return 0;
#endif
    }
};

int select_flagged(const uint8_t *flags, int64_t n, int64_t *out, int64_t *h_count,
                   cudaStream_t st) {
    *h_count = 0;
    if (n <= 0) return SPC5_OK;
    int64_t *d_count = nullptr;
    SPC5_TRY(dev_alloc(&d_count, 1));
    thrust::counting_iterator<int64_t> it(0);
    size_t bytes = 0;
    SPC5_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, it, flags, out, d_count, n, st));
    void *tmp = nullptr;
    SPC5_TRY(dev_alloc(&tmp, bytes));
    SPC5_CUDA(cub::DeviceSelect::Flagged(tmp, bytes, it, flags, out, d_count, n, st));
    SPC5_CUDA(cudaMemcpyAsync(h_count, d_count, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    SPC5_CUDA(cudaStreamSynchronize(st));
    dev_free(tmp);
    dev_free(d_count);
    return SPC5_OK;
}

int run_checks(const Matrix &m, CheckOut *h, cudaStream_t st) {
    CheckOut init{};
    init.first_unsorted_panel = (long long)INT64_MAX;
    *h = init;
    if (m.num_panels == 0) return SPC5_OK;
    CheckOut *d = nullptr;
    SPC5_TRY(dev_alloc(&d, 1));
    SPC5_CUDA(cudaMemcpyAsync(d, &init, sizeof(CheckOut), cudaMemcpyHostToDevice, st));
    check_kernel<<<(unsigned)cdiv(m.num_panels, 256), 256, 0, st>>>(
        m.num_panels, m.num_blocks, m.num_cols, m.r, m.vs, m.rowptr, m.colidx, m.masks, d);
    SPC5_CUDA(cudaGetLastError());
    SPC5_CUDA(cudaMemcpyAsync(h, d, sizeof(CheckOut), cudaMemcpyDeviceToHost, st));
    SPC5_CUDA(cudaStreamSynchronize(st));
    dev_free(d);
    return SPC5_OK;
}

int rowptr_ends(const Matrix &m, int64_t *first, int64_t *last, cudaStream_t st) {
    SPC5_CUDA(cudaMemcpyAsync(first, m.rowptr, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    SPC5_CUDA(cudaMemcpyAsync(last, m.rowptr + m.num_panels, sizeof(int64_t),
                              cudaMemcpyDeviceToHost, st));
    SPC5_CUDA(cudaStreamSynchronize(st));
    return SPC5_OK;
}

}  // namespace

void free_plan(Plan &p) {
    dev_free(p.chunk_b);
    dev_free(p.chunk_v);
    dev_free(p.chunk_p);
    dev_free(p.split_chunks);
    dev_free(p.carry);
    dev_free(p.empty_panels);
    dev_free(p.tile_prefix);
    dev_free(p.pstart_bits);
    dev_free(p.chunk_flags);
    dev_free(p.blob);
    dev_free(p.issue_rec);
    delete[] p.h_chunk_b;
    p = Plan{};
}

int validate_structure(const Matrix &m, cudaStream_t st) {
    int64_t first = 0, last = 0;
    SPC5_TRY(rowptr_ends(m, &first, &last, st));
    CheckOut h;
    SPC5_TRY(run_checks(m, &h, st));
    if (h.rowptr_bad || (m.num_panels >= 0 && first != 0))
        return fail(SPC5_EINVAL, "block_rowptr must be non-decreasing and start at 0");
    if (m.num_panels && last != m.num_blocks)
        return fail(SPC5_EINVAL, "block_rowptr does not cover all blocks");
    if (h.bits_beyond) return fail(SPC5_EINVAL, "mask has bits beyond vs");
    if ((int64_t)h.popc != m.nnz) return fail(SPC5_EINVAL, "sum of mask popcounts differs from NNZ");
    if (m.num_blocks) {
        if (h.anchor_missing) return fail(SPC5_EINVAL, "block without an entry at its anchor column");
        if (h.first_unsorted_panel != (long long)INT64_MAX)
            return fail(SPC5_EINVAL, "panel " + std::to_string(h.first_unsorted_panel) +
                                         ": block columns not strictly increasing");
        if (h.past_end) return fail(SPC5_EINVAL, "set mask bit maps past the last column");
    }
    return SPC5_OK;
}

// Chunk boundaries: a target every `cb` blocks snapped back to the start of
// the panel holding it, plus -- inside panels longer than kSplit blocks -- the
// GLOBAL multiples of kSplit (so a long panel is cut where its own position
// says, independent of cb, shards and ranges).  Fills chunk_b/v/p (+sentinels),
// the split-chunk list and the carry slots.
static int build_chunks(Matrix &m, int64_t cb, int64_t ppc, cudaStream_t st) {
    Plan &P = m.plan;
    const int64_t nb = m.num_blocks, np = m.num_panels;
    // ppc > 0: panel-count targets; ppc < 0: exact block multiples (LBR); 0: snapped block targets
    const int64_t num_targets = ppc > 0 ? cdiv(np, ppc)
                                : ppc < 0 ? (m.block_base + nb - 1) / cb - m.block_base / cb + 1
                                          : cdiv(nb, cb);
    int64_t *split_counts = nullptr;
    SPC5_TRY(dev_alloc(&split_counts, (size_t)np));
    split_count_kernel<<<(unsigned)cdiv(np, 256), 256, 0, st>>>(np, m.rowptr, m.block_base,
                                                                 P.split_len, split_counts);
    int64_t *split_incl = nullptr;
    SPC5_TRY(dev_alloc(&split_incl, (size_t)np));
    SPC5_TRY(scan_inclusive_i64(split_counts, split_incl, np, st));
    int64_t num_forced = 0;
    SPC5_CUDA(cudaMemcpyAsync(&num_forced, split_incl + np - 1, sizeof(int64_t),
                              cudaMemcpyDeviceToHost, st));
    SPC5_CUDA(cudaStreamSynchronize(st));
    const int64_t ncand = num_targets + num_forced;
    int64_t *cand = nullptr, *sorted = nullptr;
    SPC5_TRY(dev_alloc(&cand, (size_t)ncand));
    SPC5_TRY(dev_alloc(&sorted, (size_t)ncand + 1));
    if (ppc < 0)
        targets_exact_kernel<<<(unsigned)cdiv(num_targets, 256), 256, 0, st>>>(
            nb, m.block_base, cb, num_targets, cand);
    else if (ppc)
        targets_panels_kernel<<<(unsigned)cdiv(num_targets, 256), 256, 0, st>>>(
            np, m.rowptr, ppc, num_targets, cand);
    else
        targets_kernel<<<(unsigned)cdiv(num_targets, 256), 256, 0, st>>>(np, m.rowptr, cb,
                                                                          num_targets, cand);
    if (num_forced)
        split_fill_kernel<<<(unsigned)cdiv(np, 256), 256, 0, st>>>(np, m.rowptr, m.block_base,
                                                                    P.split_len, split_incl,
                                                                    cand + num_targets);
    SPC5_CUDA(cudaGetLastError());
    {
        size_t bytes = 0;
        SPC5_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, bytes, cand, sorted, ncand, 0, 64, st));
        void *tmp = nullptr;
        SPC5_TRY(dev_alloc(&tmp, bytes));
        SPC5_CUDA(cub::DeviceRadixSort::SortKeys(tmp, bytes, cand, sorted, ncand, 0, 64, st));
        SPC5_CUDA(cudaStreamSynchronize(st));
        dev_free(tmp);
    }
    int64_t *d_nuniq = nullptr;
    SPC5_TRY(dev_alloc(&d_nuniq, 1));
    SPC5_TRY(dev_alloc(&P.chunk_b, (size_t)ncand + 1));
    {
        size_t bytes = 0;
        SPC5_CUDA(cub::DeviceSelect::Unique(nullptr, bytes, sorted, P.chunk_b, d_nuniq, ncand, st));
        void *tmp = nullptr;
        SPC5_TRY(dev_alloc(&tmp, bytes));
        SPC5_CUDA(cub::DeviceSelect::Unique(tmp, bytes, sorted, P.chunk_b, d_nuniq, ncand, st));
        SPC5_CUDA(cudaMemcpyAsync(&P.num_chunks, d_nuniq, sizeof(int64_t), cudaMemcpyDeviceToHost,
                                  st));
        SPC5_CUDA(cudaStreamSynchronize(st));
        dev_free(tmp);
    }
    dev_free(d_nuniq);
    dev_free(cand);
    dev_free(sorted);
    dev_free(split_counts);
    dev_free(split_incl);
    const int64_t nc = P.num_chunks;
    SPC5_CUDA(cudaMemcpyAsync(P.chunk_b + nc, &nb, sizeof(int64_t), cudaMemcpyHostToDevice, st));
    SPC5_TRY(dev_alloc(&P.chunk_v, (size_t)nc + 1));
    SPC5_TRY(dev_alloc(&P.chunk_p, (size_t)nc + 1));
    SPC5_CUDA(cudaMemcpyAsync(P.chunk_v + nc, &m.nnz, sizeof(int64_t), cudaMemcpyHostToDevice, st));
    SPC5_CUDA(cudaMemcpyAsync(P.chunk_p + nc, &m.num_panels, sizeof(int64_t),
                              cudaMemcpyHostToDevice, st));
    uint8_t *split_flag = nullptr;
    SPC5_TRY(dev_alloc(&split_flag, (size_t)nc));
    chunk_desc_kernel<<<(unsigned)std::min<int64_t>(cdiv(nc, 8), 148 * 32), 256, 0, st>>>(
        nc, np, m.r, m.vs, m.rowptr, m.masks, P.tile_prefix, P.chunk_b, P.chunk_v, P.chunk_p,
        split_flag);
    SPC5_CUDA(cudaGetLastError());
    SPC5_TRY(dev_alloc(&P.split_chunks, (size_t)nc));
    SPC5_TRY(select_flagged(split_flag, nc, P.split_chunks, &P.num_split, st));
    dev_free(split_flag);
    if (P.num_split) SPC5_TRY(dev_alloc(&P.carry, (size_t)nc * m.r));
    P.h_chunk_b = new int64_t[nc + 1];
    SPC5_CUDA(cudaMemcpyAsync(P.h_chunk_b, P.chunk_b, sizeof(int64_t) * (nc + 1),
                              cudaMemcpyDeviceToHost, st));
    SPC5_CUDA(cudaStreamSynchronize(st));
    return SPC5_OK;
}

static void free_chunks(Plan &P) {
    dev_free(P.chunk_b);
    dev_free(P.chunk_v);
    dev_free(P.chunk_p);
    dev_free(P.split_chunks);
    dev_free(P.carry);
    delete[] P.h_chunk_b;
    P.chunk_b = P.chunk_v = P.chunk_p = P.split_chunks = nullptr;
    P.carry = nullptr;
    P.h_chunk_b = nullptr;
    P.num_chunks = P.num_split = 0;
}

int build_plan(Matrix &m, bool validate, cudaStream_t st) {
    if (m.plan.built) return SPC5_OK;
    Plan &P = m.plan;
    const int64_t nb = m.num_blocks, np = m.num_panels;
    if (validate) {
        // the checks the reference kernels perform implicitly
        int64_t first = 0, last = 0;
        SPC5_TRY(rowptr_ends(m, &first, &last, st));
        CheckOut h;
        SPC5_TRY(run_checks(m, &h, st));
        if (h.rowptr_bad || first != 0 || last != nb)
            return fail(SPC5_EINVAL, "block_rowptr must be non-decreasing from 0 to num_blocks");
        if (h.bits_beyond) return fail(SPC5_EINVAL, "mask has bits beyond the vs lanes");
        if ((int64_t)h.popc != m.nnz)
            return fail(SPC5_ECURSOR, "value cursor ended at " + std::to_string(h.popc) +
                                          ", expected " + std::to_string(m.nnz));
        if (h.past_end)
            return fail(SPC5_EINDEX, "active lane past end of x (mask bit maps past the last column)");
    }
    // popcount prefix per tile
    P.num_tiles = cdiv(nb, kTile);
    SPC5_TRY(dev_alloc(&P.tile_prefix, (size_t)P.num_tiles + 1));
    SPC5_CUDA(cudaMemsetAsync(P.tile_prefix, 0, sizeof(int64_t) * (P.num_tiles + 1), st));
    if (P.num_tiles) {
        int64_t *sums = nullptr;
        SPC5_TRY(dev_alloc(&sums, (size_t)P.num_tiles));
        tile_sums_kernel<<<(unsigned)std::min<int64_t>(cdiv(P.num_tiles, 8), 148 * 32), 256, 0,
                           st>>>(nb, m.r, m.vs, m.masks, P.num_tiles, sums);
        SPC5_CUDA(cudaGetLastError());
        SPC5_TRY(scan_inclusive_i64(sums, P.tile_prefix + 1, P.num_tiles, st));
        SPC5_CUDA(cudaStreamSynchronize(st));
        dev_free(sums);
    }
    // empty panels (zeroed by the SpMV kernel in y = A.x mode)
    if (np) {
        uint8_t *flags = nullptr;
        SPC5_TRY(dev_alloc(&flags, (size_t)np));
        empty_flag_kernel<<<(unsigned)cdiv(np, 256), 256, 0, st>>>(np, m.rowptr, flags);
        SPC5_TRY(dev_alloc(&P.empty_panels, (size_t)np));
        SPC5_TRY(select_flagged(flags, np, P.empty_panels, &P.num_empty, st));
        dev_free(flags);
    }
    if (nb == 0) {
        P.num_chunks = 0;
        P.h_chunk_b = new int64_t[1]{0};
        P.built = true;
        return SPC5_OK;
    }
    // Long panels are cut every split_len blocks (at global multiples) with
    // split_len the largest power of two <= 512 whose fullest window of
    // split_len blocks fits 6 KB; chunks = ring slots, the largest target size
    // whose worst chunk fits the slot target.
    {
        unsigned long long *d_mx = nullptr;
        SPC5_TRY(dev_alloc(&d_mx, 1));
        const int64_t per_block = 4 + m.r * m.mask_bytes();
        int64_t win_cap = 6 * 1024;  // bytes of the fullest split window (knob SPC5_WIN_KB)
        if (const char *e = getenv("SPC5_WIN_KB")) win_cap = std::max(1, atoi(e)) * 1024;
        // candidates: powers of two and their 3/4 (a panel of 85 blocks is
        // not cut at 96; any integer works for the global-multiple rule)
        static const int64_t kSl[] = {512, 384, 256, 192, 128, 96, 64, 48, 32, 24, 16,
                                      12, 8, 6, 4, 3, 2, 1};
        int64_t sl = 1;
        for (int64_t cand : kSl) {
            sl = cand;
            if (sl == 1) break;
            if (sl * per_block > win_cap) continue;
            unsigned long long h_mx = 0;
            SPC5_CUDA(cudaMemsetAsync(d_mx, 0, sizeof(unsigned long long), st));
            window_values_max_kernel<<<(unsigned)std::min<int64_t>(cdiv(cdiv(nb, sl) + 1, 8),
                                                                   148 * 16),
                                       256, 0, st>>>(nb, m.r, m.vs, m.masks, m.block_base, sl,
                                                     d_mx);
            SPC5_CUDA(cudaGetLastError());
            SPC5_CUDA(cudaMemcpyAsync(&h_mx, d_mx, sizeof(h_mx), cudaMemcpyDeviceToHost, st));
            SPC5_CUDA(cudaStreamSynchronize(st));
            if (sl * per_block + (int64_t)h_mx * m.value_bytes() <= win_cap) break;
        }
        dev_free(d_mx);
        P.split_len = sl;
    }
    // ring-slot size cap: 3 CTAs x 4 warps x 2 slots + 512 B each fit 228 KB
    int64_t slot_cap = 9472;  // (tuning knob SPC5_SLOT_KB)
    if (const char *e = getenv("SPC5_SLOT_KB")) slot_cap = std::max(1, atoi(e)) * 1024;
    // lane-per-panel chunks: the longest panel times the panel count may exceed
    // the chunk's blocks by lpr_bal/4 (knob SPC5_LPR_BAL, quarters)
    int lpr_bal = 4;
    if (const char *e = getenv("SPC5_LPR_BAL")) lpr_bal = std::max(4, atoi(e));
    // small matrices: chunks small enough that every resident warp of the
    // GPU (SMs x 12) gets about one, so a product is one chunk deep
    int64_t cb_max = 512;
    while (cb_max > 32 && nb / cb_max < (int64_t)m.sm_count * 12) cb_max >>= 1;
    // Chunk targets, largest first.  Regular matrices: k warp steps of panels
    // per chunk (k * 32/r panels, the whole chunk in full lane-per-panel-row
    // steps, no partly empty last step); accepted while no chunk exceeds the
    // average by 25 %.  Then block-count targets, powers of two.
    struct Target {
        int64_t cb, ppc;
    };
    std::vector<Target> targets;
    {
        const double avg = (double)nb / (double)std::max<int64_t>(np, 1);
        const int64_t lanes = 32 / m.r;
        // (at least one block per panel on average; candidates whose average
        // slot bytes already exceed the cap are not built)
        const double per_blk = 4.0 + (double)m.r * m.mask_bytes() +
                               (double)m.value_bytes() * (double)m.nnz / (double)std::max<int64_t>(nb, 1);
        if (!getenv("SPC5_CB_POW2") && avg >= 1.0) {
            int64_t kmax = (int64_t)((double)cb_max / ((double)lanes * avg));
            while (kmax > 1 && (double)(kmax * lanes) * avg * per_blk > (double)slot_cap) --kmax;
            // at most 8 panel-count candidates (each is a full build_chunks
            // pass: bounded plan-build time on sparse matrices)
            for (int64_t k = kmax; k >= 1 && targets.size() < 8; --k) {
                targets.push_back({(int64_t)((double)(k * lanes) * avg), k * lanes});
                // k-1 full steps and a 7/8-full last one, when k full ones
                // just miss the slot (fp32 beta(2,16): 30 panels, not 16)
                if (k > 1 && lanes >= 8) {
                    const int64_t ppc = k * lanes - lanes / 8;
                    targets.push_back({(int64_t)((double)ppc * avg), ppc});
                }
            }
        }
        // block-count targets: powers of two; for r = 1 also their 3/4 (config
        // 3 beta(1,16): 384-block chunks 392 us, 512: 483 us; for r > 1 the
        // 3/4 steps measured slower)
        for (int64_t cb = cb_max; cb >= 1; cb >>= 1) {
            targets.push_back({cb, 0});
            if (m.r == 1 && !getenv("SPC5_CB_POW2") && cb >= 8) targets.push_back({cb * 3 / 4, 0});
        }
        if (const char *e = getenv("SPC5_CB")) targets = {{std::max(1, atoi(e)), 0}};  // tuning
    }
    // Lane-per-block-row rounds (LBR) for matrices of long panels whose blocks
    // are well filled but whose block ROWS are mostly empty (FEM beta(8,8): 3x3
    // dense sub-blocks, 7.5 values per block, 0.94 per block row; >= 24 blocks
    // per non-empty panel): lane-per-panel-row lanes would mostly visit blocks
    // their row does not touch.  Exact chunk cuts every 32k blocks, no
    // lane-per-panel / value-range chunks, slots <= 6 KB (64 blocks of
    // beta(8,8): 352 us on config 4, 96 blocks 412 us).  Knob SPC5_LBR=0|1.
    {
        const double vpb = (double)m.nnz / (double)std::max<int64_t>(nb, 1);
        const double bpp = (double)nb / (double)std::max<int64_t>(np - P.num_empty, 1);
        P.lbr = vpb >= 2.0 && bpp >= 24.0 && vpb < 1.25 * m.r;
        if (const char *e = getenv("SPC5_LBR")) P.lbr = atoi(e) != 0;
    }
    if (P.lbr) {
        const double per_blk = 4.0 + (double)m.r * m.mask_bytes() +
                               (double)m.value_bytes() * (double)m.nnz / (double)std::max<int64_t>(nb, 1);
        slot_cap = std::min<int64_t>(slot_cap, 6144);
        int64_t k = std::max<int64_t>(1, std::min<int64_t>(cb_max / 32, (int64_t)((double)slot_cap / per_blk / 32.0) + 1));
        targets.clear();
        for (; k >= 1; --k) targets.push_back({32 * k, -1});
        if (const char *e = getenv("SPC5_CB")) targets = {{std::max(32, atoi(e) / 32 * 32), -1}};
        P.split_len = INT64_MAX / 4;  // exact cuts bound every chunk: no forced splits
    }
    if (const char *e = getenv("SPC5_SLOT_B")) slot_cap = std::max(1024, atoi(e));
    // run plans (knob SPC5_NO_RUN=1 keeps the general bit walk): is every row
    // mask one contiguous run of bits?
    bool masks_runs = false;
    if (!getenv("SPC5_NO_RUN")) {
        int *d_bad = nullptr, h_bad = 0;
        SPC5_TRY(dev_alloc(&d_bad, 1));
        SPC5_CUDA(cudaMemsetAsync(d_bad, 0, sizeof(int), st));
        runs_kernel<<<(unsigned)std::min<int64_t>(cdiv(nb * m.r, 1024), 148 * 16), 256, 0, st>>>(
            nb * m.r, m.vs, m.masks, d_bad);
        SPC5_CUDA(cudaGetLastError());
        SPC5_CUDA(cudaMemcpyAsync(&h_bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, st));
        SPC5_CUDA(cudaStreamSynchronize(st));
        dev_free(d_bad);
        masks_runs = h_bad == 0;
    }
    // The run-plan kernel of fp32 beta(2,16) needs 119 registers: with slots of
    // <= 7,040 B a fourth CTA fits each SM (16 warps instead of 12): 400^3
    // 1,866 -> 1,707 us, 128^3 63.6 -> 59.0 us.  (beta(4,16) gains nothing,
    // beta(8,16) and the f64 kernels keep 3 CTAs by their registers and only
    // lose chunk size: 400^3 beta(1,8) 2,766 -> 4,914 us.)
    int64_t lpp_cap = slot_cap;
    if (masks_runs && m.value_bytes() == 4 && m.r == 2 && !getenv("SPC5_SLOT_B") &&
        !getenv("SPC5_SLOT_KB"))
        lpp_cap = std::min<int64_t>(lpp_cap, 7040);
    // irregular r = 1 matrices (block-count targets): slots <= 8 KB
    int64_t irr_cap = m.r == 1 ? std::min<int64_t>(slot_cap, 8192) : slot_cap;
    if (const char *e = getenv("SPC5_SLOT_B_IRR")) irr_cap = std::max(1024, atoi(e));
    // flat value-range chunks (knob SPC5_FVR: 0 off, 1 scan chunks of r >= 2
    // and sparse lane-per-panel ones, 2 + scan chunks of r = 1, 3 every chunk
    // without empty panels;
    // SPC5_FVR_DENSE: values per block row below which LPP chunks go FVR, in quarters)
    int fvr_mode = 1;
    if (const char *e = getenv("SPC5_FVR")) fvr_mode = atoi(e);
    if (const char *e = getenv("SPC5_FVR_DENSE")) {
        const int q = atoi(e);
        SPC5_CUDA(cudaMemcpyToSymbol(fvr_dense_q, &q, sizeof(int)));
    }
    for (size_t ti = 0;; ++ti) {
        const int64_t cb = targets[ti].cb, ppc = targets[ti].ppc;
        SPC5_TRY(build_chunks(m, cb, ppc, st));
        SPC5_TRY(dev_alloc(&P.chunk_flags, (size_t)P.num_chunks + 1));
        chunk_flags_kernel<<<(unsigned)cdiv(P.num_chunks, 256), 256, 0, st>>>(
            P.num_chunks, nb, np, m.r, P.chunk_b, P.chunk_p, m.rowptr, P.empty_panels,
            P.num_empty,
            (P.lbr || getenv("SPC5_NO_LPR")) ? -1 : (getenv("SPC5_LPR_SPLIT") ? 1 : 0), lpr_bal, 4,
            P.lbr ? 0 : fvr_mode, kLppMinLanes, P.chunk_v, P.chunk_flags);
        SPC5_CUDA(cudaGetLastError());
        unsigned long long *d_st = nullptr, h_st[5] = {0, 0, 0, 0, 0};
        SPC5_TRY(dev_alloc(&d_st, 5));
        SPC5_CUDA(cudaMemsetAsync(d_st, 0, 5 * sizeof(unsigned long long), st));
        chunk_stats_kernel<<<(unsigned)cdiv(P.num_chunks, 256), 256, 0, st>>>(
            P.num_chunks, P.chunk_b, P.chunk_v, d_st);
        lpp_panels_kernel<<<(unsigned)cdiv(P.num_chunks, 256), 256, 0, st>>>(
            P.num_chunks, P.chunk_p, P.chunk_flags, d_st + 2, d_st + 3, d_st + 4);
        SPC5_CUDA(cudaGetLastError());
        SPC5_CUDA(cudaMemcpyAsync(h_st, d_st, sizeof(h_st), cudaMemcpyDeviceToHost, st));
        SPC5_CUDA(cudaStreamSynchronize(st));
        dev_free(d_st);
        P.max_chunk_blocks = (int64_t)h_st[0];
        P.max_chunk_values = (int64_t)h_st[1];
        P.max_lpp_panels = (int64_t)h_st[2];
        P.num_fvr = (int64_t)h_st[3];
        P.num_lpp = (int64_t)h_st[4];
        // a plan that is mostly lane-per-panel chunks (regular stencil-like
        // matrices) keeps its few scan chunks in balanced-lane-range mode:
        // the FVR code would otherwise be compiled into its kernel
        if (fvr_mode < 2 && P.num_fvr && P.num_lpp * 2 > P.num_chunks) {
            unsigned long long *d_cl = nullptr, h_cl = 0;
            SPC5_TRY(dev_alloc(&d_cl, 1));
            SPC5_CUDA(cudaMemsetAsync(d_cl, 0, sizeof(unsigned long long), st));
            unfvr_kernel<<<(unsigned)cdiv(P.num_chunks, 256), 256, 0, st>>>(P.num_chunks,
                                                                            P.chunk_flags, d_cl);
            SPC5_CUDA(cudaGetLastError());
            SPC5_CUDA(cudaMemcpyAsync(&h_cl, d_cl, sizeof(h_cl), cudaMemcpyDeviceToHost, st));
            SPC5_CUDA(cudaStreamSynchronize(st));
            dev_free(d_cl);
            P.num_fvr -= (int64_t)h_cl;
        }
        // A plan that is lane-per-panel-row but for a few chunks (panels of
        // uneven length at grid faces: 796 of 2 M chunks on the 400^3 beta(8,8)
        // stencil, 68 of 35 k on the 128^3 beta(2,16) one) takes those chunks as
        // lane-per-panel-row too, balance rule and lane minimum waived: the
        // whole plan then runs the LPP-only kernel, and the run-plan variant
        // when its masks allow (400^3 beta(8,8) 3,335 -> 3,261 us).
        if (!P.lbr && P.num_lpp < P.num_chunks && P.num_lpp * 50 >= P.num_chunks * 49 &&
            !getenv("SPC5_NO_LPR") && !getenv("SPC5_NO_LPP_RELAX")) {
            chunk_flags_kernel<<<(unsigned)cdiv(P.num_chunks, 256), 256, 0, st>>>(
                P.num_chunks, nb, np, m.r, P.chunk_b, P.chunk_p, m.rowptr, P.empty_panels,
                P.num_empty, getenv("SPC5_LPR_SPLIT") ? 1 : 0, 1 << 20, 4, 0, 1, P.chunk_v,
                P.chunk_flags);
            unsigned long long *d_st2 = nullptr, h_st2[3] = {0, 0, 0};
            SPC5_TRY(dev_alloc(&d_st2, 3));
            SPC5_CUDA(cudaMemsetAsync(d_st2, 0, 3 * sizeof(unsigned long long), st));
            lpp_panels_kernel<<<(unsigned)cdiv(P.num_chunks, 256), 256, 0, st>>>(
                P.num_chunks, P.chunk_p, P.chunk_flags, d_st2, d_st2 + 1, d_st2 + 2);
            SPC5_CUDA(cudaGetLastError());
            SPC5_CUDA(cudaMemcpyAsync(h_st2, d_st2, sizeof(h_st2), cudaMemcpyDeviceToHost, st));
            SPC5_CUDA(cudaStreamSynchronize(st));
            dev_free(d_st2);
            P.max_lpp_panels = (int64_t)h_st2[0];
            P.num_fvr = (int64_t)h_st2[1];
            P.num_lpp = (int64_t)h_st2[2];
        }
        P.chunk_target = cb;
        auto a16 = [](int64_t v) { return (v + 15) / 16 * 16; };
        const int64_t mb = P.max_chunk_blocks;
        // slot: metadata blob (header, words, records), then the matrix arrays
        P.lay_rp = 64 + a16((mb / 32 + 2) * 4 + 32);
        // records: panel records (lane-per-panel chunks) or 32 lane records
        P.lay_col = P.lay_rp + a16(std::max<int64_t>(P.max_lpp_panels + 1, 32) * 4 + 32);
        P.lay_mask = P.lay_col + a16(mb * 4 + 32);
        // + slack: lane-per-panel-row steps (U <= 18 blocks for r = 8, <= 9
        // otherwise) load up to U-1 blocks past a lane's range, masked off
        // afterwards, without bounds checks
        const int64_t lb = m.r * m.mask_bytes();
        P.lay_val = P.lay_mask + a16(mb * lb + std::max<int64_t>(32, ((m.r == 8 ? 18 : 9) - 1) * lb));
        P.slot_bytes = (int)((P.lay_val + a16(P.max_chunk_values * m.value_bytes() + 32) + 127) /
                             128 * 128);
        const bool regular = ppc <= 0 || P.max_chunk_blocks * 4 <= cb * 5;
        // FVR kernels of r = 8 keep their row sums in shared memory (r*256 B
        // per warp = r*128 B per ring slot): smaller slots keep 3 CTAs per SM
        const int64_t cap = (ppc > 0 ? lpp_cap : ppc < 0 ? slot_cap : irr_cap) -
                            (P.num_fvr && m.r == 8 ? m.r * 128 : 0);
        if (!regular) {  // fewer panels per chunk only averages worse: go to block targets
            while (ti + 1 < targets.size() && targets[ti + 1].ppc > 0) ++ti;
        }
        if (regular && (P.slot_bytes <= cap || cb == 1 || ti + 1 >= targets.size())) break;
        if (regular && cb <= 32 && P.slot_bytes <= 14 * 1024) break;
        free_chunks(P);
        dev_free(P.chunk_flags);
        P.chunk_flags = nullptr;
    }
    if (P.slot_bytes > 14 * 1024)
        return fail(SPC5_EINVAL, "a chunk of this matrix does not fit the shared-memory ring");
    P.runs = masks_runs && P.num_lpp == P.num_chunks;
    // panel-start bitmap
    const int off32 = (int)(((m.block_base % 32) + 32) % 32);
    const int64_t ng = cdiv(nb + off32, 32);
    P.num_granules = ng;
    SPC5_TRY(dev_alloc(&P.pstart_bits, (size_t)ng + 4));
    SPC5_CUDA(cudaMemsetAsync(P.pstart_bits, 0, sizeof(uint32_t) * (ng + 4), st));
    pstart_bits_kernel<<<(unsigned)cdiv(np, 256), 256, 0, st>>>(np, m.rowptr, off32,
                                                                 P.pstart_bits);
    SPC5_CUDA(cudaGetLastError());
    // per-chunk metadata blobs and issue records
    const int64_t nc = P.num_chunks;
    if (nc) {
        int64_t *size16 = nullptr, *off16 = nullptr;
        SPC5_TRY(dev_alloc(&size16, (size_t)nc));
        SPC5_TRY(dev_alloc(&off16, (size_t)nc));
        blob_size_kernel<<<(unsigned)cdiv(nc, 256), 256, 0, st>>>(nc, P.chunk_b, P.chunk_p,
                                                                   P.chunk_flags, off32, size16);
        SPC5_CUDA(cudaGetLastError());
        SPC5_TRY(scan_inclusive_i64(size16, off16, nc, st));
        int64_t total16 = 0;
        SPC5_CUDA(cudaMemcpyAsync(&total16, off16 + nc - 1, sizeof(int64_t),
                                  cudaMemcpyDeviceToHost, st));
        SPC5_CUDA(cudaStreamSynchronize(st));
        if (total16 >= (int64_t(1) << 32)) return fail(SPC5_ENOMEM, "chunk metadata too large");
        SPC5_TRY(dev_alloc(&P.blob, (size_t)total16 * 16));
        blob_fill_kernel<<<(unsigned)std::min<int64_t>(cdiv(nc, 8), 65535), 256, 0, st>>>(
            nc, m.r, m.vs, off32, P.chunk_b, P.chunk_v, P.chunk_p, P.chunk_flags, m.rowptr,
            m.masks, P.pstart_bits, off16, P.blob);
        SPC5_CUDA(cudaGetLastError());
        SPC5_TRY(dev_alloc(&P.issue_rec, (size_t)nc * 2));
        issue_rec_kernel<<<(unsigned)cdiv(nc, 256), 256, 0, st>>>(
            nc, m.r * m.mask_bytes(), m.value_bytes(), P.chunk_b, P.chunk_v, off16, P.issue_rec);
        SPC5_CUDA(cudaGetLastError());
        // (not for f64 beta(8,8): issue-bound there, 3482 -> 3560 us on the 400^3 stencil)
        if (!getenv("SPC5_NO_XPREFETCH") && !(m.r == 8 && m.value_bytes() == 8)) {
            int64_t *xmax = nullptr;
            SPC5_TRY(dev_alloc(&xmax, (size_t)nc));
            chunk_xmax_kernel<<<(unsigned)std::min<int64_t>(cdiv(nc, 8), 148 * 32), 256, 0, st>>>(
                nc, P.chunk_b, m.colidx, m.vs, m.num_cols, xmax);
            xedge_kernel<<<(unsigned)cdiv(nc, 256), 256, 0, st>>>(nc, xmax, m.value_bytes(),
                                                                  P.issue_rec);
            SPC5_CUDA(cudaGetLastError());
            SPC5_CUDA(cudaStreamSynchronize(st));
            dev_free(xmax);
        }
        SPC5_CUDA(cudaStreamSynchronize(st));
        dev_free(size16);
        dev_free(off16);
    }
    if (getenv("SPC5_PLAN_DEBUG")) {  // diagnostics: chunk modes and slot shape
        std::vector<uint8_t> f((size_t)nc);
        if (nc)
            SPC5_CUDA(cudaMemcpy(f.data(), P.chunk_flags, (size_t)nc, cudaMemcpyDeviceToHost));
        int64_t cnt[8] = {0};
        for (uint8_t v : f) {
            ++cnt[v & 7];
        }
        fprintf(stderr,
                "spc5 plan: r=%d vs=%d lbr=%d runs=%d nb=%lld np=%lld chunks=%lld target=%lld split_len=%lld "
                "slot=%d B (rec@%lld col@%lld mask@%lld val@%lld) max_blocks=%lld max_values=%lld "
                "max_lpp_panels=%lld split=%lld empty=%lld | flags: scan=%lld mid=%lld "
                "empty=%lld lpr=%lld other=%lld\n",
                m.r, m.vs, (int)P.lbr, (int)P.runs, (long long)nb, (long long)np, (long long)nc,
                (long long)P.chunk_target, (long long)P.split_len, P.slot_bytes,
                (long long)P.lay_rp, (long long)P.lay_col, (long long)P.lay_mask,
                (long long)P.lay_val, (long long)P.max_chunk_blocks,
                (long long)P.max_chunk_values, (long long)P.max_lpp_panels,
                (long long)P.num_split, (long long)P.num_empty, (long long)cnt[0],
                (long long)(cnt[1] + cnt[3]), (long long)(cnt[2]), (long long)cnt[4],
                (long long)(nc - cnt[0] - cnt[1] - cnt[3] - cnt[2] - cnt[4]));
    }
    P.built = true;
    return SPC5_OK;
}

// stage s of the host pipeline reads x columns < need[s]: per block, col + vs
// (clipped), max over the stage's blocks
__global__ void stage_need_kernel(int64_t nb, const uint32_t *__restrict__ colidx, int vs,
                                  int64_t num_cols, const int64_t *__restrict__ bnd, int K,
                                  unsigned long long *need) {
    int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int best = -1, bs = 0;
    for (; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
        int s = 0;
        while (s + 1 < K && b >= bnd[s + 1]) ++s;
        const int64_t e = min((int64_t)colidx[b] + vs, num_cols);
        if (s != bs && best >= 0) {
            atomicMax(need + bs, (unsigned long long)best);
            best = -1;
        }
        bs = s;
        best = max(best, (int)e);
    }
    if (best >= 0) atomicMax(need + bs, (unsigned long long)best);
}

int host_stages(const Matrix &m, int K, int64_t *p, int64_t *b, int64_t *need, cudaStream_t st) {
    std::vector<int64_t> ranges(2 * K);
    SPC5_TRY(partition_by_nnz(m, K, ranges.data(), st));
    for (int k = 0; k < K; ++k) p[k] = ranges[2 * k];
    p[K] = m.num_panels;
    for (int k = 0; k <= K; ++k)
        SPC5_CUDA(cudaMemcpyAsync(b + k, m.rowptr + p[k], sizeof(int64_t), cudaMemcpyDeviceToHost,
                                  st));
    SPC5_CUDA(cudaStreamSynchronize(st));
    int64_t *d_bnd = nullptr;
    unsigned long long *d_need = nullptr;
    SPC5_TRY(dev_alloc(&d_bnd, (size_t)K + 1));
    SPC5_TRY(dev_alloc(&d_need, (size_t)K));
    SPC5_CUDA(cudaMemcpyAsync(d_bnd, b, sizeof(int64_t) * (K + 1), cudaMemcpyHostToDevice, st));
    SPC5_CUDA(cudaMemsetAsync(d_need, 0, sizeof(unsigned long long) * K, st));
    if (m.num_blocks)
        stage_need_kernel<<<(unsigned)std::min<int64_t>(cdiv(m.num_blocks, 256), 148 * 16), 256, 0,
                            st>>>(m.num_blocks, m.colidx, m.vs, m.num_cols, d_bnd, K, d_need);
    SPC5_CUDA(cudaGetLastError());
    std::vector<unsigned long long> h(K);
    SPC5_CUDA(cudaMemcpyAsync(h.data(), d_need, sizeof(unsigned long long) * K,
                              cudaMemcpyDeviceToHost, st));
    SPC5_CUDA(cudaStreamSynchronize(st));
    dev_free(d_bnd);
    dev_free(d_need);
    int64_t run = 0;  // prefix max: stage k may start once x[0, need[k]) has landed
    for (int k = 0; k < K; ++k) {
        run = std::max<int64_t>(run, (int64_t)h[k]);
        need[k] = run;
    }
    return SPC5_OK;
}

int partition_by_nnz(const Matrix &m, int workers, int64_t *h_ranges, cudaStream_t st) {
    if (workers < 1) return fail(SPC5_EINVAL, "workers must be >= 1");
    std::vector<int64_t> bounds(workers + 1, 0);
    bounds[workers] = m.num_panels;
    if (workers > 1 && m.num_panels > 0) {
        int64_t *d = nullptr;
        SPC5_TRY(dev_alloc(&d, (size_t)workers + 1));
        const int64_t threads = (int64_t)(workers - 1) * 32;
        partition_kernel<<<(unsigned)cdiv(threads, 128), 128, 0, st>>>(
            m.num_panels, m.r, m.vs, m.rowptr, m.masks, m.plan.tile_prefix, m.plan.num_tiles,
            workers, d);
        SPC5_CUDA(cudaGetLastError());
        SPC5_CUDA(cudaMemcpyAsync(bounds.data() + 1, d + 1, sizeof(int64_t) * (workers - 1),
                                  cudaMemcpyDeviceToHost, st));
        SPC5_CUDA(cudaStreamSynchronize(st));
        dev_free(d);
    }
    for (int k = 0; k < workers; ++k) {
        h_ranges[2 * k] = bounds[k];
        h_ranges[2 * k + 1] = bounds[k + 1];
    }
    note_launches(workers > 1 && m.num_panels > 0 ? 1 : 0);
    return SPC5_OK;
}

int block_value_offsets(const Matrix &m, int64_t *d_offsets, cudaStream_t st) {
    SPC5_CUDA(cudaMemsetAsync(d_offsets, 0, sizeof(int64_t), st));
    if (m.num_blocks == 0) return SPC5_OK;
    BlockPopc f{m.masks, m.r, m.vs};
    thrust::transform_iterator<BlockPopc, thrust::counting_iterator<int64_t>> it(
        thrust::counting_iterator<int64_t>(0), f);
    size_t bytes = 0;
    SPC5_CUDA(cub::DeviceScan::InclusiveSum(nullptr, bytes, it, d_offsets + 1, m.num_blocks, st));
    void *tmp = nullptr;
    SPC5_TRY(dev_alloc(&tmp, bytes));
    SPC5_CUDA(cub::DeviceScan::InclusiveSum(tmp, bytes, it, d_offsets + 1, m.num_blocks, st));
    SPC5_CUDA(cudaStreamSynchronize(st));
    dev_free(tmp);
    return SPC5_OK;
}

}  // namespace spc5
