// spmv.cu -- K2 host side: argument block, panel-range resolution and the
// dispatch of y (+)= A.x to the kernel instance of the matrix's (precision,
// mask width, r).  The kernel templates live in spmv_kernel.cuh; every
// (T, MT, R) combination is compiled in its own translation unit
// (spmv_inst_*.cu) so the build runs in parallel.
// Replaces spmv_spc5_scalar / spmv_spc5_vector (kernels.py:121-230).
#include "spmv_kernel.cuh"

namespace spc5 {

#define SPC5_K2_DECL(NAME, T, MT, R) int NAME(const Matrix &m, const SpmvArgs &a, cudaStream_t st);
SPC5_K2_INSTANCES(SPC5_K2_DECL)
#undef SPC5_K2_DECL

namespace {

constexpr unsigned kFullMask = 0xffffffffu;

// Number of entries of the sorted a[0, n) that are <= v (LE) or < v: a
// 32-ary search by one warp, ~log32(n) rounds of one probe per lane.
template <bool LE>
__device__ int64_t warp_count(const int64_t *__restrict__ a, int64_t n, int64_t v, int lane) {
    int64_t lo = 0, hi = n;  // the count is in [lo, hi]
    while (hi - lo > 32) {
        const int64_t step = (hi - lo + 31) / 32;
        const int64_t i = lo + (int64_t)(lane + 1) * step - 1;
        const bool ok = i < hi && (LE ? a[i] <= v : a[i] < v);
        const int c = __popc(__ballot_sync(kFullMask, ok));  // probes that hold form a prefix
        const int64_t nlo = min(hi, lo + (int64_t)c * step);
        hi = min(hi, lo + (int64_t)(c + 1) * step - 1);
        lo = nlo;
    }
    const int64_t i = lo + lane;
    const bool ok = i < hi && (LE ? a[i] <= v : a[i] < v);
    return lo + __popc(__ballot_sync(kFullMask, ok));
}

// Range products without a host round trip: the blocks of panels
// [p_lo, p_hi) and the chunks holding them (as launch_spmv computes on the
// host when the caller knows the block bounds).
__global__ void range_kernel(const int64_t *__restrict__ rowptr, const int64_t *__restrict__ chunk_b,
                             int64_t nc, int64_t p_lo, int64_t p_hi, int64_t *out) {
    const int lane = threadIdx.x & 31;
    const int64_t blo = rowptr[p_lo], bhi = rowptr[p_hi];
    int64_t clo = warp_count<true>(chunk_b, nc, blo, lane) - 1;
    if (clo < 0) clo = 0;
    int64_t chi = warp_count<false>(chunk_b, nc, bhi, lane);
    if (blo >= bhi) chi = clo;  // no blocks: only empty-panel zeroing
    if (lane == 0) {
        out[0] = blo;
        out[1] = bhi;
        out[2] = clo;
        out[3] = chi;
    }
}


template <int F64, int WIDE>
int dispatch_r(const Matrix &m, const SpmvArgs &a, cudaStream_t st);
#define SPC5_K2_CASE(F, W, SUF)                                             \
    template <>                                                              \
    int dispatch_r<F, W>(const Matrix &m, const SpmvArgs &a, cudaStream_t st) { \
        switch (m.r) {                                                       \
            case 1: return launch_k2_##SUF##_r1(m, a, st);                   \
            case 2: return launch_k2_##SUF##_r2(m, a, st);                   \
            case 4: return launch_k2_##SUF##_r4(m, a, st);                   \
            default: return launch_k2_##SUF##_r8(m, a, st);                  \
        }                                                                    \
    }
SPC5_K2_CASE(1, 0, f64_u8)
SPC5_K2_CASE(1, 1, f64_u16)
SPC5_K2_CASE(0, 0, f32_u8)
SPC5_K2_CASE(0, 1, f32_u16)
#undef SPC5_K2_CASE

}  // namespace

int launch_spmv(const Matrix &m, int64_t p_lo, int64_t p_hi, const void *x, void *y,
                int accumulate, cudaStream_t st, const Scratch &scratch, const Mirror *mirror,
                const int64_t *blk) {
    const Plan &P = m.plan;
    SpmvArgs a{};
    a.yscale = 1.0;
    if (mirror) {
        if (mirror->n < 0 || mirror->n > kMaxMirrors)
            return fail(SPC5_EINVAL, "at most 8 mirror buffers");
        a.nmirror = mirror->n;
        for (int i = 0; i < mirror->n; ++i) a.mirror[i] = mirror->ptr[i];
        a.mirror_row0 = mirror->row0;
        a.yscale = mirror->scale;
    }
    a.rowptr = m.rowptr;
    a.colidx = m.colidx;
    a.masks = m.masks;
    a.values = m.values;
    a.x = x;
    a.y = y;
    a.num_rows = m.num_rows;
    a.num_cols = m.num_cols;
#if SPC5_CHECKED
    // self-test of the checked build: a one-column x bound makes the first
    // gather past column 0 trap (tools/checked_build.sh expects the failure)
    if (getenv("SPC5_CHECKED_SELFTEST")) a.num_cols = 1;
#endif
    a.num_panels = m.num_panels;
    a.chunk_b = P.chunk_b;
    a.chunk_v = P.chunk_v;
    a.chunk_p = P.chunk_p;
    a.chunk_flags = P.chunk_flags;
    a.pstart_bits = P.pstart_bits;
    a.blob = P.blob;
    a.issue_rec = P.issue_rec;
    a.carry = scratch.carry;
    if (P.num_split && !a.carry) return fail(SPC5_EINVAL, "no carry scratch for this stream");
    a.empty_panels = P.empty_panels;
    a.num_empty = P.num_empty;
    a.off32 = (int)(((m.block_base % 32) + 32) % 32);
    a.accumulate = accumulate;
    a.lay_col = (uint32_t)P.lay_col;
    a.lay_mask = (uint32_t)P.lay_mask;
    a.lay_val = (uint32_t)P.lay_val;
    a.lay_bytes = (uint32_t)P.slot_bytes;
    a.p_lo = p_lo;
    a.p_hi = p_hi;
    if (p_lo == 0 && p_hi == m.num_panels) {
        a.c_lo = 0;
        a.c_hi = P.num_chunks;
        a.b_lo = 0;
        a.b_hi = m.num_blocks;
    } else {
        if (!blk && P.num_chunks) {
            // block and chunk bounds resolved on the device (no host sync;
            // capturable): the launch covers every chunk, warps past the
            // resolved range exit at once
            if (!scratch.range) return fail(SPC5_EINVAL, "no range scratch for this stream");
            range_kernel<<<1, 32, 0, st>>>(m.rowptr, P.chunk_b, P.num_chunks, p_lo, p_hi,
                                           scratch.range);
            SPC5_CUDA(cudaGetLastError());
            note_launches(1);
            a.range = scratch.range;
            a.c_lo = 0;
            a.c_hi = P.num_chunks;
            a.b_lo = 0;
            a.b_hi = m.num_blocks;
        } else if (blk) {  // block range known to the caller (host pipeline stages)
            const int64_t blo = blk[0], bhi = blk[1];
            a.b_lo = blo;
            a.b_hi = bhi;
            const int64_t *cb = P.h_chunk_b;
            const int64_t nc = P.num_chunks;
            a.c_lo = std::upper_bound(cb, cb + nc, blo) - cb - 1;
            if (a.c_lo < 0) a.c_lo = 0;
            a.c_hi = std::lower_bound(cb, cb + nc, bhi) - cb;
            if (blo >= bhi) a.c_hi = a.c_lo;  // no blocks: only empty-panel zeroing
        }
    }
    if (P.num_chunks == 0 || a.c_hi <= a.c_lo) {
        a.c_lo = a.c_hi = 0;
        a.range = nullptr;
        if (accumulate || a.num_empty == 0) {
            note_launches(0);
            return SPC5_OK;
        }
    }
    a.plain = !accumulate && a.nmirror == 0 && a.yscale == 1.0;
    a.x_prefetch = (reinterpret_cast<uintptr_t>(x) & 15) == 0;
    const bool f64 = m.precision == SPC5_F64;
    const bool wide = m.vs > 8;
    if (f64) return wide ? dispatch_r<1, 1>(m, a, st) : dispatch_r<1, 0>(m, a, st);
    return wide ? dispatch_r<0, 1>(m, a, st) : dispatch_r<0, 0>(m, a, st);
}

}  // namespace spc5
