// spmv.cu -- K2: y (+)= A.x over the SPC5 beta(r,vs) arrays on sm_100a.
//
// Replaces spmv_spc5_scalar / spmv_spc5_vector (kernels.py:121-230), i.e.
// Algorithm 1 of the paper re-mapped to a warp:
//
//  * lane-per-block: a warp walks its chunk in 32-block windows aligned to
//    GLOBAL block indices; lane l owns block w+l.  Its column start and its r
//    masks come in with one coalesced load each (r*mask_bytes <= 16 B).
//  * value offsets: popcount of the lane's masks + a warp inclusive scan
//    (5 shuffles) on top of the chunk's offset from the plan -- the
//    "value cursor" of kernels.py:211-212 in parallel form.
//  * panel of each block: one coalesced load of the next 32 block_rowptr
//    entries and a 5-step shuffle binary search (empty panels and >32 panel
//    ends per window take a global binary search).
//  * the lane walks its set bits (__ffs), multiplying packed values by x
//    (read-only path; x is the only re-read array and stays L2 resident) into
//    r per-row accumulators (fp64; products formed in the matrix precision).
//  * per-row reduction: a segmented warp scan over lanes of the same panel;
//    the segment tail writes y (or carries into the next window).  Chunks
//    that start inside a giant panel write their head segment to a carry slot
//    and a tiny fixup kernel adds those in chunk order.  Every panel is summed
//    in an order fixed by global block positions only, so results are
//    bitwise reproducible across runs, spmv_parallel ranges and GPU shards.
#include <algorithm>

#include "common.cuh"

namespace spc5 {
namespace {

struct SpmvArgs {
    const int64_t *rowptr;
    const uint32_t *colidx;
    const void *masks;
    const void *values;
    const void *x;
    void *y;
    int64_t num_rows, num_panels;
    const int64_t *chunk_b, *chunk_v, *chunk_p;
    int64_t c_lo, c_hi;  // chunk range
    int64_t b_lo, b_hi;  // compute-active block range
    int64_t p_lo, p_hi;  // panels whose rows may be written
    double *carry;
    const int64_t *empty_panels;
    int64_t num_empty;
    int base_mod;  // block_base mod 32
    int accumulate;
    // TMA stage plan
    const int64_t *stage_v, *stage_p;
    int stage_k;  // 32-block granules per stage
    int off32;    // block_base mod 32 (granule alignment)
    int rp_cap;   // staged rowptr entries per stage
    uint32_t lay_mask, lay_rp, lay_val, lay_bytes;  // slot layout (bytes)
};


template <typename T>
__device__ __forceinline__ double mul_acc(double acc, T v, T xv);
template <>
__device__ __forceinline__ double mul_acc<double>(double acc, double v, double xv) {
    return fma(v, xv, acc);
}
template <>
__device__ __forceinline__ double mul_acc<float>(double acc, float v, float xv) {
    return acc + (double)(v * xv);  // product rounded in f32, as the reference forms it
}

constexpr unsigned kFull = 0xffffffffu;

// ---- TMA (cp.async.bulk) + mbarrier helpers -------------------------------
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}
// 1-D bulk copy global -> shared, completion counted on `bar` (SASS: UBLKCP)
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes,
                                         uint64_t *bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1], %2, [%3], %4;" ::"r"(smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

// Exclusive prefix sum over the warp of a small count (< 2^NP) via bit-plane
// ballots: independent BALLOT/POPC pairs instead of a dependent shuffle chain.
template <int NP>
__device__ __forceinline__ void warp_prefix(int cnt, int lane, int &excl, int &total) {
    const unsigned lt = (1u << lane) - 1u;
    excl = 0;
    total = 0;
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        const unsigned bal = __ballot_sync(kFull, (cnt >> p) & 1);
        excl += __popc(bal & lt) << p;
        total += __popc(bal) << p;
    }
}

// One stage = the blocks [start, end) of a chunk that fall in one plan stage.
struct StageDesc {
    int64_t start, end;  // blocks
    int64_t v_s, v_e;    // values
    int64_t p_s, p_e;    // panel holding `start`, panel holding `end` (num_panels at nb)
};

__device__ __forceinline__ int64_t stage_of(int64_t b, int off32, int k) {
    return ((b + off32) >> 5) / k;
}

__device__ __forceinline__ StageDesc stage_desc(const SpmvArgs &a, int64_t c, int64_t j) {
    const int64_t cb0 = a.chunk_b[c], cb1 = a.chunk_b[c + 1];
    const int64_t g0 = j * a.stage_k, g1 = (j + 1) * a.stage_k;
    const int64_t s0 = g0 == 0 ? 0 : g0 * 32 - a.off32;
    const int64_t s1 = g1 * 32 - a.off32;
    StageDesc d;
    const bool first = s0 <= cb0, lastc = s1 >= cb1;
    d.start = first ? cb0 : s0;
    d.end = lastc ? cb1 : s1;
    d.v_s = first ? a.chunk_v[c] : a.stage_v[j];
    d.v_e = lastc ? a.chunk_v[c + 1] : a.stage_v[j + 1];
    d.p_s = first ? a.chunk_p[c] : a.stage_p[j];
    d.p_e = lastc ? a.chunk_p[c + 1] : a.stage_p[j + 1];
    return d;
}

// Warp-uniform cursor over the warp's (chunk, stage) stream.
struct Cursor {
    int64_t gi;  // chunk-group index (blockIdx.x + t * gridDim.x)
    int64_t c;   // chunk
    int64_t j, jl;  // current stage, last stage of the chunk
    bool valid;
};

__device__ __forceinline__ bool chunk_stages(const SpmvArgs &a, int64_t c, int64_t &j0,
                                             int64_t &j1) {
    const int64_t cb0 = a.chunk_b[c], cb1 = a.chunk_b[c + 1];
    const int64_t b0 = max(cb0, a.b_lo), b1 = min(cb1, a.b_hi);
    if (b0 >= b1) return false;
    j0 = stage_of(b0, a.off32, a.stage_k);
    j1 = stage_of(b1 - 1, a.off32, a.stage_k);
    return true;
}

__device__ __forceinline__ void cursor_seek(const SpmvArgs &a, Cursor &cu, int warp) {
    // first chunk at or after cu.gi that has work
    const int64_t nc = a.c_hi - a.c_lo;
    for (;;) {
        if (cu.gi * kWarpsPerCta >= nc) {
            cu.valid = false;
            return;
        }
        cu.c = a.c_lo + cu.gi * kWarpsPerCta + warp;
        if (cu.c >= a.c_hi) {
            cu.valid = false;
            return;
        }
        if (chunk_stages(a, cu.c, cu.j, cu.jl)) {
            cu.valid = true;
            return;
        }
        cu.gi += gridDim.x;
    }
}

__device__ __forceinline__ void cursor_next(const SpmvArgs &a, Cursor &cu, int warp) {
    if (cu.j < cu.jl) {
        ++cu.j;
        return;
    }
    cu.gi += gridDim.x;
    cursor_seek(a, cu, warp);
}

struct SlotLayout {
    uint32_t off_mask, off_rp, off_val, bytes;
};

__device__ __forceinline__ uint64_t align_dn16(uint64_t v) { return v & ~uint64_t(15); }
__device__ __forceinline__ uint64_t align_up16(uint64_t v) { return (v + 15) & ~uint64_t(15); }

// Lane 0 of the warp: copy one stage's four regions into a slot.
template <typename T, typename MT, int R>
__device__ __forceinline__ void issue_stage(const SpmvArgs &a, const StageDesc &d, uint8_t *slot,
                                            const SlotLayout &lay, uint64_t *bar, uint64_t pol) {
    constexpr int MB = (int)sizeof(MT);
    const uint64_t c0 = (uint64_t)(a.colidx + d.start), c1 = (uint64_t)(a.colidx + d.end);
    const uint64_t m0 = (uint64_t)((const uint8_t *)a.masks + d.start * R * MB);
    const uint64_t m1 = (uint64_t)((const uint8_t *)a.masks + d.end * R * MB);
    const int64_t rp_last = min(d.p_e + 1, a.num_panels);
    const bool rp_staged = rp_last - d.p_s + 1 <= a.rp_cap;
    const uint64_t r0 = (uint64_t)(a.rowptr + d.p_s), r1 = (uint64_t)(a.rowptr + rp_last + 1);
    const uint64_t v0 = (uint64_t)((const T *)a.values + d.v_s);
    const uint64_t v1 = (uint64_t)((const T *)a.values + d.v_e);
    const uint32_t bc = (uint32_t)(align_up16(c1) - align_dn16(c0));
    const uint32_t bm = (uint32_t)(align_up16(m1) - align_dn16(m0));
    const uint32_t br = rp_staged ? (uint32_t)(align_up16(r1) - align_dn16(r0)) : 0u;
    const uint32_t bv = d.v_e > d.v_s ? (uint32_t)(align_up16(v1) - align_dn16(v0)) : 0u;
    mbar_expect_tx(bar, bc + bm + br + bv);
    bulk_g2s(slot, (const void *)align_dn16(c0), bc, bar, pol);
    bulk_g2s(slot + lay.off_mask, (const void *)align_dn16(m0), bm, bar, pol);
    if (br) bulk_g2s(slot + lay.off_rp, (const void *)align_dn16(r0), br, bar, pol);
    if (bv) bulk_g2s(slot + lay.off_val, (const void *)align_dn16(v0), bv, bar, pol);
}

template <int BYTES>
__device__ __forceinline__ uint32_t lds_lane_mask(const uint8_t *p) {
    if constexpr (BYTES == 1) return *p;
    else if constexpr (BYTES == 2) return *reinterpret_cast<const uint16_t *>(p);
    else return *reinterpret_cast<const uint32_t *>(p);
}

constexpr int kSlots = 2;  // stages in flight per warp

// K2.  R rows per panel, G rows per lane, L = R/G lanes per block,
// BW = 32/L blocks per window (windows aligned to global multiples of BW).
// Each warp streams its chunks stage by stage through a private ring of
// kSlots shared-memory slots filled by cp.async.bulk (TMA); the lanes only
// touch HBM for the x gathers and the y stores.
template <typename T, typename MT, int R, int G>
__global__ void __launch_bounds__(kWarpsPerCta * 32, 2) spmv_kernel(const SpmvArgs a) {
    constexpr int MB = (int)sizeof(MT);
    constexpr int MBITS = 8 * MB;
    constexpr int L = R / G;
    constexpr int BW = 32 / L;
    constexpr int LB = G * MB;  // mask bytes per lane
    static_assert(LB <= 4, "a lane's masks must fit 32 bits");
    constexpr int NP = (G * MBITS >= 32) ? 6 : (G * MBITS >= 16 ? 5 : 4);
    constexpr int NB = 4;  // value slots per batch
    extern __shared__ __align__(128) uint8_t smem[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int blk = lane / L;
    const int sub = lane % L;
    const T *__restrict__ x = static_cast<const T *>(a.x);
    T *__restrict__ y = static_cast<T *>(a.y);

    SlotLayout lay;
    lay.off_mask = a.lay_mask;
    lay.off_rp = a.lay_rp;
    lay.off_val = a.lay_val;
    lay.bytes = a.lay_bytes;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem) + warp * kSlots;
    uint8_t *slots = smem + 128 + (size_t)warp * kSlots * lay.bytes +
                     (size_t)0;  // barriers live in the first 128 bytes
    if (lane == 0) {
#pragma unroll
        for (int i = 0; i < kSlots; ++i) mbar_init(bars + i, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();

    if (!a.accumulate) {  // y = A.x: rows of empty panels are zero
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.num_empty;
             i += (int64_t)gridDim.x * blockDim.x) {
            const int64_t p = a.empty_panels[i];
            if (p < a.p_lo || p >= a.p_hi) continue;
#pragma unroll
            for (int rr = 0; rr < R; ++rr)
                if (p * R + rr < a.num_rows) y[p * R + rr] = T(0);
        }
    }

    const uint64_t pol = evict_first_policy();
    Cursor prod, cons;
    prod.gi = blockIdx.x;
    cursor_seek(a, prod, warp);
    cons = prod;
    // prologue: fill the ring
#pragma unroll
    for (int i = 0; i < kSlots; ++i) {
        if (prod.valid) {
            if (lane == 0)
                issue_stage<T, MT, R>(a, stage_desc(a, prod.c, prod.j), slots + i * lay.bytes, lay,
                                      bars + i, pol);
            cursor_next(a, prod, warp);
        }
    }

    uint32_t it = 0;  // stages consumed by this warp
    int64_t cur_chunk = -1;
    double carry[G];
    int64_t carry_panel = -1;
    int64_t pc = 0;
    while (cons.valid) {
        const int slot_i = it % kSlots;
        const uint32_t parity = (it / kSlots) & 1u;
        uint8_t *slot = slots + slot_i * lay.bytes;
        const int64_t c = cons.c;
        const StageDesc d = stage_desc(a, c, cons.j);
        const int64_t cb0 = a.chunk_b[c], cb1 = a.chunk_b[c + 1];
        const int64_t b0 = max(cb0, a.b_lo), b1 = min(cb1, a.b_hi);
        const int64_t p0 = a.chunk_p[c];
        if (c != cur_chunk) {  // chunk entry: fresh reduction state
            cur_chunk = c;
#pragma unroll
            for (int g = 0; g < G; ++g) carry[g] = 0.0;
            carry_panel = -1;
        }
        pc = d.p_s;
        const bool head_mid = __ldg(a.rowptr + p0) < cb0;  // chunk starts inside panel p0
        // element offsets of the stage inside its (16-byte widened) slot regions
        const uint32_t *s_col = reinterpret_cast<const uint32_t *>(slot) +
                                (((uint64_t)(a.colidx + d.start) & 15u) >> 2);
        const uint8_t *s_mask = slot + lay.off_mask +
                                ((uint64_t)((const uint8_t *)a.masks + d.start * R * MB) & 15u);
        const int64_t rp_last = min(d.p_e + 1, a.num_panels);
        const bool rp_staged = rp_last - d.p_s + 1 <= a.rp_cap;
        const int64_t *s_rp = rp_staged ? reinterpret_cast<const int64_t *>(slot + lay.off_rp) +
                                              (((uint64_t)(a.rowptr + d.p_s) & 15u) >> 3)
                                        : a.rowptr + d.p_s;
        const int n_rp = (int)(rp_last - d.p_s + 1);
        const T *s_val = reinterpret_cast<const T *>(slot + lay.off_val) +
                         (((uint64_t)((const T *)a.values + d.v_s) & 15u) / sizeof(T));
        const int64_t wfirst = d.start - ((d.start + a.base_mod) % BW);
        const int64_t cstart = max(cb0, d.start);  // first counted block of this stage
        uint32_t vrel = 0;

        mbar_wait(bars + slot_i, parity);

        for (int64_t wb = wfirst; wb < d.end; wb += BW) {
            const int64_t wn = wb + BW;
            const bool last = wn >= b1;
            const int64_t b = wb + blk;
            const bool counted = b >= cstart && b < d.end;
            const bool act = counted && b >= b0 && b < b1;
            const int irel = (int)(b - d.start);
            uint32_t col = 0, fm = 0;
            if (counted) {
                col = s_col[irel];
                fm = lds_lane_mask<LB>(s_mask + (irel * R + sub * G) * MB);
            }
            // ---- issue the x gathers and value reads first (latency overlap)
            const int cnt = __popc(fm);
            const int cmax = __reduce_max_sync(kFull, act ? cnt : 0);
            int excl, total;
            warp_prefix<NP>(cnt, lane, excl, total);
            T vv[NB], xv[NB];
            int gsel[NB];
            uint32_t fmc = act ? fm : 0u;
            const T *xp = x + col;
            const T *vp = s_val + vrel + excl;
#pragma unroll
            for (int u = 0; u < NB; ++u) {
                const bool valid = fmc != 0u;
                const int pos = __ffs(fmc) - 1;
                fmc &= fmc - 1u;
                gsel[u] = valid ? (G == 1 ? 0 : pos / MBITS) : -1;
                if (valid) {
                    xv[u] = __ldg(xp + (pos & (MBITS - 1)));
                    vv[u] = vp[u];
                }
            }
            // ---- panel of each block (block-level start bits) from the staged rowptr
            const int pk = (int)(pc - d.p_s) + 1 + lane;
            const int64_t E = pk < n_rp ? s_rp[pk] : INT64_MAX;
            const int64_t dd64 = E - wb;
            const bool in = dd64 >= 1 && dd64 < BW;
            unsigned starts = __reduce_or_sync(kFull, in ? (1u << (int)dd64) : 0u);
            const int nin = __popc(__ballot_sync(kFull, in));
            int64_t pl, pend_last;
            const unsigned blk_le = (BW == 32 && blk == 31) ? kFull : ((2u << blk) - 1u);
            if (__popc(starts) == nin) {  // no empty panel inside the window
                pl = pc + __popc(starts & blk_le);
                pend_last = __shfl_sync(kFull, E, __popc(starts));
            } else {  // empty panels: per-lane search over the loaded ends
                const int64_t bq = max(b, cb0);
                int cp = 0;
#pragma unroll
                for (int s2 = 16; s2 >= 1; s2 >>= 1) {
                    const int64_t e = __shfl_sync(kFull, E, cp + s2 - 1);
                    if (e <= bq) cp += s2;
                }
                const int64_t e31 = __shfl_sync(kFull, E, 31);
                pl = pc + cp;
                if (cp == 31 && e31 <= bq) {
                    int64_t lo = pc, hi = a.num_panels;
                    while (lo < hi) {
                        const int64_t mid = lo + (hi - lo + 1) / 2;
                        if (__ldg(a.rowptr + mid) <= bq) lo = mid;
                        else hi = mid - 1;
                    }
                    pl = lo;
                }
                const int64_t pprev = __shfl_up_sync(kFull, pl, L);
                const unsigned hb = __ballot_sync(kFull, sub == 0 && blk > 0 && pl != pprev);
                starts = 0;
#pragma unroll
                for (int t = 1; t < BW; ++t) starts |= ((hb >> (t * L)) & 1u) << t;
                const int64_t pl_last = __shfl_sync(kFull, pl, 31);
                pend_last = __ldg(a.rowptr + pl_last + 1);
            }
            // blocks past the chunk/range end: their own (silent) segment
            if (b1 - wb < BW) starts |= 1u << (int)(b1 - wb);
            const unsigned hbits = starts | 1u;
            // next window's first panel
            int64_t pcn = pc;
            if (!last && wn < d.end) {
                const int cn = __popc(__ballot_sync(kFull, E <= wn));
                if (cn < 32) {
                    pcn = pc + cn;
                } else {
                    int64_t lo = pc, hi = a.num_panels;
                    while (lo < hi) {
                        const int64_t mid = lo + (hi - lo + 1) / 2;
                        if (__ldg(a.rowptr + mid) <= wn) lo = mid;
                        else hi = mid - 1;
                    }
                    pcn = lo;
                }
            }

            // ---- products
            double acc[G];
#pragma unroll
            for (int g = 0; g < G; ++g) acc[g] = 0.0;
#pragma unroll
            for (int u = 0; u < NB; ++u) {
                if (G == 1) {
                    if (gsel[u] == 0) acc[0] = mul_acc<T>(acc[0], vv[u], xv[u]);
                } else if (gsel[u] >= 0) {
                    const double p = mul_acc<T>(0.0, vv[u], xv[u]);
#pragma unroll
                    for (int g = 0; g < G; ++g) acc[g] += (gsel[u] == g) ? p : 0.0;
                }
            }
            for (int j0 = NB; j0 < cmax; j0 += NB) {  // dense blocks: more batches
#pragma unroll
                for (int u = 0; u < NB; ++u) {
                    const bool valid = fmc != 0u;
                    const int pos = __ffs(fmc) - 1;
                    fmc &= fmc - 1u;
                    gsel[u] = valid ? (G == 1 ? 0 : pos / MBITS) : -1;
                    if (valid) {
                        xv[u] = __ldg(xp + (pos & (MBITS - 1)));
                        vv[u] = vp[j0 + u];
                    }
                }
#pragma unroll
                for (int u = 0; u < NB; ++u) {
                    if (G == 1) {
                        if (gsel[u] == 0) acc[0] = mul_acc<T>(acc[0], vv[u], xv[u]);
                    } else if (gsel[u] >= 0) {
                        const double p = mul_acc<T>(0.0, vv[u], xv[u]);
#pragma unroll
                        for (int g = 0; g < G; ++g) acc[g] += (gsel[u] == g) ? p : 0.0;
                    }
                }
            }
            vrel += (uint32_t)total;
            if (blk == 0 && pl == carry_panel) {
#pragma unroll
                for (int g = 0; g < G; ++g) acc[g] += carry[g];
            }

            // ---- segmented scan over blocks of the same panel (stride L lanes)
            const int segstart = 31 - __clz(hbits & blk_le);
#pragma unroll
            for (int dd = 1; dd < BW; dd <<= 1) {
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    const double t = __shfl_up_sync(kFull, acc[g], dd * L);
                    if (blk - dd >= segstart) acc[g] += t;
                }
            }
            const bool tailb = blk == BW - 1 || ((hbits >> (blk + 1)) & 1u);
            const bool cont = pend_last > wn;  // last block's panel continues past the window
            if (tailb && act && !(blk == BW - 1 && cont && !last) && pl >= a.p_lo &&
                pl < a.p_hi) {
                if (head_mid && pl == p0) {
#pragma unroll
                    for (int g = 0; g < G; ++g) a.carry[c * R + sub * G + g] = acc[g];
                } else {
#pragma unroll
                    for (int g = 0; g < G; ++g) {
                        const int64_t row = pl * R + sub * G + g;
                        if (row < a.num_rows) {
                            const T sv = (T)acc[g];
                            y[row] = a.accumulate ? y[row] + sv : sv;
                        }
                    }
                }
            }
            if (last) break;
            // ---- carry into the next window
            const int64_t pl_last = __shfl_sync(kFull, pl, 31);
#pragma unroll
            for (int g = 0; g < G; ++g) carry[g] = __shfl_sync(kFull, acc[g], (BW - 1) * L + sub);
            carry_panel = cont ? pl_last : -1;
            pc = pcn;
        }

        // ---- release the slot and refill it with the stage kSlots ahead
        __syncwarp();
        if (prod.valid) {
            if (lane == 0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                issue_stage<T, MT, R>(a, stage_desc(a, prod.c, prod.j), slot, lay,
                                      bars + slot_i, pol);
            }
            cursor_next(a, prod, warp);
        }
        ++it;
        cursor_next(a, cons, warp);
    }
}

template <typename T, int R>
__global__ void fixup_kernel(const int64_t *__restrict__ split, int64_t num_split,
                             const int64_t *__restrict__ chunk_p, const double *__restrict__ carry,
                             T *y, int64_t num_rows, int64_t c_lo, int64_t c_hi, int64_t p_lo,
                             int64_t p_hi) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= num_split) return;
    const int64_t c = split[i];
    if (c < c_lo || c >= c_hi) return;
    const int64_t P = chunk_p[c];
    if (P < p_lo || P >= p_hi) return;
    if (i > 0 && split[i - 1] == c - 1 && chunk_p[c - 1] == P) return;  // not the first
    double s[R];
#pragma unroll
    for (int rr = 0; rr < R; ++rr) s[rr] = carry[c * R + rr];
    for (int64_t j = i + 1; j < num_split; ++j) {
        const int64_t cj = split[j];
        if (cj != split[j - 1] + 1 || cj >= c_hi || chunk_p[cj] != P) break;
#pragma unroll
        for (int rr = 0; rr < R; ++rr) s[rr] += carry[cj * R + rr];
    }
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
        const int64_t row = P * R + rr;
        if (row < num_rows) y[row] = y[row] + (T)s[rr];
    }
}

template <typename T, typename MT, int R, int G>
int launch_typed(const Matrix &m, const SpmvArgs &a, cudaStream_t st) {
    const size_t smem = 128 + (size_t)kWarpsPerCta * kSlots * a.lay_bytes;
    static size_t smem_set = 0;
    static int max_blocks_per_sm = 0;
    if (smem > smem_set) {
        SPC5_CUDA(cudaFuncSetAttribute(spmv_kernel<T, MT, R, G>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        smem_set = smem;
        max_blocks_per_sm = 0;
    }
    static size_t occ_smem = 0;
    if (!max_blocks_per_sm || occ_smem != smem) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&max_blocks_per_sm,
                                                      spmv_kernel<T, MT, R, G>,
                                                      kWarpsPerCta * 32, smem);
        if (max_blocks_per_sm < 1) max_blocks_per_sm = 1;
        occ_smem = smem;
    }
    const int64_t nc = a.c_hi - a.c_lo;
    int64_t grid = std::max<int64_t>(cdiv(std::max<int64_t>(nc, 1), kWarpsPerCta),
                                     a.accumulate ? 1 : cdiv(a.num_empty, 256));
    grid = std::min<int64_t>(grid, (int64_t)m.sm_count * max_blocks_per_sm);
    grid = std::max<int64_t>(grid, 1);
    spmv_kernel<T, MT, R, G><<<(unsigned)grid, kWarpsPerCta * 32, smem, st>>>(a);
    SPC5_CUDA(cudaGetLastError());
    int launches = 1;
    if (m.plan.num_split) {
        fixup_kernel<T, R><<<(unsigned)cdiv(m.plan.num_split, 128), 128, 0, st>>>(
            m.plan.split_chunks, m.plan.num_split, m.plan.chunk_p, m.plan.carry,
            static_cast<T *>(a.y), m.num_rows, a.c_lo, a.c_hi, a.p_lo, a.p_hi);
        SPC5_CUDA(cudaGetLastError());
        ++launches;
    }
    note_launches(launches);
    return SPC5_OK;
}

template <typename T, typename MT>
int dispatch_r(const Matrix &m, const SpmvArgs &a, cudaStream_t st) {
    // G rows per lane: a lane's masks must fit 32 bits (G*sizeof(MT) <= 4)
    constexpr int G2 = sizeof(MT) == 1 ? 2 : 2;
    constexpr int G4 = sizeof(MT) == 1 ? 4 : 2;
    switch (m.r) {
        case 1: return launch_typed<T, MT, 1, 1>(m, a, st);
        case 2: return launch_typed<T, MT, 2, G2>(m, a, st);
        case 4: return launch_typed<T, MT, 4, G4>(m, a, st);
        default: return launch_typed<T, MT, 8, G4>(m, a, st);
    }
}

}  // namespace

int launch_spmv(const Matrix &m, int64_t p_lo, int64_t p_hi, const void *x, void *y,
                int accumulate, cudaStream_t st) {
    const Plan &P = m.plan;
    SpmvArgs a{};
    a.rowptr = m.rowptr;
    a.colidx = m.colidx;
    a.masks = m.masks;
    a.values = m.values;
    a.x = x;
    a.y = y;
    a.num_rows = m.num_rows;
    a.num_panels = m.num_panels;
    a.chunk_b = P.chunk_b;
    a.chunk_v = P.chunk_v;
    a.chunk_p = P.chunk_p;
    a.carry = P.carry;
    a.empty_panels = P.empty_panels;
    a.num_empty = P.num_empty;
    a.base_mod = (int)(((m.block_base % 32) + 32) % 32);  // windows divide 32
    a.accumulate = accumulate;
    a.stage_v = P.stage_v;
    a.stage_p = P.stage_p;
    a.stage_k = P.stage_granules;
    a.off32 = (int)(((m.block_base % 32) + 32) % 32);
    a.rp_cap = P.rp_cap;
    {
        auto a16 = [](int64_t v) { return (uint32_t)((v + 15) / 16 * 16); };
        const int64_t sb = 32LL * P.stage_granules;
        a.lay_mask = a16(sb * 4 + 32);
        a.lay_rp = a.lay_mask + a16(sb * m.r * m.mask_bytes() + 32);
        a.lay_val = a.lay_rp + a16((int64_t)P.rp_cap * 8 + 32);
        a.lay_bytes = (uint32_t)P.slot_bytes;
    }
    a.p_lo = p_lo;
    a.p_hi = p_hi;
    if (p_lo == 0 && p_hi == m.num_panels) {
        a.c_lo = 0;
        a.c_hi = P.num_chunks;
        a.b_lo = 0;
        a.b_hi = m.num_blocks;
    } else {
        int64_t blo = 0, bhi = 0;
        SPC5_CUDA(cudaMemcpyAsync(&blo, m.rowptr + p_lo, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        SPC5_CUDA(cudaMemcpyAsync(&bhi, m.rowptr + p_hi, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        SPC5_CUDA(cudaStreamSynchronize(st));
        a.b_lo = blo;
        a.b_hi = bhi;
        const int64_t *cb = P.h_chunk_b;
        const int64_t nc = P.num_chunks;
        a.c_lo = std::upper_bound(cb, cb + nc, blo) - cb - 1;
        if (a.c_lo < 0) a.c_lo = 0;
        a.c_hi = std::lower_bound(cb, cb + nc, bhi) - cb;
        if (blo >= bhi) a.c_hi = a.c_lo;  // no blocks: only empty-panel zeroing
    }
    if (P.num_chunks == 0 || a.c_hi <= a.c_lo) {
        a.c_lo = a.c_hi = 0;
        if (accumulate || a.num_empty == 0) {
            note_launches(0);
            return SPC5_OK;
        }
    }
    const bool f64 = m.precision == SPC5_F64;
    const bool wide = m.vs > 8;
    if (f64) return wide ? dispatch_r<double, uint16_t>(m, a, st) : dispatch_r<double, uint8_t>(m, a, st);
    return wide ? dispatch_r<float, uint16_t>(m, a, st) : dispatch_r<float, uint8_t>(m, a, st);
}

}  // namespace spc5
