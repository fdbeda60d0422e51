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
};

__device__ __forceinline__ uint32_t ldg_nc_u32(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

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

template <int BYTES>
__device__ __forceinline__ uint32_t load_lane_mask(const uint8_t *p) {
    if constexpr (BYTES == 1) {
        return *p;
    } else if constexpr (BYTES == 2) {
        return *reinterpret_cast<const uint16_t *>(p);
    } else {
        return ldg_nc_u32(reinterpret_cast<const uint32_t *>(p));
    }
}

// Window state: one lane = G consecutive rows of one block.
struct WinState {
    uint32_t col;  // block column start
    uint32_t fm;   // the lane's G masks, concatenated (row g at bits [g*MBITS, ...))
    int64_t E;     // block_rowptr[pc + 1 + lane]: end of panel pc + lane
};

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

// K2.  R rows per panel, G rows per lane, L = R/G lanes per block,
// BW = 32/L blocks per window (windows aligned to global multiples of BW).
template <typename T, typename MT, int R, int G>
__global__ void __launch_bounds__(256, 3) spmv_kernel(const SpmvArgs a) {
    constexpr int MB = (int)sizeof(MT);
    constexpr int MBITS = 8 * MB;
    constexpr int L = R / G;
    constexpr int BW = 32 / L;
    constexpr int LB = G * MB;  // mask bytes per lane
    static_assert(LB <= 4, "a lane's masks must fit 32 bits");
    constexpr int NP = (G * MBITS >= 32) ? 6 : (G * MBITS >= 16 ? 5 : 4);
    constexpr int NB = 4;  // value slots per batch
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int blk = lane / L;
    const int sub = lane % L;
    const T *__restrict__ vals = static_cast<const T *>(a.values);
    const T *__restrict__ x = static_cast<const T *>(a.x);
    T *__restrict__ y = static_cast<T *>(a.y);
    const int64_t *__restrict__ rowptr = a.rowptr;
    const uint8_t *__restrict__ masks = static_cast<const uint8_t *>(a.masks);

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

    const int64_t nc = a.c_hi - a.c_lo;
    for (int64_t gi = blockIdx.x; gi * kWarpsPerCta < nc; gi += gridDim.x) {
        const int64_t c = a.c_lo + gi * kWarpsPerCta + warp;
        if (c >= a.c_hi) break;
        const int64_t cb0 = a.chunk_b[c], cb1 = a.chunk_b[c + 1];
        const int64_t b0 = max(cb0, a.b_lo), b1 = min(cb1, a.b_hi);
        if (b0 >= b1) continue;
        const int64_t p0 = a.chunk_p[c];
        const bool head_mid = __ldg(rowptr + p0) < cb0;  // chunk starts inside panel p0
        const T *__restrict__ vbase = vals + a.chunk_v[c];
        uint32_t vrel = 0;  // value cursor relative to the chunk
        int64_t pc = p0;
        int64_t wb = cb0 - ((cb0 + a.base_mod) % BW);

        auto load_win = [&](int64_t w, int64_t pcw, WinState &st) {
            const int64_t b = w + blk;
            st.col = 0;
            st.fm = 0;
            if (b >= cb0 && b < b1) {
                st.col = ldg_nc_u32(a.colidx + b);
                st.fm = load_lane_mask<LB>(masks + (b * R + sub * G) * MB);
            }
            const int64_t e = pcw + 1 + lane;
            st.E = e <= a.num_panels ? __ldg(rowptr + e) : INT64_MAX;
        };
        WinState cur, nxt;
        load_win(wb, pc, cur);

        double carry[G];
#pragma unroll
        for (int g = 0; g < G; ++g) carry[g] = 0.0;
        int64_t carry_panel = -1;

        for (;;) {
            const int64_t wn = wb + BW;
            const bool last = wn >= b1;
            // ---- panel containing the next window's first block, then prefetch it
            int64_t pcn = pc;
            if (!last) {
                const int cn = __popc(__ballot_sync(kFull, cur.E <= wn));
                if (cn < 32) {
                    pcn = pc + cn;
                } else {
                    int64_t lo = pc, hi = a.num_panels;
                    while (lo < hi) {
                        const int64_t mid = lo + (hi - lo + 1) / 2;
                        if (__ldg(rowptr + mid) <= wn) lo = mid;
                        else hi = mid - 1;
                    }
                    pcn = lo;
                }
                load_win(wn, pcn, nxt);
            }

            // ---- value offsets
            const int64_t b = wb + blk;
            const bool act = b >= b0 && b < b1;
            const int cnt = __popc(cur.fm);
            int excl, total;
            warp_prefix<NP>(cnt, lane, excl, total);

            // ---- panel of each block (block-level start bits)
            const int64_t d = cur.E - wb;
            const bool in = d >= 1 && d < BW;
            unsigned starts = __reduce_or_sync(kFull, in ? (1u << (int)d) : 0u);
            const int nin = __popc(__ballot_sync(kFull, in));
            int64_t pl, pend_last;
            const unsigned blk_le = (BW == 32 && blk == 31) ? kFull : ((2u << blk) - 1u);
            if (__popc(starts) == nin) {  // no empty panel inside the window
                pl = pc + __popc(starts & blk_le);
                pend_last = __shfl_sync(kFull, cur.E, __popc(starts));
            } else {  // empty panels: per-lane search over the loaded ends
                const int64_t bq = max(b, cb0);
                int cp = 0;
#pragma unroll
                for (int s = 16; s >= 1; s >>= 1) {
                    const int64_t e = __shfl_sync(kFull, cur.E, cp + s - 1);
                    if (e <= bq) cp += s;
                }
                const int64_t e31 = __shfl_sync(kFull, cur.E, 31);
                pl = pc + cp;
                if (cp == 31 && e31 <= bq) {
                    int64_t lo = pc, hi = a.num_panels;
                    while (lo < hi) {
                        const int64_t mid = lo + (hi - lo + 1) / 2;
                        if (__ldg(rowptr + mid) <= bq) lo = mid;
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
                pend_last = __ldg(rowptr + pl_last + 1);
            }
            // blocks past the chunk/range end: their own (silent) segment
            if (b1 - wb < BW) starts |= 1u << (int)(b1 - wb);
            const unsigned hbits = starts | 1u;

            // ---- the lane's rows of its block: batched loads, then FMAs
            double acc[G];
#pragma unroll
            for (int g = 0; g < G; ++g) acc[g] = 0.0;
            const int cmax = __reduce_max_sync(kFull, act ? cnt : 0);
            if (cmax > 0) {
                const T *__restrict__ vp = vbase + (vrel + (uint32_t)excl);
                const T *__restrict__ xp = x + cur.col;
                uint32_t fmc = act ? cur.fm : 0u;
                for (int j0 = 0; j0 < cmax; j0 += NB) {
                    T vv[NB], xv[NB];
                    int gsel[NB];
#pragma unroll
                    for (int u = 0; u < NB; ++u) {
                        const bool valid = fmc != 0u;
                        const int pos = __ffs(fmc) - 1;
                        fmc &= fmc - 1u;
                        gsel[u] = valid ? (G == 1 ? 0 : pos / MBITS) : -1;
                        const int k = pos & (MBITS - 1);
                        vv[u] = valid ? __ldg(vp + j0 + u) : T(0);
                        xv[u] = valid ? __ldg(xp + k) : T(0);
                    }
#pragma unroll
                    for (int u = 0; u < NB; ++u) {
                        if (G == 1) {
                            if (gsel[u] == 0) acc[0] = mul_acc<T>(acc[0], vv[u], xv[u]);
                        } else {
                            // every accumulator is written (a zero where the row differs)
                            // so the compiler keeps acc[] in registers
                            const double p = mul_acc<T>(0.0, vv[u], xv[u]);
#pragma unroll
                            for (int g = 0; g < G; ++g) acc[g] += (gsel[u] == g) ? p : 0.0;
                        }
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
            wb = wn;
            cur = nxt;
        }
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
    static int max_blocks_per_sm = 0;
    if (!max_blocks_per_sm) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&max_blocks_per_sm,
                                                      spmv_kernel<T, MT, R, G>, 256, 0);
        if (max_blocks_per_sm < 1) max_blocks_per_sm = 1;
    }
    const int64_t nc = a.c_hi - a.c_lo;
    int64_t grid = std::max<int64_t>(cdiv(std::max<int64_t>(nc, 1), kWarpsPerCta),
                                     a.accumulate ? 1 : cdiv(a.num_empty, 256));
    grid = std::min<int64_t>(grid, (int64_t)m.sm_count * max_blocks_per_sm);
    grid = std::max<int64_t>(grid, 1);
    spmv_kernel<T, MT, R, G><<<(unsigned)grid, 256, 0, st>>>(a);
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
