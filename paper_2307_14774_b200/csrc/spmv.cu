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

template <int BYTES>
struct MaskWords {
    static constexpr int N = (BYTES + 3) / 4;
    uint32_t w[N];
    __device__ __forceinline__ void load(const uint8_t *p) {
        if constexpr (BYTES == 1) {
            w[0] = *p;
        } else if constexpr (BYTES == 2) {
            w[0] = *reinterpret_cast<const uint16_t *>(p);
        } else if constexpr (BYTES == 4) {
            w[0] = ldg_nc_u32(reinterpret_cast<const uint32_t *>(p));
        } else if constexpr (BYTES == 8) {
            uint2 v;
            asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0, %1}, [%2];"
                         : "=r"(v.x), "=r"(v.y) : "l"(p));
            w[0] = v.x;
            w[1] = v.y;
        } else {
            uint4 v;
            asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
            w[0] = v.x;
            w[1] = v.y;
            w[2] = v.z;
            w[3] = v.w;
        }
    }
    __device__ __forceinline__ void zero() {
#pragma unroll
        for (int i = 0; i < N; ++i) w[i] = 0;
    }
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

template <typename T, typename MT, int R>
__global__ void __launch_bounds__(256) spmv_kernel(const SpmvArgs a) {
    constexpr int MB = (int)sizeof(MT);
    constexpr int MBITS = 8 * MB;
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const T *__restrict__ vals = static_cast<const T *>(a.values);
    const T *__restrict__ x = static_cast<const T *>(a.x);
    T *__restrict__ y = static_cast<T *>(a.y);
    const int64_t *__restrict__ rowptr = a.rowptr;

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
    for (int64_t g = blockIdx.x; g * kWarpsPerCta < nc; g += gridDim.x) {
        const int64_t c = a.c_lo + g * kWarpsPerCta + warp;
        if (c >= a.c_hi) break;
        const int64_t cb0 = a.chunk_b[c], cb1 = a.chunk_b[c + 1];
        const int64_t b0 = max(cb0, a.b_lo), b1 = min(cb1, a.b_hi);
        if (b0 >= b1) continue;
        int64_t v = a.chunk_v[c];
        int64_t pc = a.chunk_p[c];
        int64_t ps = __ldg(rowptr + pc);
        double carry[R];
#pragma unroll
        for (int rr = 0; rr < R; ++rr) carry[rr] = 0.0;
        int64_t carry_panel = -1;
        const int64_t w0 = cb0 - ((cb0 + a.base_mod) & 31);
        for (int64_t w = w0; w < b1; w += 32) {
            const int64_t b = w + lane;
            const bool counted = b >= cb0 && b < b1;  // contributes to the value cursor
            const bool act = b >= b0 && b < b1;       // contributes to y
            uint32_t col = 0;
            MaskWords<R * MB> mw;
            mw.zero();
            if (counted) {
                col = ldg_nc_u32(a.colidx + b);
                mw.load(static_cast<const uint8_t *>(a.masks) + b * (R * MB));
            }
            int cnt = 0;
#pragma unroll
            for (int i = 0; i < MaskWords<R * MB>::N; ++i) cnt += __popc(mw.w[i]);
            int incl = cnt;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int t = __shfl_up_sync(kFull, incl, d);
                if (lane >= d) incl += t;
            }
            int64_t off = v + incl - cnt;
            v += __shfl_sync(kFull, incl, 31);

            // ---- panel of the lane's block
            const int64_t bq = min(max(b, cb0), b1 - 1);
            const int64_t eidx = pc + 1 + lane;
            const int64_t E = eidx <= a.num_panels ? __ldg(rowptr + eidx) : INT64_MAX;
            int cp = 0;
#pragma unroll
            for (int s = 16; s >= 1; s >>= 1) {
                const int64_t e = __shfl_sync(kFull, E, cp + s - 1);
                if (e <= bq) cp += s;
            }
            const int64_t e31 = __shfl_sync(kFull, E, 31);
            const int64_t e_lo = __shfl_sync(kFull, E, cp > 0 ? cp - 1 : 0);
            const int64_t e_hi = __shfl_sync(kFull, E, cp);
            int64_t pl = pc + cp;
            int64_t pstart = cp ? e_lo : ps;
            int64_t pend = e_hi;
            const bool ovf = (cp == 31) && (e31 <= bq);
            if (__any_sync(kFull, ovf) && ovf) {
                int64_t lo = pc, hi = a.num_panels;  // last p with rowptr[p] <= bq
                while (lo < hi) {
                    const int64_t mid = lo + (hi - lo + 1) / 2;
                    if (__ldg(rowptr + mid) <= bq) lo = mid;
                    else hi = mid - 1;
                }
                pl = lo;
                pstart = __ldg(rowptr + pl);
                pend = __ldg(rowptr + pl + 1);
            }
            // lanes past the chunk (or range) end form their own segment: appending
            // zero lanes to the last panel's segment would change its sum's association
            if (b >= b1) pl = INT64_MAX;

            // ---- the block's dot products (one per panel row)
            double acc[R];
#pragma unroll
            for (int rr = 0; rr < R; ++rr) {
                uint32_t mm = (mw.w[(rr * MB) / 4] >> (((rr * MB) % 4) * 8)) &
                              (MBITS == 32 ? 0xffffffffu : ((1u << MBITS) - 1u));
                double s = 0.0;
                if (act) {
                    while (mm) {
                        const int k = __ffs(mm) - 1;
                        mm &= mm - 1;
                        s = mul_acc<T>(s, __ldg(vals + off), __ldg(x + col + k));
                        ++off;
                    }
                } else {
                    off += __popc(mm);
                }
                acc[rr] = s;
            }
            if (lane == 0 && pl == carry_panel) {
#pragma unroll
                for (int rr = 0; rr < R; ++rr) acc[rr] += carry[rr];
            }

            // ---- segmented reduction over lanes of the same panel
            const int64_t pl_prev = __shfl_up_sync(kFull, pl, 1);
            const bool head = lane == 0 || pl != pl_prev;
            const unsigned heads = __ballot_sync(kFull, head);
            const unsigned le = heads & (kFull >> (31 - lane));
            const int segstart = 31 - __clz(le);
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
                for (int rr = 0; rr < R; ++rr) {
                    const double t = __shfl_up_sync(kFull, acc[rr], d);
                    if (lane - d >= segstart) acc[rr] += t;
                }
            }
            const bool tail = lane == 31 || ((heads >> (lane + 1)) & 1u);
            const bool last_window = w + 32 >= b1;
            const bool cont = pend > w + 32;
            if (tail && !(cont && !last_window) && pl >= a.p_lo && pl < a.p_hi) {
                if (pstart < cb0) {
#pragma unroll
                    for (int rr = 0; rr < R; ++rr) a.carry[c * R + rr] = acc[rr];
                } else {
#pragma unroll
                    for (int rr = 0; rr < R; ++rr) {
                        const int64_t row = pl * R + rr;
                        if (row < a.num_rows) {
                            const T sv = (T)acc[rr];
                            y[row] = a.accumulate ? y[row] + sv : sv;
                        }
                    }
                }
            }
            if (last_window) break;
            // ---- state for the next window
            const bool c31 = __shfl_sync(kFull, cont, 31);
            const int64_t pl31 = __shfl_sync(kFull, pl, 31);
#pragma unroll
            for (int rr = 0; rr < R; ++rr) carry[rr] = __shfl_sync(kFull, acc[rr], 31);
            carry_panel = c31 ? pl31 : -1;
            const int64_t bn = w + 32;
            const unsigned le_bn = __ballot_sync(kFull, E <= bn);
            const int cn = __popc(le_bn);
            if (cn < 32) {
                const int64_t e_prev = __shfl_sync(kFull, E, cn > 0 ? cn - 1 : 0);
                ps = cn ? e_prev : ps;
                pc = pc + cn;
            } else {
                int64_t lo = pc, hi = a.num_panels;
                while (lo < hi) {
                    const int64_t mid = lo + (hi - lo + 1) / 2;
                    if (__ldg(rowptr + mid) <= bn) lo = mid;
                    else hi = mid - 1;
                }
                pc = lo;
                ps = __ldg(rowptr + pc);
            }
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

template <typename T, typename MT, int R>
int launch_typed(const Matrix &m, const SpmvArgs &a, cudaStream_t st) {
    static int max_blocks_per_sm = 0;
    if (!max_blocks_per_sm) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&max_blocks_per_sm, spmv_kernel<T, MT, R>,
                                                      256, 0);
        if (max_blocks_per_sm < 1) max_blocks_per_sm = 1;
    }
    const int64_t nc = a.c_hi - a.c_lo;
    int64_t grid = std::max<int64_t>(cdiv(std::max<int64_t>(nc, 1), kWarpsPerCta),
                                     a.accumulate ? 1 : cdiv(a.num_empty, 256));
    grid = std::min<int64_t>(grid, (int64_t)m.sm_count * max_blocks_per_sm);
    grid = std::max<int64_t>(grid, 1);
    spmv_kernel<T, MT, R><<<(unsigned)grid, 256, 0, st>>>(a);
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
    switch (m.r) {
        case 1: return launch_typed<T, MT, 1>(m, a, st);
        case 2: return launch_typed<T, MT, 2>(m, a, st);
        case 4: return launch_typed<T, MT, 4>(m, a, st);
        default: return launch_typed<T, MT, 8>(m, a, st);
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
    a.base_mod = (int)(((m.block_base % 32) + 32) % 32);
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
