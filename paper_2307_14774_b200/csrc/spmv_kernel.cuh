#pragma once
// spmv_kernel.cuh -- K2 (kernel templates; instantiated per (T, MT, R) by spmv_inst_*.cu,
// dispatched by spmv.cu): y (+)= A.x over the SPC5 beta(r,vs) arrays on sm_100a.
//
// Replaces spmv_spc5_scalar / spmv_spc5_vector (kernels.py:121-230), i.e.
// Algorithm 1 of the paper re-mapped to a B200 warp:
//
//  * TMA streaming.  The plan cuts the block array into chunks of ~32-256
//    blocks (starts snapped to panel starts).  Each warp owns a ring of
//    kSlots shared-memory slots; one lane fills a slot with a chunk's
//    panel-start bits, column starts, masks and packed values using four
//    cp.async.bulk copies completing on one mbarrier (SASS UBLKCP /
//    SYNCS), so the matrix stream never sits in registers and the next
//    kSlots-1 chunks are in flight while one is consumed.
//  * lane-per-block.  The warp walks its chunk in 32-block windows aligned to
//    GLOBAL block indices; lane l owns block w+l (all R rows of it).
//  * value offsets: popcount of the lane's masks + a warp inclusive scan --
//    the "value cursor" of kernels.py:211-212 in parallel form.
//  * panel membership: one bit per block from the plan's panel-start bitmap
//    (a popcount gives the panel of every lane); chunks holding empty panels
//    search block_rowptr instead.
//  * products: each panel row's set bits, highest first (bfind), x gathered
//    through the read-only path (x is the only re-read array and stays L2
//    resident; the matrix stream is loaded evict-first), fp64 accumulation
//    of products formed in the matrix precision.
//  * per-row reduction: a segmented warp scan over lanes of the same panel;
//    segment tails store y; the last segment of a window is carried into the
//    next one.  Chunks starting inside a long panel write their head segment
//    to a carry slot that a fixup kernel adds in chunk order.  Every panel is
//    summed in an order fixed by global block positions only, so results are
//    bitwise reproducible across runs, spmv_parallel ranges and GPU shards.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>
#include <type_traits>

#include "common.cuh"

// Every kernel instance: X(function name, T, MT, R).  spmv_inst_*.cu defines
// one function each (launch_typed<T, MT, R>), spmv.cu declares and calls them.
#define SPC5_K2_INSTANCES(X)                         \
    X(launch_k2_f64_u8_r1, double, uint8_t, 1) \
    X(launch_k2_f64_u8_r2, double, uint8_t, 2) \
    X(launch_k2_f64_u8_r4, double, uint8_t, 4) \
    X(launch_k2_f64_u8_r8, double, uint8_t, 8) \
    X(launch_k2_f64_u16_r1, double, uint16_t, 1) \
    X(launch_k2_f64_u16_r2, double, uint16_t, 2) \
    X(launch_k2_f64_u16_r4, double, uint16_t, 4) \
    X(launch_k2_f64_u16_r8, double, uint16_t, 8) \
    X(launch_k2_f32_u8_r1, float, uint8_t, 1) \
    X(launch_k2_f32_u8_r2, float, uint8_t, 2) \
    X(launch_k2_f32_u8_r4, float, uint8_t, 4) \
    X(launch_k2_f32_u8_r8, float, uint8_t, 8) \
    X(launch_k2_f32_u16_r1, float, uint16_t, 1) \
    X(launch_k2_f32_u16_r2, float, uint16_t, 2) \
    X(launch_k2_f32_u16_r4, float, uint16_t, 4) \
    X(launch_k2_f32_u16_r8, float, uint16_t, 8)

namespace spc5 {

constexpr int kMaxMirrors = 8;  // peer buffers of the fused exchange

struct SpmvArgs {
    const int64_t *rowptr;
    const uint32_t *colidx;
    const void *masks;
    const void *values;
    const void *x;
    void *y;
    int64_t num_rows, num_cols, num_panels;
    const int64_t *chunk_b, *chunk_v, *chunk_p;
    const uint8_t *chunk_flags;   // bit0 starts inside a panel, bit1 has empty panels
    const uint32_t *pstart_bits;  // panel-start bitmap over 32-block granules
    int64_t c_lo, c_hi;           // chunk index range
    int64_t b_lo, b_hi;           // blocks contributing to y
    int64_t p_lo, p_hi;           // panels whose rows may be written
    const int64_t *range;         // range products: {b_lo, b_hi, c_lo, c_hi} resolved on the device
    double *carry;
    const int64_t *empty_panels;
    int64_t num_empty;
    int off32;         // block_base mod 32 (window alignment)
    int accumulate;
    uint32_t lay_col, lay_mask, lay_val, lay_bytes;  // slot layout (bytes)
    const uint8_t *blob;      // per-chunk metadata blobs (header, panel-start words, records)
    const uint4 *issue_rec;   // per chunk: bulk-copy sources / sizes (plan.cu issue_rec_kernel)
    int nslot;                // ring slots per warp (2..kMaxSlots)
    // fused exchange (iterated products over GPUs): every y row is also
    // stored, scaled, at mirror[i][mirror_row0 + row] (peer GPUs' next-x
    // buffers over NVLink); y itself is scaled by yscale (1 unless mirrored)
    void *mirror[kMaxMirrors];
    int nmirror;
    int64_t mirror_row0;
    double yscale;
    int plain;  // !accumulate && !nmirror && yscale == 1
    int x_prefetch;  // x is 16-byte aligned: the chunks' x leading edges are prefetched to L2
    uint32_t acc_off;  // FVR kernels with R = 8: per-warp row sums in shared memory (R*256 B)
};

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kMaxSlots = 4;  // ring slots per warp (SpmvArgs::nslot)
constexpr uint32_t kHdr = 64;  // slot header bytes (chunk descriptor)
constexpr uint32_t kRecOff = 256;   // per-warp staging of the next issue record (32 B)
constexpr uint32_t kRingOff = 512;  // barriers (8 warps x kMaxSlots), records, then the ring

// ---- TMA (cp.async.bulk) + mbarrier helpers -------------------------------
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
// ---- checked build (-DSPC5_CHECKED=1; tools/checked_build.sh) ---------------
// compute-sanitizer is closed on the GPU pool, so the memcheck part is built
// in: every shared-memory access of the slot readers must fall inside the
// CTA's dynamic shared memory, every x gather inside x[0, num_cols) and every
// y store inside y[0, num_rows); a violation prints where and traps (the
// launch fails loudly).  Off in the product build: the checks compile away.
#ifndef SPC5_CHECKED
#define SPC5_CHECKED 0
#endif
#if SPC5_CHECKED
__shared__ unsigned long long chk_bounds[4];  // x lo/hi, y lo/hi (set by the kernel prologue)
__device__ __noinline__ void chk_fail(const char *what, unsigned long long v) {
    printf("SPC5_CHECKED violation: %s at %llx (block %d thread %d)\n", what, v, (int)blockIdx.x,
           (int)threadIdx.x);
    __trap();
}
__device__ __forceinline__ void chk_smem(uint32_t addr, uint32_t bytes) {
    extern __shared__ uint8_t chk_dyn[];
    uint32_t total;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(total));
    const uint32_t base = smem_addr(chk_dyn);
    if (addr < base || addr + bytes > base + total) chk_fail("shared-memory access", addr);
}
__device__ __forceinline__ void chk_x(const void *p, uint32_t bytes) {
    const unsigned long long v = (unsigned long long)p;
    if (v < chk_bounds[0] || v + bytes > chk_bounds[1]) chk_fail("x gather", v);
}
__device__ __forceinline__ void chk_y(const void *p, uint32_t bytes) {
    const unsigned long long v = (unsigned long long)p;
    if (v < chk_bounds[2] || v + bytes > chk_bounds[3]) chk_fail("y store", v);
}
#else
__device__ __forceinline__ void chk_smem(uint32_t, uint32_t) {}
__device__ __forceinline__ void chk_x(const void *, uint32_t) {}
__device__ __forceinline__ void chk_y(const void *, uint32_t) {}
#endif

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
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes,
                                         uint64_t *bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1], %2, [%3], %4;" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
    chk_smem(addr, 4);
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}

// A lane's R masks (R * sizeof(MT) <= 16 bytes) from shared memory.
template <int BYTES>
struct LaneMasks {
    static constexpr int N = (BYTES + 3) / 4;
    uint32_t w[N];
    __device__ __forceinline__ void load(uint32_t addr) {
        chk_smem(addr, BYTES);
        if constexpr (BYTES == 1) {
            asm volatile("ld.shared.u8 %0, [%1];" : "=r"(w[0]) : "r"(addr));
        } else if constexpr (BYTES == 2) {
            asm volatile("ld.shared.u16 %0, [%1];" : "=r"(w[0]) : "r"(addr));
        } else if constexpr (BYTES == 4) {
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w[0]) : "r"(addr));
        } else if constexpr (BYTES == 8) {
            asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(w[0]), "=r"(w[1]) : "r"(addr));
        } else {
            asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3])
                         : "r"(addr));
        }
    }
    __device__ __forceinline__ void clear_if(bool keep) {
#pragma unroll
        for (int i = 0; i < N; ++i) w[i] = keep ? w[i] : 0u;
    }
    __device__ __forceinline__ int popc() const {
        int c = 0;
#pragma unroll
        for (int i = 0; i < N; ++i) c += __popc(w[i]);
        return c;
    }
    template <int MB>
    __device__ __forceinline__ uint32_t row(int g) const {  // g: compile-time index
        constexpr uint32_t M = MB == 1 ? 0xffu : 0xffffu;
        return (w[(g * MB) / 4] >> (((g * MB) % 4) * 8)) & M;
    }
};

// x gathers: read-only path; with SPC5_X_EVICT_LAST an L2 evict-last policy
// (the per-load form of an L2 persistence window for x)
#ifndef SPC5_X_EVICT_LAST
#define SPC5_X_EVICT_LAST 0
#endif
#if SPC5_X_EVICT_LAST
__device__ __forceinline__ uint64_t x_policy() {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
#endif
__device__ __forceinline__ double ldg_pred(const double *p, bool pred) {
    if (pred) chk_x(p, 8);
    double v = 0.0;
#ifdef SPC5_X_PROBE_L1  // timing probe only (wrong results): gathers folded into a few 4 KB windows (L1 hits)
    p = reinterpret_cast<const double *>(reinterpret_cast<uintptr_t>(p) & ~(uintptr_t)0x1fff000);
#endif
#if SPC5_X_EVICT_LAST
    asm("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q ld.global.nc.L2::cache_hint.f64 %0, [%1], %3;\n}"
        : "+d"(v)
        : "l"(p), "r"((int)pred), "l"(x_policy()));
#else
    asm("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q ld.global.nc.f64 %0, [%1];\n}"
        : "+d"(v)
        : "l"(p), "r"((int)pred));
#endif
    return v;
}
__device__ __forceinline__ float ldg_pred(const float *p, bool pred) {
    if (pred) chk_x(p, 4);
    float v = 0.0f;
#ifdef SPC5_X_PROBE_L1
    p = reinterpret_cast<const float *>(reinterpret_cast<uintptr_t>(p) & ~(uintptr_t)0x1fff000);
#endif
#if SPC5_X_EVICT_LAST
    asm("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q ld.global.nc.L2::cache_hint.f32 %0, [%1], %3;\n}"
        : "+f"(v)
        : "l"(p), "r"((int)pred), "l"(x_policy()));
#else
    asm("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q ld.global.nc.f32 %0, [%1];\n}"
        : "+f"(v)
        : "l"(p), "r"((int)pred));
#endif
    return v;
}
template <typename T>
__device__ __forceinline__ T lds_pred(uint32_t addr, bool pred);
template <>
__device__ __forceinline__ double lds_pred<double>(uint32_t addr, bool pred) {
    if (pred) chk_smem(addr, 8);
    double v = 0.0;
    asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q ld.shared.f64 %0, [%1];\n}"
                 : "+d"(v)
                 : "r"(addr), "r"((int)pred));
    return v;
}
template <>
__device__ __forceinline__ float lds_pred<float>(uint32_t addr, bool pred) {
    if (pred) chk_smem(addr, 4);
    float v = 0.0f;
    asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q ld.shared.f32 %0, [%1];\n}"
                 : "+f"(v)
                 : "r"(addr), "r"((int)pred));
    return v;
}

// acc += v * x: fused for f64; for f32 the product is rounded in f32 (as the
// reference forms it) and accumulated in f64.  Empty slots add exact zeros.
template <typename T>
__device__ __forceinline__ void mac(double &acc, T v, T xv);
template <>
__device__ __forceinline__ void mac<double>(double &acc, double v, double xv) {
    acc = fma(v, xv, acc);
}
template <>
__device__ __forceinline__ void mac<float>(double &acc, float v, float xv) {
    acc += (double)__fmul_rn(v, xv);
}

// Slot-call partial sums: f64 products go straight into the f64 row sum; f32
// products of one call (<= U*NS of them) are summed with f32 FMAs and the
// partial is added to the f64 row sum once (SPC5_F32_PARTIAL; the error of a
// partial is <= U*NS f32 roundings of its own sum of |products|, well inside
// the reference's f32 budget nnz_row * eps * sum|p|, kernels.py:305-312).
#ifndef SPC5_F32_PARTIAL
#define SPC5_F32_PARTIAL 1
#endif
template <typename T>
struct SlotSum {  // f64 matrices: the row sum itself
    double &acc;
    __device__ __forceinline__ explicit SlotSum(double &a) : acc(a) {}
    __device__ __forceinline__ void add(double v, double x) { acc = fma(v, x, acc); }
    __device__ __forceinline__ void done() {}
};
template <>
struct SlotSum<float> {
    double &acc;
    float part = 0.0f;
    __device__ __forceinline__ explicit SlotSum(double &a) : acc(a) {}
    __device__ __forceinline__ void add(float v, float x) {
        if (SPC5_F32_PARTIAL) part = __fmaf_rn(v, x, part);
        else mac<float>(acc, v, x);
    }
    __device__ __forceinline__ void done() {
        if (SPC5_F32_PARTIAL) acc += (double)part;
    }
};

// highest set bit of a non-zero word (PTX bfind -> SASS FLO)
__device__ __forceinline__ uint32_t bfind(uint32_t m) {
    uint32_t r;
    asm("bfind.u32 %0, %1;" : "=r"(r) : "r"(m));
    return r;
}

// warp inclusive scan of small ints (shfl.up with its in-range predicate)
__device__ __forceinline__ int warp_incl_scan(int v) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        asm("{\n .reg .s32 t;\n .reg .pred p;\n"
            " shfl.sync.up.b32 t|p, %0, %1, 0, -1;\n"
            " @p add.s32 %0, %0, t;\n}"
            : "+r"(v)
            : "r"(d));
    }
    return v;
}

// one y row: y[row] (+)= v, mirrored to the peer buffers of the fused exchange
template <typename T>
__device__ __forceinline__ void put_row(const SpmvArgs &a, T *y, int64_t row, double v) {
    chk_y(y + row, (uint32_t)sizeof(T));
    if (a.plain) {  // y = A.x, no mirrors: one store (a uniform branch, not predication)
        y[row] = (T)v;
        return;
    }
    T sv = (T)(v * a.yscale);
    if (a.accumulate) sv = y[row] + sv;
    y[row] = sv;
#pragma unroll 1  // (unrolled at every store site it bloats the hot loops out of the i-cache)
    for (int i = 0; i < a.nmirror; ++i) static_cast<T *>(a.mirror[i])[a.mirror_row0 + row] = sv;
}
template <typename T, int G>
__device__ __forceinline__ void store_rows(const SpmvArgs &a, T *y, int64_t row0,
                                           const double *acc) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
        const int64_t row = row0 + g;
        if (row < a.num_rows) put_row<T>(a, y, row, acc[g]);
    }
}

// A warp-uniform slot count compared through an opaque register copy: keeps
// the compiler from turning the dispatch if-chains into a jump table (BRX
// through the constant bank, a long branch-resolution stall per step).
#ifndef SPC5_NO_BRX
#define SPC5_NO_BRX 1
#endif
__device__ __forceinline__ bool ueq(int v, int k) {
#if SPC5_NO_BRX
    int r;
    asm volatile("{\n .reg .pred q;\n setp.eq.s32 q, %1, %2;\n selp.s32 %0, 1, 0, q;\n}"
                 : "=r"(r)
                 : "r"(v), "r"(k));
    return r != 0;
#else
    return v == k;
#endif
}

// Products of one panel row for U blocks: up to NS set bits per block,
// highest first.  All U*NS gathers are issued before the first FMA; products
// are accumulated block by block (storage order).  Slots past a block's count
// load nothing and add exact zeros.
// RUN (plans whose every row mask is one contiguous run of bits -- stencils,
// bands, dense sub-blocks; plan.cu runs_kernel): the columns of a block row are
// consecutive, so slot u gathers x[top - u] at an immediate offset from the
// address of the row's highest bit: 2 instructions per slot (predicate, load)
// instead of 7 (find bit, clear it, column, address, predicate, load).  Same
// products in the same order as the general walk: bitwise the same sums.
template <typename T, int U, int NS, bool RUN = false>
__device__ __forceinline__ void row_slots(double &acc, uint32_t (&m)[U], int (&h)[U],
                                          const T *__restrict__ x, const uint32_t (&col)[U],
                                          const uint32_t (&vaddr)[U]) {
    T xv[U][NS];
    uint32_t vtop[U];  // value of the block's highest remaining bit; slot u reads vtop - u
    int h0[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
        h0[k] = h[k];
        vtop[k] = vaddr[k] + (uint32_t)(h[k] - 1) * (uint32_t)sizeof(T);
        h[k] = max(h[k] - NS, 0);
    }
    // all x gathers first (the long-latency loads), then values and products
    if constexpr (RUN) {
        const T *top[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const uint32_t pos = bfind(m[k]);
            top[k] = x + (col[k] + pos);
            // the run's top NS bits are consumed (only dense rows come back for more)
            m[k] = pos + 1u >= (uint32_t)NS ? (m[k] & ((1u << (pos + 1u - NS)) - 1u)) : 0u;
        }
#pragma unroll
        for (int u = 0; u < NS; ++u) {
#pragma unroll
            for (int k = 0; k < U; ++k) xv[k][u] = ldg_pred(top[k] - u, u < h0[k]);
        }
    } else {
#pragma unroll
        for (int u = 0; u < NS; ++u) {
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const uint32_t pos = bfind(m[k]);
                m[k] &= ~(1u << pos);
                xv[k][u] = ldg_pred(x + (col[k] + pos), u < h0[k]);
            }
        }
    }
    SlotSum<T> sum(acc);
#pragma unroll
    for (int k = 0; k < U; ++k) {
#pragma unroll
        for (int u = 0; u < NS; ++u) {
            const T vv = lds_pred<T>(vtop[k] - (uint32_t)(u * sizeof(T)), u < h0[k]);
            sum.add(vv, xv[k][u]);
        }
    }
    sum.done();
}

// One panel row of U blocks with a warp-uniform slot count: the smallest
// unrolled variant that covers every lane, or batches of 4.
template <typename T, int U, bool RUN = false>
__device__ __forceinline__ void row_dispatch(double &acc, uint32_t (&m)[U], int (&h)[U],
                                             const T *__restrict__ x, const uint32_t (&col)[U],
                                             const uint32_t (&vaddr)[U], int cmax) {
    if (cmax <= 0) return;
    if (ueq(cmax, 1)) {
        row_slots<T, U, 1, RUN>(acc, m, h, x, col, vaddr);
    } else if (ueq(cmax, 2)) {
        row_slots<T, U, 2, RUN>(acc, m, h, x, col, vaddr);
    } else if (ueq(cmax, 3)) {
        row_slots<T, U, 3, RUN>(acc, m, h, x, col, vaddr);
    } else if (ueq(cmax, 4)) {
        row_slots<T, U, 4, RUN>(acc, m, h, x, col, vaddr);
    } else {  // dense rows: one block at a time so the products stay in order
#pragma unroll
        for (int k = 0; k < U; ++k) {
            uint32_t mk1[1] = {m[k]};
            int hk1[1] = {h[k]};
            const uint32_t ck1[1] = {col[k]}, vk1[1] = {vaddr[k]};
            for (int done = 0; done < cmax; done += 4)
                row_slots<T, 1, 4, RUN>(acc, mk1, hk1, x, ck1, vk1);
        }
    }
}

// As row_slots / row_dispatch, but block k accumulates into acc[k] (the lane's
// blocks of K different windows in lane-per-block mode).
template <typename T, int U, int NS>
__device__ __forceinline__ void row_slots_sep(double (&acc)[U], uint32_t (&m)[U], int (&h)[U],
                                              const T *__restrict__ x,
                                              const uint32_t (&col)[U],
                                              const uint32_t (&vaddr)[U]) {
    T xv[U][NS];
    uint32_t vtop[U];
    int h0[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
        h0[k] = h[k];
        vtop[k] = vaddr[k] + (uint32_t)(h[k] - 1) * (uint32_t)sizeof(T);
        h[k] = max(h[k] - NS, 0);
    }
#pragma unroll
    for (int u = 0; u < NS; ++u) {
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const uint32_t pos = bfind(m[k]);
            m[k] &= ~(1u << pos);
            xv[k][u] = ldg_pred(x + (col[k] + pos), u < h0[k]);
        }
    }
    // one product per block and slot here (~1 per block in balanced lane
    // ranges): f32 partials per block measured slower than the f64 adds
#pragma unroll
    for (int k = 0; k < U; ++k) {
#pragma unroll
        for (int u = 0; u < NS; ++u) {
            const T vv = lds_pred<T>(vtop[k] - (uint32_t)(u * sizeof(T)), u < h0[k]);
            mac<T>(acc[k], vv, xv[k][u]);
        }
    }
}
// OPQ: opaque slot-count compares (if-chains) or plain ones (the compiler's
// jump table); measured per format, the jump table is faster only in the
// r = 2 kernels (config 3 beta(2,16): 659 vs 752 us)
template <typename T, int U, bool OPQ = true>
__device__ __forceinline__ void row_dispatch_sep(double (&acc)[U], uint32_t (&m)[U], int (&h)[U],
                                                 const T *__restrict__ x,
                                                 const uint32_t (&col)[U],
                                                 const uint32_t (&vaddr)[U], int cmax) {
    if (cmax <= 0) return;
    if ((OPQ ? ueq(cmax, 1) : cmax == 1)) {
        row_slots_sep<T, U, 1>(acc, m, h, x, col, vaddr);
    } else if ((OPQ ? ueq(cmax, 2) : cmax == 2)) {
        row_slots_sep<T, U, 2>(acc, m, h, x, col, vaddr);
    } else if ((OPQ ? ueq(cmax, 3) : cmax == 3)) {
        row_slots_sep<T, U, 3>(acc, m, h, x, col, vaddr);
    } else {
        for (int done = 0; done < cmax; done += 4) row_slots_sep<T, U, 4>(acc, m, h, x, col, vaddr);
    }
}



// Lane 0 of the warp: copy one chunk into the slot at shared address `slot`
// with bulk copies completing on one mbarrier: its metadata blob (header,
// panel-start words or panel records), column starts, masks and values.
// The plan precomputed every source offset and size (16-byte units).
#ifndef SPC5_X_PREFETCH
#define SPC5_X_PREFETCH 1
#endif
// L2 prefetch of x (the chunk's new columns, plan.cu xedge_kernel): issued
// with the chunk's bulk copies, a ring slot ahead of the chunk's x gathers, so
// the first reads of a banded matrix's leading edge hit L2 instead of DRAM
__device__ __forceinline__ void prefetch_x(const SpmvArgs &a, uint32_t w) {
    if (w) {
        const uint8_t *p = static_cast<const uint8_t *>(a.x) + (size_t)(w & 0x7ffffffu) * 32;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"((w >> 27) * 32u)
                     : "memory");
    }
}

template <typename T, int LB>
__device__ __forceinline__ void issue_chunk(const SpmvArgs &a, uint4 A, uint4 B, uint32_t slot,
                                            uint64_t *bar, uint64_t pol) {
    if (SPC5_X_PREFETCH && a.x_prefetch) prefetch_x(a, B.w);
    const uint8_t *colb = reinterpret_cast<const uint8_t *>(a.colidx);
    const uint8_t *maskb = static_cast<const uint8_t *>(a.masks);
    const uint8_t *valb = static_cast<const uint8_t *>(a.values);
    mbar_expect_tx(bar, B.z);
    bulk_g2s(slot, a.blob + (size_t)A.x * 16, (B.x & 0xffffu) * 16, bar, pol);
    bulk_g2s(slot + a.lay_col, colb + (size_t)A.y * 16, (B.x >> 16) * 16, bar, pol);
    bulk_g2s(slot + a.lay_mask, maskb + (size_t)A.z * 16, (B.y & 0xffffu) * 16, bar, pol);
    if (B.y >> 16) bulk_g2s(slot + a.lay_val, valb + (size_t)A.w * 16, (B.y >> 16) * 16, bar, pol);
}
// The refill's issue record is prefetched into shared memory with cp.async
// while the chunk is consumed (held in registers across the chunk it was
// spilled to local memory, i.e. an L2 round trip at refill time).
__device__ __forceinline__ void ir_prefetch(const SpmvArgs &a, int64_t c, uint32_t dst) {
    asm volatile(
        "cp.async.cg.shared.global [%0], [%1], 16;\n"
        "cp.async.cg.shared.global [%2], [%3], 16;\n"
        "cp.async.commit_group;\n" ::"r"(dst),
        "l"(a.issue_rec + 2 * c), "r"(dst + 16u), "l"(a.issue_rec + 2 * c + 1)
        : "memory");
}
__device__ __forceinline__ void ir_staged(uint32_t src, uint4 &A, uint4 &B) {
    asm volatile("cp.async.wait_all;" ::: "memory");
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(A.x), "=r"(A.y), "=r"(A.z), "=r"(A.w)
                 : "r"(src));
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(B.x), "=r"(B.y), "=r"(B.z), "=r"(B.w)
                 : "r"(src + 16u));
}
__device__ __forceinline__ void ir_load(const SpmvArgs &a, int64_t c, bool valid, uint4 &A,
                                        uint4 &B) {
    if (valid) {
        A = __ldg(a.issue_rec + 2 * c);
        B = __ldg(a.issue_rec + 2 * c + 1);
    }
}

__device__ __forceinline__ int64_t lds_s64(uint32_t addr) {
    chk_smem(addr, 8);
    int64_t v;
    asm volatile("ld.shared.s64 %0, [%1];" : "=l"(v) : "r"(addr));
    return v;
}

// popcount of the masks of rows 0..rr-1 of a lane's block (rr at run time)
template <int LB, int MB>
__device__ __forceinline__ int popc_below(const LaneMasks<LB> &mk, int rr) {
    const int bits = rr * 8 * MB;  // bit offset of row rr in the packed masks
    int c = 0;
#pragma unroll
    for (int i = 0; i < LaneMasks<LB>::N; ++i) {
        const int lo = i * 32;
        const uint32_t keep = bits >= lo + 32 ? 0xffffffffu
                                              : (bits <= lo ? 0u : ((1u << (bits - lo)) - 1u));
        c += __popc(mk.w[i] & keep);
    }
    return c;
}
template <int LB, int MB>
__device__ __forceinline__ uint32_t row_rt(const LaneMasks<LB> &mk, int rr) {
    const int bit = rr * 8 * MB;
    constexpr uint32_t M = MB == 1 ? 0xffu : 0xffffu;
    uint32_t w = mk.w[0];
#pragma unroll
    for (int i = 1; i < LaneMasks<LB>::N; ++i) w = (bit >> 5) == i ? mk.w[i] : w;
    return (w >> (bit & 31)) & M;
}

// Lane-per-panel-row mode (chunk flag bit2): the R*G lanes of a group own
// panel p0+q; lane (rr, sub) sums row rr over the sub-th of G contiguous
// block ranges of the panel, in storage order, and the G partial sums of a
// row meet in a butterfly (G = 1 << lg, chunk flag bits 3-4).  The 32/(R*G)
// groups of a step touch consecutive panels (neighbouring x for banded
// matrices).  The plan's records give the first block and first value
// (16 bits each, relative to the chunk) of every (panel, sub-range), so a
// lane starts at once.
// Pair slots (lane-per-panel-row steps): blocks 2i and 2i+1 of the lane's row
// form one 2*BB-bit word, so a step costs max-over-lanes(bits of a PAIR)
// slots instead of twice max-over-lanes(bits of a BLOCK) -- the row's bits
// are often all in one block of the pair (beta(8,8) stencil: 3+0 / 2+1 / 1+2).
// Bits highest first: the high block's (storage-later) bits, then the low
// block's; every product is accumulated in that fixed order.
template <typename T, int UP, int NS, int BB>
__device__ __forceinline__ void pair_slots(double &acc, const uint32_t (&m)[2 * UP],
                                           const int (&h)[2 * UP], const T *__restrict__ x,
                                           const uint32_t (&col)[2 * UP],
                                           const uint32_t (&vaddr)[2 * UP]) {
    constexpr uint32_t SZ = (uint32_t)sizeof(T);
    T xv[UP][NS];
    uint32_t P[UP], vhi[UP], vlo[UP];
    int c[UP], hh[UP];
#pragma unroll
    for (int i = 0; i < UP; ++i) {
        P[i] = m[2 * i] | (m[2 * i + 1] << BB);
        hh[i] = h[2 * i + 1];
        c[i] = h[2 * i] + hh[i];
        // slot u of the pair reads vhi - u (u < hh) or vlo - u (low block)
        vhi[i] = vaddr[2 * i + 1] + (uint32_t)(hh[i] - 1) * SZ;
        vlo[i] = vaddr[2 * i] + (uint32_t)(c[i] - 1) * SZ;
    }
#pragma unroll
    for (int u = 0; u < NS; ++u) {
#pragma unroll
        for (int i = 0; i < UP; ++i) {
            const uint32_t pos = bfind(P[i]);
            P[i] &= ~(1u << pos);
            const uint32_t xi = pos >= (uint32_t)BB ? col[2 * i + 1] + pos - BB : col[2 * i] + pos;
            xv[i][u] = ldg_pred(x + xi, u < c[i]);
        }
    }
    SlotSum<T> sum(acc);
#pragma unroll
    for (int i = 0; i < UP; ++i) {
#pragma unroll
        for (int u = 0; u < NS; ++u) {
            const uint32_t va = (u < hh[i] ? vhi[i] : vlo[i]) - (uint32_t)u * SZ;
            sum.add(lds_pred<T>(va, u < c[i]), xv[i][u]);
        }
    }
    sum.done();
}

__device__ __forceinline__ uint32_t lds_mask_row(uint32_t addr, int mb) {
    chk_smem(addr, (uint32_t)mb);
    uint32_t v;
    if (mb == 1) asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(addr));
    else asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}

// Lane-per-panel-row steps, v2.  A lane loads only its own row's mask of each
// block (immediate offsets from the step base; blocks past its range are
// masked to 0).  Value offsets come from the per-block bit counts h packed
// FB bits per block into words: an exclusive scan of the words over the R
// row-lanes of the panel (shfl.up by G) gives the bits of the rows below,
// the last row-lane's inclusive word gives the block totals, and one
// multiply gives their exclusive prefix over the word's blocks.  No lane
// popcounts the other rows' masks.  Field widths: FB=8 (vs<=8: h<=8, sums
// over 8 rows <= 64, prefix of 3 totals + rows below <= 248) or FB=16.
// PAIRS (U even): steps whose pair slots beat block slots use pair_slots.
template <typename T, typename MT, int R, int U, bool PAIRS, bool RUN = false>
__device__ __forceinline__ void lpp_steps2(double &acc, int maxlen, int my, int s, int rr, int lg,
                                           int lane, uint32_t vaddr, uint32_t a_col,
                                           uint32_t a_mask, const T *__restrict__ x) {
    constexpr int MB = (int)sizeof(MT);
    constexpr int LB = R * MB;
    constexpr int FB = MB == 1 ? 8 : 16;
    constexpr int BPW = 32 / FB;
    constexpr int NW = (U + BPW - 1) / BPW;
    constexpr uint32_t FM = FB == 8 ? 0xffu : 0xffffu;
    constexpr uint32_t SZ = (uint32_t)sizeof(T);
    const int width = R << lg;
    const int src_last = (lane & ~(width - 1)) | ((R - 1) << lg) | (lane & ((1 << lg) - 1));
    const uint32_t own = (uint32_t)(rr * MB);
    for (int j = 0; j < maxlen; j += U) {
        const int rem = my - j;
        const uint32_t bj = (uint32_t)(rem > 0 ? s + j : s);
        const uint32_t cb = a_col + bj * 4u, mbase = a_mask + bj * (uint32_t)LB + own;
        uint32_t col[U], m[U], vr[U];
        int h[U];
        uint32_t H[NW];
#pragma unroll
        for (int w = 0; w < NW; ++w) H[w] = 0u;
#pragma unroll
        for (int k = 0; k < U; ++k) {
            col[k] = lds_u32(cb + (uint32_t)k * 4u);
            const uint32_t raw = lds_mask_row(mbase + (uint32_t)(k * LB), MB);
            m[k] = k < rem ? raw : 0u;
            h[k] = __popc(m[k]);
            H[k / BPW] |= (uint32_t)h[k] << (FB * (k % BPW));
        }
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            uint32_t inc = H[w], tot = H[w];
            if constexpr (R > 1) {
#pragma unroll
                for (int d = 1; d < R; d <<= 1) {
                    const uint32_t t = __shfl_up_sync(kFull, inc, d << lg, width);
                    if (rr >= d) inc += t;
                }
                tot = __shfl_sync(kFull, inc, src_last);
            }
            const uint32_t ep = FB == 8 ? tot * 0x01010100u : tot << 16;  // exclusive prefix
            const uint32_t vw = ep + (inc - H[w]);  // + rows below, per field
#pragma unroll
            for (int i = 0; i < BPW; ++i) {
                const int k = w * BPW + i;
                if (k < U) vr[k] = vaddr + ((vw >> (FB * i)) & FM) * SZ;
            }
            vaddr += ((ep >> (32 - FB)) + (tot >> (32 - FB))) * SZ;  // the word's values
        }
        int cm = 0;
#pragma unroll
        for (int k = 0; k < U; ++k) cm = max(cm, h[k]);
        const int cmax = __reduce_max_sync(kFull, cm);
        if constexpr (PAIRS && U % 2 == 0) {
            int cp = 0;
#pragma unroll
            for (int i = 0; i < U / 2; ++i) cp = max(cp, h[2 * i] + h[2 * i + 1]);
            const int cpmax = __reduce_max_sync(kFull, cp);
            // pair slots cost ~13 instructions, block slots ~11
            if (cpmax <= 3 && cpmax * 13 < cmax * 22) {
                if (cpmax == 1) pair_slots<T, U / 2, 1, 8 * MB>(acc, m, h, x, col, vr);
                else if (cpmax == 2) pair_slots<T, U / 2, 2, 8 * MB>(acc, m, h, x, col, vr);
                else pair_slots<T, U / 2, 3, 8 * MB>(acc, m, h, x, col, vr);
                continue;
            }
        }
        if constexpr (U <= 9) {
            uint32_t mm[U];
            int hh[U];
#pragma unroll
            for (int k = 0; k < U; ++k) {
                mm[k] = m[k];
                hh[k] = h[k];
            }
            row_dispatch<T, U, RUN>(acc, mm, hh, x, col, vr, cmax);
        } else {  // two halves (register budget of the gathers in flight)
            constexpr int U1 = U / 2, U2 = U - U / 2;
            uint32_t m1[U1], c1[U1], v1[U1], m2[U2], c2[U2], v2[U2];
            int h1[U1], h2[U2], cm1 = 0, cm2 = 0;
#pragma unroll
            for (int k = 0; k < U1; ++k) {
                m1[k] = m[k]; c1[k] = col[k]; v1[k] = vr[k]; h1[k] = h[k];
                cm1 = max(cm1, h[k]);
            }
#pragma unroll
            for (int k = 0; k < U2; ++k) {
                m2[k] = m[U1 + k]; c2[k] = col[U1 + k]; v2[k] = vr[U1 + k]; h2[k] = h[U1 + k];
                cm2 = max(cm2, h[U1 + k]);
            }
            row_dispatch<T, U1, RUN>(acc, m1, h1, x, c1, v1, __reduce_max_sync(kFull, cm1));
            row_dispatch<T, U2, RUN>(acc, m2, h2, x, c2, v2, __reduce_max_sync(kFull, cm2));
        }
    }
}

template <typename T, typename MT, int R, bool GENERIC, bool RUN = false>
__device__ __forceinline__ void lpp_chunk(const SpmvArgs &a, int64_t c, int64_t p0, int npc,
                                          int lg, bool head_mid, uint32_t a_rec, uint32_t a_col,
                                          uint32_t a_mask, uint32_t a_val, int lane,
                                          const T *__restrict__ x, T *__restrict__ y) {
    constexpr int LGR = R == 1 ? 0 : R == 2 ? 1 : R == 4 ? 2 : 3;
    const int G = 1 << lg;
    const int sub = lane & (G - 1);
    const int rr = (lane >> lg) & (R - 1);
    const int grp = lane >> (lg + LGR);
    const int PP = 32 >> (lg + LGR);  // panels per step
    for (int q0 = 0; q0 < npc; q0 += PP) {
        const int q = q0 + grp;
        const bool pv = q < npc;
        // this lane's block range and first value: entries t, t+1 of the
        // plan's records (t = q*G + sub)
        const uint32_t rq = a_rec + (uint32_t)((min(q, npc - 1) << lg) + sub) * 4u;
        const uint32_t r0 = lds_u32(rq), r1 = lds_u32(rq + 4u);
        const int s = (int)(r0 & 0xffffu);
        const int my = pv ? (int)(r1 & 0xffffu) - s : 0;
        const uint32_t vofs = r0 >> 16;
        const int maxlen = __reduce_max_sync(kFull, my);
        uint32_t vaddr = a_val + vofs * (uint32_t)sizeof(T);
        double acc = 0.0;
        // U blocks per step (U from the longest lane range): all their x
        // gathers are in flight before the first FMA; values still accumulate
        // in storage order
        if constexpr (R == 8) {  // pair slots: steps of 6 / 12 / 18 blocks
            // (run plans keep the pair slots for 8-bit masks -- 128^3 f64 beta(8,8)
            // 105.6 us with them, 117.9 us with run block slots -- and use run
            // block slots where a step falls back to them)
            constexpr bool PR = !RUN || sizeof(MT) == 1;
            if (maxlen <= 6) {
                lpp_steps2<T, MT, R, 6, PR, RUN>(acc, maxlen, my, s, rr, lg, lane, vaddr, a_col, a_mask, x);
            } else if (maxlen <= 9) {  // one step of block slots (beta(8,16) stencil rows)
                lpp_steps2<T, MT, R, 9, false, RUN>(acc, maxlen, my, s, rr, lg, lane, vaddr, a_col, a_mask, x);
            } else if (maxlen <= 12) {
                lpp_steps2<T, MT, R, 12, PR, RUN>(acc, maxlen, my, s, rr, lg, lane, vaddr, a_col, a_mask, x);
            } else {
                lpp_steps2<T, MT, R, 18, PR, RUN>(acc, maxlen, my, s, rr, lg, lane, vaddr, a_col, a_mask, x);
            }
        } else {
            if (maxlen <= 3) {
                lpp_steps2<T, MT, R, 3, false, RUN>(acc, maxlen, my, s, rr, lg, lane, vaddr, a_col, a_mask, x);
            } else if (maxlen <= 6) {
                lpp_steps2<T, MT, R, 6, false, RUN>(acc, maxlen, my, s, rr, lg, lane, vaddr, a_col, a_mask, x);
            } else {
                lpp_steps2<T, MT, R, 9, false, RUN>(acc, maxlen, my, s, rr, lg, lane, vaddr, a_col, a_mask, x);
            }
        }
        for (int o = 1; o < G; o <<= 1) acc += __shfl_xor_sync(kFull, acc, o);
        const int64_t p = p0 + q;
        const int64_t row = p * R + rr;
        if (sub == 0 && pv) {
            if (q == 0 && head_mid) {  // head of a split panel: carry slot, fixup adds it
                a.carry[c * R + rr] = acc;
            } else if (row < a.num_rows && (!GENERIC || (p >= a.p_lo && p < a.p_hi))) {
                put_row<T>(a, y, row, acc);
            }
        }
    }
}

// Lane-per-block mode: 32-block windows aligned to global block indices,
// lane l owns block w+l (all R rows).  K windows per step: their metadata,
// value offsets and x gathers are all issued before the first window's
// segmented reduction, so K gathers per lane are in flight at once; the
// windows are then reduced in order (carry chain).
template <typename T, typename MT, int R, bool GENERIC, int K>
__device__ __forceinline__ void lpb_chunk(const SpmvArgs &a, int64_t c, int64_t b0, int64_t p0,
                                          int64_t pe, int n, int a0, int a1, bool head_mid,
                                          bool slow, int sh0, uint32_t a_bits, uint32_t a_col,
                                          uint32_t a_mask, uint32_t a_val, int lane,
                                          const T *__restrict__ x, T *__restrict__ y) {
    constexpr int MB = (int)sizeof(MT);
    constexpr int LB = R * MB;
    const unsigned lane_le = kFull >> (31 - lane);  // bits 0..lane
    double carry[R];
    bool carry_valid = false;
    int carry_panel = 0;           // relative to p0
    int pcur = head_mid ? 0 : -1;  // panel (rel. p0) of the block before the window
    uint32_t vrel = 0;
    for (int w0 = -sh0; w0 < a1; w0 += 32 * K) {
        int pl[K];
        unsigned hbits[K];
        bool act[K];
        uint32_t colk[K], vb[K];
        LaneMasks<LB> mk[K];
        // ---- metadata, value offsets and panels of the K windows
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int w = w0 + 32 * k;
            const int br = w + lane;  // block relative to the chunk start
            const bool counted = (unsigned)br < (unsigned)n;
            act[k] = GENERIC ? (br >= a0 && br < a1) : counted;
            const int bc = min(max(br, 0), n - 1);  // clamped: loads need no branch
            colk[k] = lds_u32(a_col + (uint32_t)bc * 4u);
            mk[k].load(a_mask + (uint32_t)bc * LB);
            mk[k].clear_if(counted);
            const int cnt = mk[k].popc();  // counted blocks advance the value cursor
            const int incl = warp_incl_scan(cnt);
            vb[k] = a_val + (vrel + (uint32_t)(incl - cnt)) * (uint32_t)sizeof(T);
            vrel += (uint32_t)__shfl_sync(kFull, incl, 31);
            pl[k] = 0;
            hbits[k] = kFull;
            if (w < a1) {
                // panel starts in this window (first / last window: counted blocks only)
                uint32_t W = lds_u32(a_bits + (uint32_t)((sh0 + w) >> 5) * 4u);
                if (w < 0 || n - w < 32) {
                    const int lo_i = max(-w, 0), hi_i = min(n - w, 32);
                    W &= (hi_i >= 32 ? kFull : ((1u << hi_i) - 1u)) & ~((1u << lo_i) - 1u);
                }
                // lanes past the active range form their own segment (appending
                // zero lanes to a panel's segment would change its association)
                const unsigned sent = (a1 - w < 32) ? (1u << (a1 - w)) : 0u;
                if (!slow) {
                    pl[k] = pcur + __popc(W & lane_le);
                    hbits[k] = W | sent | 1u;
                    pcur += __popc(W);
                } else {  // empty panels inside the chunk: search block_rowptr
                    const int64_t bq = b0 + max(br, 0);
                    int64_t lo = p0, hi = min(pe, a.num_panels - 1);
                    while (lo < hi) {
                        const int64_t mid = lo + (hi - lo + 1) / 2;
                        if (__ldg(a.rowptr + mid) <= bq) lo = mid;
                        else hi = mid - 1;
                    }
                    pl[k] = (int)(lo - p0);
                    const int pprev = __shfl_up_sync(kFull, pl[k], 1);
                    hbits[k] = __ballot_sync(kFull, lane > 0 && pl[k] != pprev) | sent | 1u;
                }
            }
        }
        // ---- products of every panel row of the lane's K blocks
        double acc[R][K];
#pragma unroll
        for (int g = 0; g < R; ++g) {
            uint32_t m[K], vr[K];
            int h[K], cm = 0;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const uint32_t mrow = mk[k].template row<MB>(g);
                m[k] = act[k] ? mrow : 0u;
                h[k] = __popc(m[k]);
                cm = max(cm, h[k]);
                vr[k] = vb[k];
                vb[k] += (uint32_t)__popc(mrow) * (uint32_t)sizeof(T);
                acc[g][k] = 0.0;
            }
            row_dispatch_sep<T, K, R != 2>(acc[g], m, h, x, colk, vr, __reduce_max_sync(kFull, cm));
        }
        // ---- reduce the windows in order
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int w = w0 + 32 * k;
            if (w >= a1) break;
            const bool last = w + 32 >= a1;
            double s[R];
#pragma unroll
            for (int g = 0; g < R; ++g) s[g] = acc[g][k];
            // the panel carried from the previous window: add or flush
            if (carry_valid) {
                const bool continues = __shfl_sync(kFull, pl[k], 0) == carry_panel;
                if (lane == 0) {
                    if (continues) {
#pragma unroll
                        for (int g = 0; g < R; ++g) s[g] += carry[g];
                    } else if (head_mid && carry_panel == 0) {
#pragma unroll
                        for (int g = 0; g < R; ++g) a.carry[c * R + g] = carry[g];
                    } else {
                        store_rows<T, R>(a, y, (p0 + carry_panel) * R, carry);
                    }
                }
                carry_valid = false;
            }
            // segmented scan over lanes of the same panel
            const int segstart = 31 - __clz(hbits[k] & lane_le);
#pragma unroll
            for (int dd = 1; dd < 32; dd <<= 1) {
                const bool take = lane - dd >= segstart;
#pragma unroll
                for (int g = 0; g < R; ++g) {
                    const double t = __shfl_up_sync(kFull, s[g], dd);
                    if (take) s[g] += t;
                }
            }
            const bool tail = lane == 31 || ((hbits[k] >> (lane + 1)) & 1u);
            // the window's last segment is carried unless the chunk ends here
            if (tail && act[k] && (lane != 31 || last)) {
                if (head_mid && pl[k] == 0) {
#pragma unroll
                    for (int g = 0; g < R; ++g) a.carry[c * R + g] = s[g];
                } else {
                    store_rows<T, R>(a, y, (p0 + pl[k]) * R, s);
                }
            }
            if (last) break;
#pragma unroll
            for (int g = 0; g < R; ++g) carry[g] = __shfl_sync(kFull, s[g], 31);
            carry_panel = __shfl_sync(kFull, pl[k], 31);
            carry_valid = GENERIC ? __shfl_sync(kFull, act[k], 31) : true;
        }
    }
}

// Balanced-lane-range mode (scan chunks without empty panels): lane l owns
// the contiguous blocks [l*n/32, (l+1)*n/32) of the chunk whatever the panel
// lengths.  It walks them in order (U blocks per step, gathers first),
// stores every panel that starts and ends inside its range, and keeps two
// partials: F, the panel open from the left (closed inside the range), and L,
// the panel open at the range end.  One segmented warp scan of L per chunk
// joins panels that span lanes.  The plan's lane records give each lane's
// first value and panel.  In range mode (GENERIC) the whole chunk is summed
// the same way and only rows of panels in [p_lo, p_hi) are written, so the
// result is bitwise the full product's.
template <typename T, int R>
__device__ __forceinline__ void blr_put(const SpmvArgs &a, int64_t c, int64_t p0, int p,
                                        bool head_mid, const double *v, T *__restrict__ y,
                                        bool generic) {
    if (p == 0 && head_mid) {  // head of a split panel: carry slot, fixup adds it
#pragma unroll
        for (int g = 0; g < R; ++g) a.carry[c * R + g] = v[g];
        return;
    }
    const int64_t P = p0 + p;
    if (generic && (P < a.p_lo || P >= a.p_hi)) return;
    store_rows<T, R>(a, y, P * R, v);
}

#ifndef SPC5_BLR
#define SPC5_BLR 1
#endif
#ifndef SPC5_BLR_U
#define SPC5_BLR_U (R <= 2 ? 4 : 2)
#endif
template <typename T, typename MT, int R, bool GENERIC, int U>
__device__ __forceinline__ void blr_chunk(const SpmvArgs &a, int64_t c, int64_t p0, int n,
                                          bool head_mid, int sh0, uint32_t a_zero, uint32_t a_bits,
                                          uint32_t a_lane, uint32_t a_col, uint32_t a_mask,
                                          uint32_t a_val, int lane, const T *__restrict__ x,
                                          T *__restrict__ y) {
    constexpr int MB = (int)sizeof(MT);
    constexpr int LB = R * MB;
    const int sl = (lane * n) >> 5, el = ((lane + 1) * n) >> 5;
    const bool nonempty = sl < el;
    const uint32_t rec = lds_u32(a_lane + (uint32_t)lane * 4u);
    uint32_t vaddr = a_val + (rec & 0xffffu) * (uint32_t)sizeof(T);
    const int pf = (int)(rec >> 16);  // panel of the lane's first block
    int p = pf;
    auto start_bit = [&](int b) -> bool {
        const uint32_t wrd = lds_u32(a_bits + (uint32_t)((sh0 + b) >> 5) * 4u);
        return (wrd >> ((sh0 + b) & 31)) & 1u;
    };
    const bool first_start = nonempty && start_bit(sl);
    const bool first_open = nonempty && !first_start;
    double acc[R], F[R];
#pragma unroll
    for (int g = 0; g < R; ++g) acc[g] = F[g] = 0.0;
    bool flushed = false;
    const int my = el - sl;
    const int maxlen = __reduce_max_sync(kFull, my);
    for (int j = 0; j < maxlen; j += U) {
        uint32_t col[U], vbk[U];
        LaneMasks<LB> mk[U];
        bool st[U];
        uint32_t vnext = vaddr;
        // panel-start bits of blocks sl+j .. sl+j+U-1 (two words, one funnel shift)
        const int gb = sh0 + sl + j;
        const uint32_t w0 = lds_u32(a_bits + (uint32_t)(gb >> 5) * 4u);
        const uint32_t w1 = lds_u32(a_bits + (uint32_t)((gb >> 5) + 1) * 4u);
        const uint32_t sbits = __funnelshift_r(w0, w1, gb & 31);
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const bool ok = j + k < my;
            const int b = ok ? sl + j + k : 0;
            col[k] = lds_u32(a_col + (uint32_t)b * 4u);
            mk[k].load(ok ? a_mask + (uint32_t)b * LB : a_zero);
            st[k] = ok && j + k > 0 && ((sbits >> k) & 1u);
            vbk[k] = vnext;
            vnext += (uint32_t)mk[k].popc() * (uint32_t)sizeof(T);
        }
        vaddr = vnext;
        // gathers of all U blocks (every row), then the blocks in order
        double part[U][R];
#pragma unroll
        for (int g = 0; g < R; ++g) {
            uint32_t m[U], vr[U];
            int h[U], cm = 0;
            double pg[U];
#pragma unroll
            for (int k = 0; k < U; ++k) {
                m[k] = mk[k].template row<MB>(g);
                h[k] = __popc(m[k]);
                cm = max(cm, h[k]);
                vr[k] = vbk[k];
                vbk[k] += (uint32_t)h[k] * (uint32_t)sizeof(T);
                pg[k] = 0.0;
            }
            row_dispatch_sep<T, U, R != 2>(pg, m, h, x, col, vr, __reduce_max_sync(kFull, cm));
#pragma unroll
            for (int k = 0; k < U; ++k) part[k][g] = pg[k];
        }
        if (R == 1 && a.plain) {
            // Branch-free closes (r = 1; for r > 1 the R predicated stores
            // and selects per block cost more than the branch): a block that starts a panel stores the
            // current one (predicated) or, the first time in a lane that
            // began inside a panel, parks it in F.  The chunk's head panel
            // of a split chunk is always closed through F (its first close
            // in any lane), so no carry slot is written here.
            T *yp = y + (p0 + p) * R;
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const bool toF = st[k] && !flushed && first_open;
                const bool put = st[k] && !toF &&
                                 (!GENERIC || (p0 + p >= a.p_lo && p0 + p < a.p_hi));
#pragma unroll
                for (int g = 0; g < R; ++g) {
                    F[g] = toF ? acc[g] : F[g];
                    if (put && (R == 1 || (p0 + p) * R + g < a.num_rows)) yp[g] = (T)acc[g];
                    acc[g] = st[k] ? part[k][g] : acc[g] + part[k][g];
                }
                flushed |= st[k];
                p += st[k] ? 1 : 0;
                yp += st[k] ? R : 0;
            }
        } else {
#pragma unroll
            for (int k = 0; k < U; ++k) {
                if (st[k]) {  // block starts a new panel: close the current one
                    if (!flushed && first_open) {
#pragma unroll
                        for (int g = 0; g < R; ++g) F[g] = acc[g];
                    } else {
                        blr_put<T, R>(a, c, p0, p, head_mid, acc, y, GENERIC);
                    }
                    flushed = true;
                    ++p;
#pragma unroll
                    for (int g = 0; g < R; ++g) acc[g] = 0.0;
                }
#pragma unroll
                for (int g = 0; g < R; ++g) acc[g] += part[k][g];
            }
        }
    }
    // join the panels that span lanes: segmented inclusive scan of L = acc
    const bool seg = first_start || flushed;
    const unsigned segs = __ballot_sync(kFull, seg) | 1u;
    const unsigned lane_le = kFull >> (31 - lane);
    const int segstart = 31 - __clz(segs & lane_le);
#pragma unroll
    for (int dd = 1; dd < 32; dd <<= 1) {
        const bool take = lane - dd >= segstart;
#pragma unroll
        for (int g = 0; g < R; ++g) {
            const double t = __shfl_up_sync(kFull, acc[g], dd);
            if (take) acc[g] += t;
        }
    }
    double prev[R];
#pragma unroll
    for (int g = 0; g < R; ++g) {
        prev[g] = __shfl_up_sync(kFull, acc[g], 1);
        if (lane == 0) prev[g] = 0.0;
    }
    if (nonempty) {
        if (first_open && flushed) {  // the panel open from the left ends here
            double v[R];
#pragma unroll
            for (int g = 0; g < R; ++g) v[g] = prev[g] + F[g];
            blr_put<T, R>(a, c, p0, pf, head_mid, v, y, GENERIC);
        } else if (first_start && sl > 0) {  // it ended at this lane's boundary
            blr_put<T, R>(a, c, p0, pf - 1, head_mid, prev, y, GENERIC);
        }
        if (lane == 31) blr_put<T, R>(a, c, p0, p, head_mid, acc, y, GENERIC);
    }
}

// shared-memory load that only happens when p (else `old` is kept)
__device__ __forceinline__ uint32_t lds_u32_if(uint32_t addr, bool p, uint32_t old) {
    if (p) chk_smem(addr, 4);
    uint32_t v = old;
    asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q ld.shared.u32 %0, [%1];\n}"
                 : "+r"(v)
                 : "r"(addr), "r"((int)p));
    return v;
}

template <int LB>
struct BlockBits {  // the R masks of one block, row-major, as one bit string of 32-bit words
    static constexpr int W = (LB + 3) / 4;
    uint32_t w[W];
    // (re)load when p
    __device__ __forceinline__ void load_if(uint32_t addr, bool p) {
        if (p) chk_smem(addr, LB);
        const int q = (int)p;
        if constexpr (LB == 1) {
            asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q ld.shared.u8 %0, [%1];\n}"
                         : "+r"(w[0]) : "r"(addr), "r"(q));
        } else if constexpr (LB == 2) {
            asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q ld.shared.u16 %0, [%1];\n}"
                         : "+r"(w[0]) : "r"(addr), "r"(q));
        } else if constexpr (LB == 4) {
            asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q ld.shared.u32 %0, [%1];\n}"
                         : "+r"(w[0]) : "r"(addr), "r"(q));
        } else if constexpr (LB == 8) {  // 8-byte aligned: a block's masks start at b * LB
            asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %3, 0;\n @q ld.shared.v2.u32 {%0, %1}, [%2];\n}"
                         : "+r"(w[0]), "+r"(w[1]) : "r"(addr), "r"(q));
        } else {
            asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %5, 0;\n"
                         " @q ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];\n}"
                         : "+r"(w[0]), "+r"(w[1]), "+r"(w[2]), "+r"(w[3]) : "r"(addr), "r"(q));
        }
    }
    __device__ __forceinline__ bool empty() const {
        uint32_t o = w[0];
#pragma unroll
        for (int i = 1; i < W; ++i) o |= w[i];
        return o == 0;
    }
    __device__ __forceinline__ void take_if(bool p, const BlockBits &o) {
#pragma unroll
        for (int i = 0; i < W; ++i) w[i] = p ? o.w[i] : w[i];
    }
    // position of the lowest set bit (garbage when empty), cleared when p
    __device__ __forceinline__ int pop_if(bool p) {
        if constexpr (W == 1) {
            const int q = __ffs(w[0]) - 1;
            w[0] = p ? (w[0] & (w[0] - 1u)) : w[0];
            return q;
        } else if constexpr (W == 2) {
            const bool lo = w[0] != 0u;
            const uint32_t v = lo ? w[0] : w[1];
            const uint32_t cl = v & (v - 1u);
            w[0] = (p && lo) ? cl : w[0];
            w[1] = (p && !lo) ? cl : w[1];
            return (lo ? 0 : 32) + __ffs(v) - 1;
        } else {
            int k = W - 1;  // the first non-zero word
#pragma unroll
            for (int i = W - 2; i >= 0; --i) k = w[i] ? i : k;
            uint32_t v = w[W - 1];
#pragma unroll
            for (int i = W - 2; i >= 0; --i) v = k == i ? w[i] : v;
            const uint32_t cl = v & (v - 1u);
#pragma unroll
            for (int i = 0; i < W; ++i) w[i] = (p && k == i) ? cl : w[i];
            return 32 * k + __ffs(v) - 1;
        }
    }
};

// acc[row] += v for a run-time row: R fused multiply-adds by a one-hot 1.0 /
// 0.0 (3 instructions per row).  An if-chain is folded by the compiler into
// an indexed add (row sums in local memory), a predicated add becomes an add
// plus two selects.
template <int R>
__device__ __forceinline__ void add_row(double (&acc)[R], double v, int row) {
    if constexpr (R == 1) {
        acc[0] += v;
    } else {
#pragma unroll
        for (int g = 0; g < R; ++g) {
            // 1.0 has a zero low word: only the high word is selected
            const double one_hot = __hiloint2double(row == g ? 0x3ff00000 : 0, 0);
            acc[g] = fma(v, one_hot, acc[g]);
        }
    }
}

#ifndef SPC5_LBR_K
#define SPC5_LBR_K 2  // rounds per step in lane-per-block-row mode
#endif
#ifndef SPC5_FVR_U
#define SPC5_FVR_U (R == 1 ? 8 : 4)
#endif
// Flat value-range mode (chunk flag bit6): lane l owns the chunk's values
// [l*nv/32, (l+1)*nv/32) -- the same count for every lane, whatever the block
// fill -- and walks them in storage order: a block's R masks form one
// row-major bit string (the value order within a block), whose lowest set
// bit gives the next value's row (bit / bits-per-row) and column (colidx +
// bit % bits-per-row).  The plan's lane records give the block holding the
// lane's first value, the set bits of that block before it and its panel.
// The walk is branch-free: the next block's column start, masks and
// panel-start bit are loaded one block ahead (predicated shared loads).  U
// values per step: their x gathers are all issued before the first product.
// Products go to R per-row sums of the current panel (predicated adds); a
// block that starts a panel closes the current one exactly as in
// balanced-lane-range mode (F for the panel open from the left, stores
// otherwise) and one segmented warp scan per chunk joins panels that span
// lanes.  For chunks of about one value per block row or fewer (power-law
// rows, FEM beta(8,8)), where per-row modes mostly visit empty rows.
template <typename T, typename MT, int R, bool GENERIC, int U>
__device__ __forceinline__ void fvr_chunk(const SpmvArgs &a, int64_t c, int64_t p0, int n,
                                          bool head_mid, int sh0, uint32_t a_bits,
                                          uint32_t a_rec, uint32_t a_col, uint32_t a_mask,
                                          const T *sval, int lane, const T *__restrict__ x,
                                          T *__restrict__ y) {
    constexpr int MB = (int)sizeof(MT);
    constexpr int LB = R * MB;
    constexpr int BPR = 8 * MB;  // bits per block row in the bit string
    const uint32_t rec = lds_u32(a_rec + (uint32_t)lane * 4u);
    const int nv = (int)lds_u32(a_rec + 128u);
    const int j0 = (lane * nv) >> 5, j1 = ((lane + 1) * nv) >> 5;
    const int V = j1 - j0;
    const bool nonempty = V > 0;
    int b = (int)(rec & 0xfffu);
    const int skip = (int)((rec >> 12) & 0x7fu);
    const int pf = (int)(rec >> 19);
    int p = pf;
    uint32_t col = lds_u32(a_col + (uint32_t)b * 4u);
    BlockBits<LB> cur;
#pragma unroll
    for (int i = 0; i < BlockBits<LB>::W; ++i) cur.w[i] = 0;
    cur.load_if(a_mask + (uint32_t)b * LB, true);
    for (int k = 0; k < skip; ++k) cur.pop_if(true);
    // panel-start bits of the blocks after b (bit 0 = block b+1), refilled
    // before a step that could walk past them
    auto window = [&](int bb) -> uint32_t {  // start bits of blocks bb .. bb+31
        const int g = sh0 + bb;
        const uint32_t w0 = lds_u32(a_bits + (uint32_t)(g >> 5) * 4u);
        const uint32_t w1 = lds_u32(a_bits + (uint32_t)((g >> 5) + 1) * 4u);
        return __funnelshift_r(w0, w1, g & 31);
    };
    const uint32_t w_here = window(b);
    // the lane's first value starts a panel (else the panel is open from the left)
    const bool first_start = nonempty && skip == 0 && (w_here & 1u);
    const bool first_open = nonempty && !first_start;
    uint32_t sw = w_here >> 1;
    int left = 31;  // valid bits in sw
    // the next block, loaded ahead
    int bn = min(b + 1, n - 1);
    uint32_t ncol = lds_u32(a_col + (uint32_t)bn * 4u);
    BlockBits<LB> nxt = cur;
    nxt.load_if(a_mask + (uint32_t)bn * LB, true);
    const T *vp = sval + j0;
    double acc[R], F[R];
#pragma unroll
    for (int g = 0; g < R; ++g) acc[g] = F[g] = 0.0;
    // R = 8: the row sums of the current panel live in shared memory (row g
    // of this lane at sacc[g*32 + lane]): one load-add-store per value
    // instead of R one-hot fused multiply-adds
    constexpr bool SACC = R == 8;  // (measured: R = 4 is faster with one-hot adds)
    double *sacc = nullptr;  // row sums of this lane, stride 32
    if constexpr (SACC) {
        extern __shared__ __align__(128) uint8_t smem_dyn[];
        sacc = reinterpret_cast<double *>(smem_dyn + a.acc_off) + (threadIdx.x >> 5) * (R * 32) + lane;
#pragma unroll
        for (int g = 0; g < R; ++g) sacc[g * 32] = 0.0;
    }
    bool flushed = false;
    const int vmax = (nv + 31) >> 5;
    for (int s = 0; s < vmax; s += U) {
        if (left < U) {  // the start-bit window may run out in this step: refill (rare)
            sw = window(b + 1);
            left = 32;
        }
        T xv[U], vv[U];
        int rowk[U];
        bool newp[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (s + u >= vmax) break;  // warp-uniform: the last step may be short
            const bool valid = s + u < V;
            const bool adv = valid && cur.empty();  // this value is the next block's first
            b = adv ? bn : b;
            col = adv ? ncol : col;
            cur.take_if(adv, nxt);
            newp[u] = adv && (sw & 1u);
            sw = adv ? sw >> 1 : sw;
            left -= adv ? 1 : 0;
            bn = min(b + 1, n - 1);
            ncol = lds_u32_if(a_col + (uint32_t)bn * 4u, adv, ncol);
            nxt.load_if(a_mask + (uint32_t)bn * LB, adv);
            const int pos = cur.pop_if(valid);
            rowk[u] = pos / BPR;
            xv[u] = T(0);
            vv[u] = T(0);
            if (valid) {
                chk_x(x + (col + (uint32_t)(pos % BPR)), (uint32_t)sizeof(T));
                chk_smem(smem_addr(vp + u), (uint32_t)sizeof(T));
                xv[u] = __ldg(x + (col + (uint32_t)(pos % BPR)));
                vv[u] = vp[u];
            }
        }
        vp += U;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (s + u >= vmax) break;
            double pr;
            if constexpr (sizeof(T) == 8) pr = (double)vv[u] * (double)xv[u];
            else pr = (double)__fmul_rn((float)vv[u], (float)xv[u]);
            if constexpr (R == 1) {
                // a block starting a panel closes the current one: the lane's
                // first close parks it in F when the panel was open from the left
                const bool toF = newp[u] && !flushed && first_open;
                const bool put = newp[u] && !toF &&
                                 (!GENERIC || (p0 + p >= a.p_lo && p0 + p < a.p_hi));
                F[0] = toF ? acc[0] : F[0];
                if (put) blr_put<T, 1>(a, c, p0, p, head_mid, acc, y, false);
                acc[0] = newp[u] ? pr : acc[0] + pr;
                flushed = flushed || newp[u];
                p += newp[u] ? 1 : 0;
            } else {
                // a block starting a panel closes the current one; the
                // warp-uniform test keeps the rare close a real branch (the
                // compiler would otherwise predicate its whole body into every step)
                if (newp[u]) {  // a block starting a panel: close the current one
                    if constexpr (SACC) {
#pragma unroll
                        for (int g = 0; g < R; ++g) {
                            acc[g] = sacc[g * 32];
                            sacc[g * 32] = 0.0;
                        }
                    }
                    if (!flushed && first_open) {
#pragma unroll
                        for (int g = 0; g < R; ++g) F[g] = acc[g];
                    } else {
                        blr_put<T, R>(a, c, p0, p, head_mid, acc, y, GENERIC);
                    }
                    flushed = true;
                    ++p;
#pragma unroll
                    for (int g = 0; g < R; ++g) acc[g] = 0.0;
                }
                if constexpr (SACC) sacc[rowk[u] * 32] += pr;
                else add_row<R>(acc, pr, rowk[u]);
            }
        }
    }
    if constexpr (SACC) {
#pragma unroll
        for (int g = 0; g < R; ++g) acc[g] = sacc[g * 32];
    }
    // join the panels that span lanes: segmented inclusive scan of L = acc
    const bool seg = first_start || flushed;
    const unsigned segs = __ballot_sync(kFull, seg) | 1u;
    const unsigned lane_le = kFull >> (31 - lane);
    const int segstart = 31 - __clz(segs & lane_le);
#pragma unroll
    for (int dd = 1; dd < 32; dd <<= 1) {
        const bool take = lane - dd >= segstart;
#pragma unroll
        for (int g = 0; g < R; ++g) {
            const double t = __shfl_up_sync(kFull, acc[g], dd);
            if (take) acc[g] += t;
        }
    }
    double prev[R];
#pragma unroll
    for (int g = 0; g < R; ++g) {
        prev[g] = __shfl_up_sync(kFull, acc[g], 1);
        if (lane == 0) prev[g] = 0.0;
    }
    if (nonempty) {
        if (first_open && flushed) {  // the panel open from the left ends here
            double v[R];
#pragma unroll
            for (int g = 0; g < R; ++g) v[g] = prev[g] + F[g];
            blr_put<T, R>(a, c, p0, pf, head_mid, v, y, GENERIC);
        } else if (first_start && j0 > 0) {  // it ended at this lane's boundary
            blr_put<T, R>(a, c, p0, pf - 1, head_mid, prev, y, GENERIC);
        }
        if (lane == 31) blr_put<T, R>(a, c, p0, p, head_mid, acc, y, GENERIC);
    }
}

// ---------------------------------------------------------------------------
// Lane-per-block-row mode (LBR; plan.cu P.lbr: matrices whose blocks hold
// about one value per block row or more in long panels, e.g. the FEM config).
// The chunk's n*R row masks are walked in storage order, 32 per round: lane l
// of round i owns mask 32*i + l, i.e. row l % R of block (32*i + l) / R -- a
// lane always works on the same row-in-panel, so its row sum is ONE register
// and the R*... lanes of a panel row meet in a log2(32/R)-step butterfly when
// the panel closes.  Value offsets: one warp scan per K rounds (the rounds'
// counts packed 16 bits each).  A round costs max-over-lanes(values of a block
// ROW) slots: 3 for dense 3x3 FEM blocks whatever r is, where lane-per-block
// windows pay for the fullest BLOCK and lane-per-panel-row steps for the
// blocks a row does not touch.  K rounds per step: their gathers are all in
// flight before the first product.  Chunks are cut at exact global multiples
// of the chunk target (no snapping to panel starts), so rounds are full; chunk
// heads inside a panel go through the carry slots / fixup kernel as for every
// split chunk.  The whole chunk is always summed (range products only filter
// the stores), so range products are bitwise the full product's.
template <typename T, typename MT, int R, bool GENERIC, int K>
__device__ __forceinline__ void lbr_chunk(const SpmvArgs &a, int64_t c, int64_t p0, int n,
                                          bool head_mid, int sh0, uint32_t a_bits, uint32_t a_col,
                                          uint32_t a_mask, uint32_t a_val, int lane,
                                          const T *__restrict__ x, T *__restrict__ y) {
    constexpr int MB = (int)sizeof(MT);
    constexpr int LGR = R == 1 ? 0 : R == 2 ? 1 : R == 4 ? 2 : 3;
    constexpr int BPRD = 32 >> LGR;  // blocks per round
    constexpr uint32_t SZ = (uint32_t)sizeof(T);
    constexpr uint32_t SM = BPRD == 32 ? kFull : ((1u << BPRD) - 1u);
    const int g = lane & (R - 1), grp = lane >> LGR;
    auto put = [&](int pr, double v) {  // lanes < R: row `lane` of the closed panel pr (rel. p0)
        if (lane >= R) return;
        if (pr == 0 && head_mid) {
            a.carry[c * R + g] = v;
            return;
        }
        const int64_t P = p0 + pr;
        if (GENERIC && (P < a.p_lo || P >= a.p_hi)) return;
        const int64_t row = P * R + g;
        if (row < a.num_rows) put_row<T>(a, y, row, v);
    };
    auto reduce_g = [&](double v) -> double {  // over the lanes of the same row-in-panel
#pragma unroll
        for (int o = R; o < 32; o <<= 1) v += __shfl_xor_sync(kFull, v, o);
        return v;
    };
    int pcur = head_mid ? 0 : -1;  // the open panel (rel. p0); -1: none yet
    double acc = 0.0;
    uint32_t vrel = 0;
    for (int b0r = 0; b0r < n; b0r += K * BPRD) {
        uint32_t m[K], col[K], vr[K], S[K];
        int h[K];
        uint32_t packed = 0;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int bb = b0r + k * BPRD;  // first block of the round
            const int b = bb + grp;
            const bool counted = b < n;
            const int bc = min(b, n - 1);
            col[k] = lds_u32(a_col + (uint32_t)bc * 4u);
            const uint32_t raw = lds_mask_row(a_mask + (uint32_t)(bc * R + g) * MB, MB);
            m[k] = counted ? raw : 0u;
            h[k] = __popc(m[k]);
            packed |= (uint32_t)h[k] << (16 * (k & 1));
            // panel starts among the round's blocks
            const int gb = sh0 + bb;
            const uint32_t w0 = lds_u32(a_bits + (uint32_t)(gb >> 5) * 4u);
            const uint32_t w1 = lds_u32(a_bits + (uint32_t)((gb >> 5) + 1) * 4u);
            uint32_t sb = __funnelshift_r(w0, w1, gb & 31) & SM;
            const int nleft = n - bb;  // counted blocks of the round
            sb = nleft >= BPRD ? sb : (nleft > 0 ? sb & ((1u << nleft) - 1u) : 0u);
            S[k] = sb;
            if ((k & 1) == 1 || k == K - 1) {  // one scan per two rounds
                const uint32_t incl = (uint32_t)warp_incl_scan((int)packed);
                const uint32_t tot = __shfl_sync(kFull, incl, 31);
                if ((k & 1) == 1) {
                    const uint32_t t0 = tot & 0xffffu;
                    vr[k - 1] = a_val + (vrel + (incl & 0xffffu) - (uint32_t)h[k - 1]) * SZ;
                    vr[k] = a_val + (vrel + t0 + (incl >> 16) - (uint32_t)h[k]) * SZ;
                    vrel += t0 + (tot >> 16);
                } else {
                    vr[k] = a_val + (vrel + (incl & 0xffffu) - (uint32_t)h[k]) * SZ;
                    vrel += tot & 0xffffu;
                }
                packed = 0;
            }
        }
        int cm = 0;
#pragma unroll
        for (int k = 0; k < K; ++k) cm = max(cm, h[k]);
        double ar[K];
#pragma unroll
        for (int k = 0; k < K; ++k) ar[k] = 0.0;
        row_dispatch_sep<T, K, true>(ar, m, h, x, col, vr, __reduce_max_sync(kFull, cm));
#pragma unroll
        for (int k = 0; k < K; ++k) {
            if (S[k] == 0u) {  // warp-uniform: no panel starts in the round
                acc += ar[k];
                continue;
            }
            // panels closing in this round: the open one takes the lanes before
            // the first start, each further start closes the panel before it
            uint32_t sbits = S[k];
            int lo = 0;
            while (sbits) {
                const int kb = __ffs(sbits) - 1;
                sbits &= sbits - 1u;
                const double v = acc + ((grp >= lo && grp < kb) ? ar[k] : 0.0);
                const double tot = reduce_g(v);
                if (pcur >= 0) put(pcur, tot);
                acc = 0.0;
                ++pcur;
                lo = kb;
            }
            acc = grp >= lo ? ar[k] : 0.0;
        }
    }
    // the chunk's last panel (it may continue in the next chunk: carry / fixup)
    const double tot = reduce_g(acc);
    if (pcur >= 0) put(pcur, tot);
}

// K2.  Each warp takes chunks c_lo + (blockIdx.x + k*gridDim.x)*W + warp,
// k = 0, 1, ...; the CTA's warps work on neighbouring chunks (x reuse in L1).
// GENERIC=true restricts the product to a panel range (spc5_spmv_panels /
// spmv_parallel); the arithmetic per panel is identical.
// Chunk modes compiled into a kernel (a plan whose chunks all use one or two
// modes runs a kernel without the others' code: the hot loop stays small in
// the instruction cache and the register allocation is its own).  MODE 0:
// lane-per-panel-row, balanced lane ranges and lane-per-block (no flat value
// ranges); 1: flat value ranges only; 2: every mode (mixed plans and range
// products); 3: lane-per-panel-row only; 4: lane-per-block-row rounds (LBR
// plans; chunks holding empty panels fall back to lane-per-block); 6:
// lane-per-panel-row only, every row mask one run of bits (immediate-offset
// gathers, row_slots RUN).
template <typename T, typename MT, int R, bool GENERIC, int MODE>
// 168 registers: 12 warps per SM (3 CTAs x 4 warps) fit the register file;
// the shared-memory ring allows no more
#ifndef SPC5_K2_MAXREG
#define SPC5_K2_MAXREG 168
#endif
#ifndef SPC5_K2_MAXREG_F32
#define SPC5_K2_MAXREG_F32 SPC5_K2_MAXREG
#endif
__global__ void __maxnreg__(sizeof(T) == 4 ? SPC5_K2_MAXREG_F32 : SPC5_K2_MAXREG)
    spmv_kernel(const SpmvArgs a) {
    constexpr int MB = (int)sizeof(MT);
    constexpr int LB = R * MB;  // mask bytes per lane (<= 16)
    extern __shared__ __align__(128) uint8_t smem[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const T *__restrict__ x = static_cast<const T *>(a.x);
    T *__restrict__ y = static_cast<T *>(a.y);

#if SPC5_CHECKED
    if (threadIdx.x == 0) {
        chk_bounds[0] = (unsigned long long)a.x;
        // (a shard reads x up to the matrix's last column: num_cols of the handle)
        chk_bounds[1] = (unsigned long long)a.x + (unsigned long long)a.num_cols * sizeof(T);
        chk_bounds[2] = (unsigned long long)a.y;
        chk_bounds[3] = (unsigned long long)a.y + (unsigned long long)a.num_rows * sizeof(T);
    }
    __syncthreads();
#endif
    const int S = a.nslot;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem) + warp * kMaxSlots;
    const uint32_t ring = smem_addr(smem) + kRingOff + (uint32_t)(warp * S) * a.lay_bytes;
    if (lane == 0) {
#pragma unroll
        for (int i = 0; i < S; ++i) mbar_init(bars + i, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();

    if (!a.accumulate) {  // y = A.x: rows of empty panels are zero
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.num_empty;
             i += (int64_t)gridDim.x * blockDim.x) {
            const int64_t p = a.empty_panels[i];
            if (GENERIC && (p < a.p_lo || p >= a.p_hi)) continue;
#pragma unroll
            for (int rr = 0; rr < R; ++rr)
                if (p * R + rr < a.num_rows) put_row<T>(a, y, p * R + rr, 0.0);
        }
    }

    const uint64_t pol = evict_first_policy();
    const int wpc = blockDim.x >> 5;  // warps per CTA
    const int64_t stride = (int64_t)gridDim.x * wpc;
    int64_t c_lo = a.c_lo, c_end = a.c_hi, b_lo = a.b_lo, b_hi = a.b_hi;
    if (GENERIC && a.range) {  // range resolved on the device by range_kernel
        b_lo = a.range[0];
        b_hi = a.range[1];
        c_lo = a.range[2];
        c_end = a.range[3];
    }
    const int64_t cfirst = c_lo + (int64_t)blockIdx.x * wpc + warp;
    // prologue: fill the ring with the warp's first S chunks
    if (lane == 0) {
        for (int i = 0; i < S; ++i) {
            const int64_t ci = cfirst + i * stride;
            if (ci >= c_end) break;
            uint4 A, B;
            ir_load(a, ci, true, A, B);
            issue_chunk<T, LB>(a, A, B, ring + (uint32_t)i * a.lay_bytes, bars + i, pol);
        }
    }

    int slot_i = 0;
    uint32_t parity = 0;
    for (int64_t c = cfirst; c < c_end; c += stride) {
        const int64_t cn = c + S * stride;  // the chunk that refills this slot
        // its issue record: prefetched now, the latency hides behind this chunk's work
        const uint32_t rec_stage = smem_addr(smem) + kRecOff + (uint32_t)warp * 32u;
        if (lane == 0 && cn < c_end) ir_prefetch(a, cn, rec_stage);
        const uint32_t sbase = ring + (uint32_t)slot_i * a.lay_bytes;
        mbar_wait(bars + slot_i, parity);
        // this chunk's descriptor, written into the slot header by the producer
        const int64_t b0 = lds_s64(sbase), b1 = lds_s64(sbase + 8);
        const int64_t v0 = lds_s64(sbase + 16), p0 = lds_s64(sbase + 24);
        const int64_t pe = lds_s64(sbase + 32);
        const int flags = (int)lds_u32(sbase + 40);
        const uint32_t rec_off = lds_u32(sbase + 44);
        const bool head_mid = flags & 1;  // first block continues a panel of earlier chunks
        const bool slow = flags & 2;      // empty panels inside: search block_rowptr
        const int n = (int)(b1 - b0);
        int a0 = 0, a1 = n;  // blocks contributing to y
        if (GENERIC) {
            a0 = (int)(max(b0, b_lo) - b0);
            a1 = (int)(min(b1, b_hi) - b0);
        }
        // arrays are 256-byte aligned: a region's offset in its slot is its start mod 16
        const uint32_t a_bits = sbase + kHdr;  // words from granule (b0 + off32) >> 5
        const uint32_t a_rp = sbase + rec_off;
        const uint32_t a_col = sbase + a.lay_col + (uint32_t)((b0 * 4) & 15);
        const uint32_t a_mask = sbase + a.lay_mask + (uint32_t)((b0 * LB) & 15);
        const uint32_t a_val = sbase + a.lay_val + (uint32_t)((v0 * (int64_t)sizeof(T)) & 15);
        // the same values through a typed pointer (compiler-visible shared loads)
        const T *slot_values = reinterpret_cast<const T *>(smem + (a_val - smem_addr(smem)));
        const int sh0 = (int)((b0 + a.off32) & 31);

        if (MODE == 4 && !slow) {  // lane-per-block-row rounds (LBR plans)
            lbr_chunk<T, MT, R, GENERIC, SPC5_LBR_K>(a, c, p0, n, head_mid, sh0, a_bits, a_col,
                                                     a_mask, a_val, lane, x, y);
        } else if (MODE == 1) {
            fvr_chunk<T, MT, R, GENERIC, SPC5_FVR_U>(a, c, p0, n, head_mid, sh0, a_bits, a_rp,
                                                     a_col, a_mask, slot_values, lane, x, y);
        } else if (MODE == 6) {  // lane-per-panel chunks of a run plan
            lpp_chunk<T, MT, R, GENERIC, true>(a, c, p0, (int)(pe - p0), (flags >> 3) & 3,
                                               head_mid, a_rp, a_col, a_mask, a_val, lane, x, y);
        } else if (MODE < 4 && (MODE == 3 || (flags & 4))) {  // lane-per-panel chunk
            lpp_chunk<T, MT, R, GENERIC>(a, c, p0, (int)(pe - p0), (flags >> 3) & 3, head_mid,
                                         a_rp, a_col, a_mask, a_val, lane, x, y);
        } else if (MODE == 2 && (flags & 64)) {  // flat value ranges
            fvr_chunk<T, MT, R, GENERIC, SPC5_FVR_U>(a, c, p0, n, head_mid, sh0, a_bits, a_rp,
                                                     a_col, a_mask, slot_values, lane, x, y);
        } else if (MODE < 4 && !slow && SPC5_BLR) {  // balanced lane ranges
            blr_chunk<T, MT, R, GENERIC, SPC5_BLR_U>(a, c, p0, n, head_mid, sh0, sbase + 48, a_bits,
                                                           a_rp, a_col, a_mask, a_val, lane, x, y);
        } else {
            constexpr int KW = R <= 2 ? 4 : (R == 4 ? 2 : 1);  // windows per step
            lpb_chunk<T, MT, R, GENERIC, KW>(a, c, b0, p0, pe, n, a0, a1, head_mid, slow, sh0,
                                             a_bits, a_col, a_mask, a_val, lane, x, y);
        }
        // ---- release the slot and refill it with the chunk S ahead
        __syncwarp();
        if (lane == 0 && cn < c_end) {
            uint4 nA, nB;
            ir_staged(rec_stage, nA, nB);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue_chunk<T, LB>(a, nA, nB, sbase, bars + slot_i, pol);
        }
        if (++slot_i == S) {
            slot_i = 0;
            parity ^= 1u;
        }
    }
}

template <typename T, int R>
__global__ void fixup_kernel(const int64_t *__restrict__ split, int64_t num_split,
                             const int64_t *__restrict__ chunk_p, const SpmvArgs a) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= num_split) return;
    const int64_t c = split[i];
    const int64_t c_lo = a.range ? a.range[2] : a.c_lo, c_hi = a.range ? a.range[3] : a.c_hi;
    if (c < c_lo || c >= c_hi) return;
    const int64_t P = chunk_p[c];
    if (P < a.p_lo || P >= a.p_hi) return;
    if (i > 0 && split[i - 1] == c - 1 && chunk_p[c - 1] == P) return;  // not the first
    double s[R];
#pragma unroll
    for (int rr = 0; rr < R; ++rr) s[rr] = a.carry[c * R + rr];
    for (int64_t j = i + 1; j < num_split; ++j) {
        const int64_t cj = split[j];
        if (cj != split[j - 1] + 1 || cj >= c_hi || chunk_p[cj] != P) break;
#pragma unroll
        for (int rr = 0; rr < R; ++rr) s[rr] += a.carry[cj * R + rr];
    }
    // y already holds the panel's first-chunk part: add the carries (scaled
    // like every stored row) and mirror the result
    T *y = static_cast<T *>(a.y);
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
        const int64_t row = P * R + rr;
        if (row < a.num_rows) {
            const T sv = y[row] + (T)(s[rr] * a.yscale);
            y[row] = sv;
#pragma unroll 1
            for (int k = 0; k < a.nmirror; ++k)
                static_cast<T *>(a.mirror[k])[a.mirror_row0 + row] = sv;
        }
    }
}

template <typename K>
int launch_ring_kernel(K kernel, const Matrix &m, SpmvArgs a, int64_t nslots,
                       cudaStream_t st, int acc_per_warp = 0) {
    // 4 warps per CTA: with 168 registers per thread three CTAs share an SM
    // tuning knobs, read once per process: SPC5_WPC (warps per CTA), SPC5_NSLOT
    static const int env_wpc = [] {
        const char *e = getenv("SPC5_WPC");
        return e ? std::min(8, std::max(1, atoi(e))) : 0;
    }();
    static const int env_nslot = [] {
        const char *e = getenv("SPC5_NSLOT");
        return e ? std::min(kMaxSlots, std::max(2, atoi(e))) : 2;
    }();
    int wpc = env_wpc ? env_wpc : 4;
    const int S = env_nslot;
    a.nslot = S;
    // barriers + ring (+ the FVR row sums of R >= 4 kernels)
    a.acc_off = kRingOff + (uint32_t)(wpc * S) * a.lay_bytes;
    const size_t smem = kRingOff + (size_t)wpc * S * a.lay_bytes + (size_t)wpc * acc_per_warp;
    // launch shape per (kernel, warps, shared memory), computed once: the
    // attribute/occupancy queries cost more host time than a launch
    int per_sm = 0;
    {
        static std::mutex mu;
        static std::map<std::tuple<const void *, int, size_t>, int> cache;
        std::lock_guard<std::mutex> lk(mu);
        const auto key = std::make_tuple((const void *)kernel, wpc, smem);
        auto it = cache.find(key);
        if (it == cache.end()) {
            // (the checked build's static bounds words count against the 227 KB)
            SPC5_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           227 * 1024 - (SPC5_CHECKED ? 1024 : 0)));
            // SPC5_CARVEOUT: ask for no more shared memory than the ring of the
            // resident CTAs needs, so the rest stays L1 for the x gathers
            if (getenv("SPC5_CARVEOUT")) {
                int ps = 0;
                SPC5_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ps, kernel, wpc * 32, smem));
                const int pct = (int)std::min<size_t>(
                    100, (std::max(ps, 1) * (smem + 1024) * 100 + 228 * 1024 - 1) / (228 * 1024));
                SPC5_CUDA(cudaFuncSetAttribute(kernel,
                                               cudaFuncAttributePreferredSharedMemoryCarveout, pct));
            }
            SPC5_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, wpc * 32,
                                                                    smem));
            it = cache.emplace(key, std::max(per_sm, 1)).first;
            if (getenv("SPC5_PLAN_DEBUG"))
                fprintf(stderr, "spc5 launch: %d warps/CTA, %zu B shared, %d CTAs/SM\n", wpc,
                        smem, per_sm);
        }
        per_sm = it->second;
    }
    int64_t grid = std::max<int64_t>(cdiv(std::max<int64_t>(nslots, 1), wpc),
                                     a.accumulate ? 1 : cdiv(a.num_empty, 256));
    grid = std::min<int64_t>(grid, (int64_t)m.sm_count * per_sm);
    grid = std::max<int64_t>(grid, 1);
    // SPC5_X_WINDOW=1: an L2 persistence window over x as a launch attribute
    // (the north star's x-load item).  The set-aside is the
    // device maximum; a window larger than it persists with hit ratio
    // set-aside / window.  Off by default: the matrix stream is already
    // evict-first, and the A/B on configs 2/5 (profiles/SUMMARY_r2.md) shows no gain.
    static const int x_window = [] {
        const char *e = getenv("SPC5_X_WINDOW");
        return e ? atoi(e) : 0;
    }();
    if (x_window) {
        static int max_window = 0, max_persist = 0;
        static std::once_flag once;
        std::call_once(once, [] {
            int dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, dev);
            cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev);
            if (max_persist > 0) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, max_persist);
            if (getenv("SPC5_PLAN_DEBUG"))
                fprintf(stderr, "spc5 x window: max window %d B, persisting set-aside %d B\n",
                        max_window, max_persist);
        });
        const size_t xb = (size_t)m.num_cols * (m.precision == SPC5_F64 ? 8 : 4);
        const size_t wb = std::min<size_t>(xb, (size_t)std::max(max_window, 0));
        if (wb && max_persist > 0) {
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeAccessPolicyWindow;
            attr[0].val.accessPolicyWindow.base_ptr = const_cast<void *>(a.x);
            attr[0].val.accessPolicyWindow.num_bytes = wb;
            attr[0].val.accessPolicyWindow.hitRatio =
                (float)std::min(1.0, (double)max_persist / (double)wb);
            attr[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
            attr[0].val.accessPolicyWindow.missProp = cudaAccessPropertyNormal;
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3((unsigned)grid);
            cfg.blockDim = dim3((unsigned)(wpc * 32));
            cfg.dynamicSmemBytes = smem;
            cfg.stream = st;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            SPC5_CUDA(cudaLaunchKernelEx(&cfg, kernel, a));
            return SPC5_OK;
        }
    }
    kernel<<<(unsigned)grid, wpc * 32, smem, st>>>(a);
    SPC5_CUDA(cudaGetLastError());
    return SPC5_OK;
}

template <typename T, typename MT, int R>
int launch_typed(const Matrix &m, const SpmvArgs &a, cudaStream_t st) {
    const Plan &P = m.plan;
    int launches = 1;
    const int64_t nc = a.c_hi - a.c_lo;
    constexpr int ACC = R == 8 ? R * 256 : 0;  // FVR row sums per warp (kernels with FVR code)
    if (P.lbr) {
        if (a.p_lo == 0 && a.p_hi == m.num_panels)
            SPC5_TRY(launch_ring_kernel(spmv_kernel<T, MT, R, false, 4>, m, a, nc, st));
        else
            SPC5_TRY(launch_ring_kernel(spmv_kernel<T, MT, R, true, 4>, m, a, nc, st));
    } else if (a.p_lo == 0 && a.p_hi == m.num_panels) {  // full product: the plan's modes only
        if (P.num_fvr == P.num_chunks)
            SPC5_TRY(launch_ring_kernel(spmv_kernel<T, MT, R, false, 1>, m, a, nc, st, ACC));
        else if (P.num_lpp == P.num_chunks && P.runs)
            SPC5_TRY(launch_ring_kernel(spmv_kernel<T, MT, R, false, 6>, m, a, nc, st));
        else if (P.num_lpp == P.num_chunks)
            SPC5_TRY(launch_ring_kernel(spmv_kernel<T, MT, R, false, 3>, m, a, nc, st));
        else if (P.num_fvr == 0)
            SPC5_TRY(launch_ring_kernel(spmv_kernel<T, MT, R, false, 0>, m, a, nc, st));
        else
            SPC5_TRY(launch_ring_kernel(spmv_kernel<T, MT, R, false, 2>, m, a, nc, st, ACC));
    } else {
        SPC5_TRY(launch_ring_kernel(spmv_kernel<T, MT, R, true, 2>, m, a, nc, st, ACC));
    }
    if (P.num_split) {
        fixup_kernel<T, R><<<(unsigned)cdiv(P.num_split, 128), 128, 0, st>>>(
            P.split_chunks, P.num_split, P.chunk_p, a);
        SPC5_CUDA(cudaGetLastError());
        ++launches;
    }
    note_launches(launches);
    return SPC5_OK;
}

}  // namespace
}  // namespace spc5
