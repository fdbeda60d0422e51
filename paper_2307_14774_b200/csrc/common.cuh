// common.cuh -- shared types of the B200 SPC5 library (internal, C++).
//
// Layout in HBM: exactly the reference Spc5Matrix
// arrays (blocks.py:55-62) -- block_rowptr int64[num_panels+1], block_colidx
// uint32[nb], block_masks u8|u16[nb*r] (row-major within a block), values
// f32|f64[nnz] packed block-major / row-within-block / ascending column.
// Everything else on the handle is a derived plan (chunk descriptors,
// per-tile popcount prefix, empty-panel list, carry slots), built once.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/spc5_b200.h"

namespace spc5 {

constexpr int kTile = 1024;       // blocks per popcount-prefix tile

struct Plan {
    bool built = false;
    int64_t num_chunks = 0;
    int64_t *chunk_b = nullptr;  // [num_chunks+1] first block of each chunk (+ nb)
    int64_t *chunk_v = nullptr;  // [num_chunks+1] value offset of that block (+ nnz)
    int64_t *chunk_p = nullptr;  // [num_chunks+1] panel containing that block (+ num_panels)
    int64_t *h_chunk_b = nullptr;  // host copy of chunk_b (range launches)
    int64_t num_split = 0;       // chunks whose first block is inside a panel
    int64_t *split_chunks = nullptr;  // [num_split] their indices, ascending
    double *carry = nullptr;     // [num_chunks*r] head-segment partials of split chunks
    int64_t num_empty = 0;
    int64_t *empty_panels = nullptr;  // [num_empty] panels with no block
    int64_t num_tiles = 0;
    int64_t *tile_prefix = nullptr;   // [num_tiles+1] value offset at tile starts
    // ring slots: one chunk per shared-memory slot
    int64_t chunk_target = 0;       // blocks per chunk target (snapped to panel starts)
    int64_t split_len = 256;        // long panels are cut at global multiples of this
    int64_t max_chunk_blocks = 0, max_chunk_values = 0;
    int64_t max_lpp_panels = 0;     // panels of the largest lane-per-panel chunk
    int64_t num_fvr = 0;            // flat value-range chunks (kernel variant choice)
    int64_t num_lpp = 0;            // lane-per-panel-row chunks
    bool lbr = false;               // lane-per-block-row rounds over exact chunk cuts (plan.cu)
    bool runs = false;              // every row mask is one contiguous run of bits (K2 RUN gathers)
    int64_t lay_rp = 0, lay_col = 0, lay_mask = 0, lay_val = 0;  // slot: hdr|bits|rec|col|mask|val
    int slot_bytes = 0;
    int64_t num_granules = 0;
    uint32_t *pstart_bits = nullptr;  // [num_granules] bit i of word g: block 32g-off32+i starts a panel
    uint8_t *chunk_flags = nullptr;   // [num_chunks] bit0: starts inside a panel, bit1: has empty panels
    uint8_t *blob = nullptr;          // per-chunk metadata blobs (plan.cu blob_fill_kernel)
    uint4 *issue_rec = nullptr;       // [2*num_chunks] bulk-copy sources/sizes per chunk
};

struct Matrix {
    int64_t num_rows = 0, num_cols = 0, num_panels = 0, num_blocks = 0, nnz = 0;
    int r = 1, vs = 8, precision = SPC5_F64;
    int64_t block_base = 0;
    int device = 0;
    int64_t *rowptr = nullptr;
    uint32_t *colidx = nullptr;
    void *masks = nullptr;
    void *values = nullptr;
    Plan plan;
    // scratch of the host-buffer path
    void *dx = nullptr, *dy = nullptr;
    int sm_count = 148;
    // CUDA-event times of the conversion that built this matrix (ms; 0 for
    // imported matrices): K1 count pass, K1 fill pass (+ the r = 1 value
    // copy), plan build -- spc5_convert_timing
    float k1_count_ms = 0.f, k1_fill_ms = 0.f, plan_ms = 0.f;

    int mask_bytes() const { return vs <= 8 ? 1 : 2; }
    int value_bytes() const { return precision == SPC5_F64 ? 8 : 4; }
};

// ---- error plumbing -------------------------------------------------------
void set_error(const std::string &msg);
int fail(int status, const std::string &msg);
int cuda_fail(cudaError_t e, const char *what);
void note_launches(int n);

#define SPC5_CUDA(call)                                              \
    do {                                                             \
        cudaError_t _e = (call);                                     \
        if (_e != cudaSuccess) return ::spc5::cuda_fail(_e, #call);  \
    } while (0)

#define SPC5_TRY(call)               \
    do {                             \
        int _s = (call);             \
        if (_s != SPC5_OK) return _s; \
    } while (0)

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ---- device helpers -------------------------------------------------------
__device__ __forceinline__ uint32_t load_mask(const void *masks, int64_t i, int vs) {
    return vs <= 8 ? (uint32_t)((const uint8_t *)masks)[i]
                   : (uint32_t)((const uint16_t *)masks)[i];
}

// ---- launchers implemented across the .cu files ----------------------------
int convert_csr(Matrix &m, const int64_t *d_row_ptr, const int32_t *d_col_idx,
                const void *d_values, cudaStream_t st);
int build_plan(Matrix &m, bool validate, cudaStream_t st);
void free_plan(Plan &p);
// fused exchange of iterated products: y rows also stored at ptr[i][row0 + row]
struct Mirror {
    void *ptr[8];
    int n = 0;
    int64_t row0 = 0;
    double scale = 1.0;
};
// Per-call mutable device state of a product, one set per stream (capi.cu
// scratch_for): the carry slots of split chunks and, for range products, the
// device-resolved block/chunk range.  Calls on different streams never share
// it, so one handle is safe under concurrent products.
struct Scratch {
    double *carry = nullptr;   // [num_chunks * r] when the plan has split chunks
    int64_t *range = nullptr;  // [4]: b_lo, b_hi, c_lo, c_hi of a range product
};
// blk: the range's block bounds when the caller knows them (else they are
// resolved on the device into scratch.range, with no host synchronisation)
int launch_spmv(const Matrix &m, int64_t p_lo, int64_t p_hi, const void *x, void *y,
                int accumulate, cudaStream_t st, const Scratch &scratch,
                const Mirror *mirror = nullptr, const int64_t *blk = nullptr);
// host-buffer pipeline: K nnz-balanced panel stages, their block bounds and
// the x prefix (columns) each stage reads
int host_stages(const Matrix &m, int K, int64_t *p, int64_t *b, int64_t *need, cudaStream_t st);
int partition_by_nnz(const Matrix &m, int workers, int64_t *h_ranges, cudaStream_t st);
int block_value_offsets(const Matrix &m, int64_t *d_offsets, cudaStream_t st);
int validate_structure(const Matrix &m, cudaStream_t st);
int to_csr(const Matrix &m, int64_t *d_row_ptr, int32_t *d_col_idx, void *d_values,
           cudaStream_t st);
int csr_exact(int64_t num_rows, int precision, const int64_t *rp, const int32_t *ci,
              const void *v, const void *x, double *y, double *a, cudaStream_t st);
int gen_stencil27_rowptr(int64_t n, int64_t nz, int64_t lo, int64_t hi, int64_t *rp,
                         cudaStream_t st);
int gen_powerlaw_rowptr(int64_t n, int64_t lo, int64_t hi, uint64_t seed, const int32_t *table,
                        int bits, int64_t *rp, cudaStream_t st);
int gen_powerlaw_fill(int64_t n, int64_t lo, int64_t hi, int precision, uint64_t seed,
                      const int32_t *table, int bits, const int64_t *rp, int32_t *ci, void *v,
                      cudaStream_t st);
int gen_fem_rowptr(int64_t nodes, int64_t lo, int64_t hi, int64_t *rp, cudaStream_t st);
int gen_fem_fill(int64_t nodes, int64_t lo, int64_t hi, int precision, uint64_t seed,
                 const int64_t *rp, int32_t *ci, void *v, cudaStream_t st);
int gen_stencil27_fill(int64_t n, int64_t nz, int64_t lo, int64_t hi, int precision,
                       uint64_t seed, double diag, const int64_t *rp, int32_t *ci, void *v,
                       cudaStream_t st);

// device allocation helpers (stream-ordered for temporaries)
int dev_alloc(void **p, size_t bytes);
template <typename T>
int dev_alloc(T **p, size_t count) {
    return dev_alloc(reinterpret_cast<void **>(p), count * sizeof(T) + 64);
}
void dev_free(void *p);

}  // namespace spc5
