/*
 * spc5_b200.h -- C ABI of the B200-native SPC5 beta(r,c) SpMV library
 * (libspc5_b200.so, built from paper_2307_14774_b200/csrc/).
 *
 * Plain pointers, sizes and int status codes; no torch or C++ types.  Every
 * entry point replaces one function of the reference Python package
 * /root/reference/pkg/src/spc5 (cited per function).  INTEGRATION.md shows the
 * ctypes binding the reference side would add.
 *
 * Conventions
 *  - precision: SPC5_F32 = 0, SPC5_F64 = 1 (the save_spc5 header byte,
 *    blocks.py:240-243).
 *  - "d_" pointers are device memory of the current device, "h_" host memory.
 *  - stream: a cudaStream_t passed as void* (NULL = legacy default stream).
 *    Work is stream ordered; calls that must return a host-visible result
 *    (sizes, ranges, status of a validation) synchronise that stream.
 *  - All functions return SPC5_OK (0) or an error status; the message of the
 *    last error on the calling thread is spc5_last_error().  Status -> Python
 *    exception mapping mirrors the reference:
 *      SPC5_EINVAL  -> ValueError   (bad r/vs, bad dtype, short x/y, bad CSR,
 *                                    mask bits beyond vs; blocks.py:89-93,
 *                                    kernels.py:99-103, 219-223)
 *      SPC5_ECURSOR -> RuntimeError (sum of popcounts != nnz; kernels.py:211-212)
 *      SPC5_EINDEX  -> IndexError   (set bit addresses a column >= num_cols;
 *                                    vlane.py:58-77)
 *      SPC5_ECUDA / SPC5_ENOMEM -> RuntimeError
 *  - A matrix handle may be used from several threads and streams at once
 *    (SPEC.md:373-374): the plan is built once and then only read; products
 *    on different streams use different scratch (carry slots of split
 *    chunks, the device-resolved range of a range product), made on a
 *    stream's first product; spc5_spmv_host calls on one handle are
 *    serialised (one staging-buffer set per handle).  Products issued while
 *    a stream is being captured into a CUDA graph use the handle's graph
 *    scratch: replays of two graphs holding products of the same handle must
 *    not overlap.
 *  - Allocation: converted matrices are planned at construction; imported
 *    ones by spc5_prepare or on their first product (which then validates,
 *    allocates and synchronises).  spc5_prepare(m, stream) also makes that
 *    stream's scratch, after which products on it never allocate or
 *    synchronise and may be captured.  spc5_spmv_host allocates its staging
 *    buffers on first use.  The plan depends on the structure arrays
 *    (rowptr, colidx, masks) only: values may be rewritten in place between
 *    products, a structure change needs a new handle.
 */
#ifndef SPC5_B200_H
#define SPC5_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPC5_OK 0
#define SPC5_EINVAL 1
#define SPC5_ECURSOR 2
#define SPC5_EINDEX 3
#define SPC5_ECUDA 4
#define SPC5_ENOMEM 5

#define SPC5_F32 0
#define SPC5_F64 1

typedef struct spc5_matrix *spc5_matrix_t;

typedef struct spc5_info {
    int64_t num_rows, num_cols, num_panels, num_blocks, nnz;
    int32_t r, vs, precision, mask_bytes;
    int64_t block_base;  /* global index of block 0 (row-panel shards), else 0 */
    int64_t num_chunks;  /* work units of the SpMV plan                        */
    int64_t num_split_chunks; /* chunks that start inside a panel (carry path) */
    int64_t footprint_bytes;  /* filling_stats(s).footprint_bytes, blocks.py:180-183 */
} spc5_info_t;

/* Library identity / diagnostics. */
int spc5_version(void);
const char *spc5_last_error(void);
int spc5_device_count(int *count);

/*
 * csr_to_spc5 (blocks.py:96-143) on the GPU.  CSR arrays are device memory
 * (row_ptr int64[num_rows+1], col_idx int32[nnz] strictly increasing per row,
 * values f32/f64[nnz]).  block_base: global block index of this matrix's first
 * block when it is a row-panel shard of a larger matrix (0 otherwise); it only
 * keeps the warp windows on the global block grid, so a shard's rows agree
 * with the full matrix's y to <= 1e-15 relative.  The result owns its device
 * arrays.
 */
int spc5_convert_csr(int64_t num_rows, int64_t num_cols, int64_t nnz, int precision,
                     int r, int vs, const int64_t *d_row_ptr, const int32_t *d_col_idx,
                     const void *d_values, int64_t block_base, void *stream,
                     spc5_matrix_t *out);

/*
 * Wrap four existing format arrays (the Spc5Matrix fields, blocks.py:55-62):
 * rowptr int64[num_panels+1], colidx uint32[nb], masks u8 (vs<=8) / u16 [nb*r],
 * values [nnz].  from_host != 0: the pointers are host memory (copied H2D).
 * The arrays are validated like the reference kernels would on first use
 * (status mapping above); the copy is owned by the handle.
 */
int spc5_import(int64_t num_rows, int64_t num_cols, int r, int vs, int precision,
                int64_t num_blocks, int64_t nnz, const int64_t *rowptr,
                const uint32_t *colidx, const void *masks, const void *values,
                int from_host, int64_t block_base, void *stream, spc5_matrix_t *out);

int spc5_info(spc5_matrix_t m, spc5_info_t *info);

/*
 * Device times (CUDA events, ms) of the spc5_convert_csr call that built m:
 * the K1 count pass, the K1 fill pass (incl. the r = 1 value copy) and the
 * SpMV plan build.  Zeros for imported matrices.  Measurement only; the
 * reference times conversion with perf_counter around csr_to_spc5
 * (bench.py:158-160).
 */
int spc5_convert_timing(spc5_matrix_t m, double *k1_count_ms, double *k1_fill_ms,
                        double *plan_ms);

/*
 * Build the SpMV plan now (validating imported arrays, status mapping above).
 * Converted matrices are planned at construction; imported ones on their
 * first product or here.  After it returns, spc5_spmv never allocates or
 * synchronises and may be captured in a CUDA graph.
 */
int spc5_prepare(spc5_matrix_t m, void *stream);

/* Copy the four arrays out (to_host != 0: host buffers; else device buffers). */
int spc5_export(spc5_matrix_t m, int64_t *rowptr, uint32_t *colidx, void *masks,
                void *values, int to_host, void *stream);

/* Device pointers of the handle's arrays (valid until spc5_free). */
int spc5_device_arrays(spc5_matrix_t m, const int64_t **rowptr, const uint32_t **colidx,
                       const void **masks, const void **values);

/*
 * y = A.x (accumulate == 0) or y += A.x (accumulate != 0), x/y device arrays
 * in the matrix precision; only y[0:num_rows] is written.  Replaces
 * spmv_spc5_scalar / spmv_spc5_vector (kernels.py:205-230).  Never
 * allocates; safe inside CUDA-graph capture.
 */
int spc5_spmv(spc5_matrix_t m, const void *d_x, void *d_y, int accumulate, void *stream);

/*
 * Iterated products over several GPUs, fused exchange: y = scale * A.x on
 * this rank's row shard (y = its slice of the next x), and every stored row
 * is also written to d_peer_bases[k][row0 + row] -- the next-x buffers of
 * the peer GPUs (NVLink peer or symmetric-memory pointers), so no separate
 * all-gather follows the product.  scale should be exact (a power of two).
 * The caller orders iterations with a cross-GPU barrier.  Replaces the
 * product + allgather of the iterated config-5 form.
 */
int spc5_spmv_mirrored(spc5_matrix_t m, const void *d_x, void *d_y, double scale,
                       const void *const *d_peer_bases, int npeers, int64_t row0, void *stream);

/*
 * Same product restricted to the panel range [panel_lo, panel_hi): rows
 * [panel_lo*r, min(panel_hi*r, num_rows)) of y are written, nothing else.
 * One worker of spmv_parallel (parallel.py:55-92); results are bitwise equal
 * to the full product's rows.  The range's block and chunk bounds are
 * resolved on the device (a one-warp search launched before K2): no host
 * synchronisation, capturable.
 */
int spc5_spmv_panels(spc5_matrix_t m, int64_t panel_lo, int64_t panel_hi, const void *d_x,
                     void *d_y, int accumulate, void *stream);

/*
 * End-to-end product on HOST buffers: H2D copy of x (and of y when
 * accumulating), the kernel, D2H copy of y, stream synchronised.  The
 * reference-facing call of the e2e benchmark leg.
 */
int spc5_spmv_host(spc5_matrix_t m, const void *h_x, void *h_y, int accumulate, void *stream);

/* partition_by_nnz (parallel.py:31-52): h_ranges = int64[2*workers] (lo, hi). */
int spc5_partition_by_nnz(spc5_matrix_t m, int workers, int64_t *h_ranges, void *stream);

/* block_value_offsets (kernels.py:91-96) into device int64[num_blocks+1]. */
int spc5_block_value_offsets(spc5_matrix_t m, int64_t *d_offsets, void *stream);

/*
 * validate_spc5 (blocks.py:201-232) on the device: returns SPC5_OK or
 * SPC5_EINVAL with the reference's message for the first violated invariant.
 */
int spc5_validate(spc5_matrix_t m, void *stream);

/* spc5_to_csr (blocks.py:146-168): d_row_ptr int64[num_rows+1], d_col_idx int32[nnz], d_values[nnz]. */
int spc5_to_csr(spc5_matrix_t m, int64_t *d_row_ptr, int32_t *d_col_idx, void *d_values,
                void *stream);

int spc5_free(spc5_matrix_t m);

/*
 * Exact row products of a device CSR (csr_reference, kernels.py:233-250):
 * products in the matrix precision, summed in double-double; d_y / d_abs are
 * float64[num_rows] (rounded exact sum, exact sum of |products|).
 */
int spc5_csr_exact(int64_t num_rows, int precision, const int64_t *d_row_ptr,
                   const int32_t *d_col_idx, const void *d_values, const void *d_x,
                   double *d_y, double *d_abs, void *stream);

/*
 * Workload generator (BASELINE configs 2 and 5): rows [row_lo, row_hi) of the
 * 27-point stencil on an n^3 grid, position-keyed U(-1,1) values, diagonal
 * `diag` (paper_2307_14774_b200/workloads.py is the bit-identical host twin).
 * Two steps: row pointers (int64[rows+1]), then columns/values.
 */
int spc5_gen_stencil27_rowptr(int64_t n, int64_t row_lo, int64_t row_hi, int64_t *d_row_ptr,
                              void *stream);
int spc5_gen_stencil27_fill(int64_t n, int64_t row_lo, int64_t row_hi, int precision,
                            uint64_t seed, double diag, const int64_t *d_row_ptr,
                            int32_t *d_col_idx, void *d_values, void *stream);
/*
 * The same stencil on an n x n x nz box (nz = n is the cube above): the
 * weak-scaling workload of bench.py --gpus N, where rank k owns z-slab k of an
 * n x n x (n * N) box, i.e. one config-2 cube of rows per GPU.
 */
int spc5_gen_stencil27_box_rowptr(int64_t n, int64_t nz, int64_t row_lo, int64_t row_hi,
                                  int64_t *d_row_ptr, void *stream);
int spc5_gen_stencil27_box_fill(int64_t n, int64_t nz, int64_t row_lo, int64_t row_hi,
                                int precision, uint64_t seed, double diag,
                                const int64_t *d_row_ptr, int32_t *d_col_idx, void *d_values,
                                void *stream);

/*
 * Workload generator, BASELINE config 3: rows [row_lo, row_hi) of the n x n
 * power-law matrix.  Row i draws its length from d_len_table (2^table_bits
 * lognormal quantiles, workloads.py:powerlaw_len_table), then 80 % of its
 * columns stratified over i +- 4096 and the rest stratified over [0, n),
 * merged, duplicates dropped; values U(-1,1) position keyed.  Host twin:
 * workloads.py:powerlaw_rows.
 */
int spc5_gen_powerlaw_rowptr(int64_t n, int64_t row_lo, int64_t row_hi, uint64_t seed,
                             const int32_t *d_len_table, int table_bits, int64_t *d_row_ptr,
                             void *stream);
int spc5_gen_powerlaw_fill(int64_t n, int64_t row_lo, int64_t row_hi, int precision,
                           uint64_t seed, const int32_t *d_len_table, int table_bits,
                           const int64_t *d_row_ptr, int32_t *d_col_idx, void *d_values,
                           void *stream);

/*
 * Workload generator, BASELINE config 4: rows [row_lo, row_hi) of the
 * FEM-like matrix over `nodes` nodes x 3 dof.  Node q couples to itself and
 * 26 nodes stratified over q +- 2048; row 3q+d holds the dense 3x3 blocks of
 * those 27 nodes (81 entries), values ~N(0,1) (Irwin-Hall of 4 keyed
 * uniforms).  Host twin: workloads.py:fem_rows.
 */
int spc5_gen_fem_rowptr(int64_t nodes, int64_t row_lo, int64_t row_hi, int64_t *d_row_ptr,
                        void *stream);
int spc5_gen_fem_fill(int64_t nodes, int64_t row_lo, int64_t row_hi, int precision,
                      uint64_t seed, const int64_t *d_row_ptr, int32_t *d_col_idx,
                      void *d_values, void *stream);

/*
 * Multi-GPU row-panel sharding (one process per GPU, NCCL), the C-ABI form of
 * spmv_parallel's partitioned product (parallel.py:55-92) and of BASELINE
 * config 5's iterated loop.  NCCL (libnccl.so.2) is loaded on first use.
 *
 *  spc5_mg_unique_id   rank 0 makes the 128-byte NCCL id; the caller ships it
 *                      to the other ranks (MPI, a file, torch.distributed...).
 *  spc5_mg_init        one communicator per rank on the current CUDA device.
 *  spc5_mg_partition   partition_by_nnz (parallel.py:31-52) of a CSR's panels
 *                      from its DEVICE row pointers alone (int64[num_rows+1]):
 *                      h_ranges = int64[2*workers] panel ranges (lo, hi),
 *                      identical to the reference's for the converted matrix.
 *  spc5_mg_shard       attach this rank's matrix (rows h_row_ranges[2*rank] ..
 *                      h_row_ranges[2*rank+1] of a square matrix, converted on
 *                      its own with spc5_convert_csr; borrowed, not freed);
 *                      h_row_ranges = int64[2*nranks] ROW ranges of all ranks.
 *  spc5_mg_spmv_step   x_next = scale * A . x: the local K2 writes this rank's
 *                      rows of x_next, then one NCCL group of point-to-point
 *                      sends/receives all-gathers the slices (unequal sizes),
 *                      stream ordered.  x and x_next are full-length device
 *                      vectors on every rank.
 */
typedef struct spc5_mg *spc5_mg_t;
int spc5_mg_unique_id(void *id /* 128 bytes */);
int spc5_mg_init(const void *id, int nranks, int rank, spc5_mg_t *out);
int spc5_mg_partition(const int64_t *d_row_ptr, int64_t num_rows, int r, int workers,
                      int64_t *h_ranges, void *stream);
int spc5_mg_shard(spc5_mg_t mg, spc5_matrix_t local, const int64_t *h_row_ranges);
int spc5_mg_spmv_step(spc5_mg_t mg, const void *d_x, void *d_x_next, double scale,
                      void *stream);
int spc5_mg_free(spc5_mg_t mg);

/* Number of kernel launches the last spc5_spmv* call on this thread issued. */
int spc5_last_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* SPC5_B200_H */
