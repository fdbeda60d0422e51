// capi.cu -- the extern "C" boundary (include/spc5_b200.h).
//
// Handles own their device arrays; every entry point validates its arguments
// the way the reference Python functions do (blocks.py:89-93,
// kernels.py:99-103, 219-223) and reports through an int status plus a
// thread-local message (spc5_last_error).
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>
#include <map>
#include <mutex>
#include <new>
#include <string>
#include <thread>
#include <vector>
#include <cstring>

#include "common.cuh"

// host-buffer pipeline of spc5_spmv_host (built on first use)
struct HostPipe {
    int K = 0;                 // stages (0: not built)
    int64_t p[9], b[9], need[8];
    cudaStream_t h2d = nullptr, d2h = nullptr, comp = nullptr;
    cudaEvent_t start = nullptr, done = nullptr, xin[8], yout[8], ycopied[8];
};

// A handle: the matrix, its plan (built once, then read-only) and the
// per-stream mutable scratch of its products.  Thread safety (header
// contract): the plan is published through `ready` (acquire/release) under
// plan_mu; products on different streams use different Scratch (carry slots,
// device range), created on a stream's first product; the host-buffer
// pipeline (one set of staging buffers and streams per handle) is serialised
// by host_mu.
struct spc5_matrix {
    spc5::Matrix m;
    std::mutex plan_mu;
    std::atomic<bool> ready{false};
    std::mutex scratch_mu;
    std::map<cudaStream_t, spc5::Scratch> scratch;  // per stream
    spc5::Scratch graph_scratch;  // products issued during stream capture
    std::mutex host_mu;
    HostPipe pipe;
    void free_scratch() {
        for (auto &kv : scratch) {
            spc5::dev_free(kv.second.carry);
            spc5::dev_free(kv.second.range);
        }
        scratch.clear();
        spc5::dev_free(graph_scratch.carry);
        spc5::dev_free(graph_scratch.range);
        graph_scratch = spc5::Scratch{};
    }
    ~spc5_matrix() {
        free_scratch();
        if (pipe.K) {
            cudaStreamDestroy(pipe.h2d);
            cudaStreamDestroy(pipe.d2h);
            cudaStreamDestroy(pipe.comp);
            cudaEventDestroy(pipe.start);
            cudaEventDestroy(pipe.done);
            for (int k = 0; k < pipe.K; ++k) {
                cudaEventDestroy(pipe.xin[k]);
                cudaEventDestroy(pipe.yout[k]);
                cudaEventDestroy(pipe.ycopied[k]);
            }
        }
    }
};

namespace spc5 {

static thread_local std::string g_err;
static thread_local int g_launches = 0;

void set_error(const std::string &msg) { g_err = msg; }
int fail(int status, const std::string &msg) {
    g_err = msg;
    return status;
}
int cuda_fail(cudaError_t e, const char *what) {
    g_err = std::string("CUDA error ") + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) +
            ") in " + what;
    return e == cudaErrorMemoryAllocation ? SPC5_ENOMEM : SPC5_ECUDA;
}
void note_launches(int n) { g_launches += n; }

int dev_alloc(void **p, size_t bytes) {
    *p = nullptr;
    if (bytes == 0) bytes = 64;
    cudaError_t e = cudaMalloc(p, bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        *p = nullptr;
        return cuda_fail(e, "cudaMalloc");
    }
    return SPC5_OK;
}
void dev_free(void *p) {
    if (p) cudaFree(p);
}

static int check_shape(int r, int vs, int precision) {
    if (r != 1 && r != 2 && r != 4 && r != 8)
        return fail(SPC5_EINVAL, "r must be one of (1, 2, 4, 8), got " + std::to_string(r));
    if (vs != 4 && vs != 8 && vs != 16)
        return fail(SPC5_EINVAL, "vs must be one of (4, 8, 16), got " + std::to_string(vs));
    if (precision != SPC5_F32 && precision != SPC5_F64)
        return fail(SPC5_EINVAL, "precision must be 'f32' or 'f64'");
    return SPC5_OK;
}

static void free_matrix(Matrix &m) {
    free_plan(m.plan);
    dev_free(m.rowptr);
    dev_free(m.colidx);
    dev_free(m.masks);
    dev_free(m.values);
    dev_free(m.dx);
    dev_free(m.dy);
    m.rowptr = nullptr;
    m.colidx = nullptr;
    m.masks = m.values = m.dx = m.dy = nullptr;
}

static void init_common(Matrix &m, int64_t num_rows, int64_t num_cols, int r, int vs,
                        int precision, int64_t block_base) {
    m.num_rows = num_rows;
    m.num_cols = num_cols;
    m.r = r;
    m.vs = vs;
    m.precision = precision;
    m.num_panels = (num_rows + r - 1) / r;
    m.block_base = block_base;
    cudaGetDevice(&m.device);
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, m.device) == cudaSuccess &&
        sms > 0)
        m.sm_count = sms;
    cudaGetLastError();
}

static int alloc_scratch(const Matrix &m, Scratch *s) {
    if (m.plan.num_split) SPC5_TRY(dev_alloc(&s->carry, (size_t)m.plan.num_chunks * m.r));
    SPC5_TRY(dev_alloc(&s->range, 4));
    return SPC5_OK;
}

// Builds the plan once (validating imported arrays) and the scratch used by
// products issued during CUDA-graph capture (allocation is not capturable).
static int ensure_plan(spc5_matrix *h, cudaStream_t st) {
    if (h->ready.load(std::memory_order_acquire)) return SPC5_OK;
    std::lock_guard<std::mutex> lk(h->plan_mu);
    if (h->ready.load(std::memory_order_relaxed)) return SPC5_OK;
    int s = h->m.plan.built ? SPC5_OK : build_plan(h->m, /*validate=*/true, st);
    if (s == SPC5_OK) s = alloc_scratch(h->m, &h->graph_scratch);
    if (s != SPC5_OK) {
        std::string keep = g_err;
        free_plan(h->m.plan);
        h->free_scratch();
        g_err = keep;
        return s;
    }
    h->ready.store(true, std::memory_order_release);
    return SPC5_OK;
}

// The scratch of products on stream `st`: one set per stream, so concurrent
// products on different streams never share carry slots or range words
// (products on one stream are ordered by the stream).  A stream under
// capture gets the handle's graph scratch: replays of graphs holding
// products of the same handle must not run concurrently.
static int scratch_for(spc5_matrix *h, cudaStream_t st, Scratch *out) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess) {
        cudaGetLastError();
        cs = cudaStreamCaptureStatusNone;
    }
    if (cs != cudaStreamCaptureStatusNone) {
        *out = h->graph_scratch;
        return SPC5_OK;
    }
    std::lock_guard<std::mutex> lk(h->scratch_mu);
    auto it = h->scratch.find(st);
    if (it == h->scratch.end()) {
        Scratch s;
        int rc = alloc_scratch(h->m, &s);
        if (rc != SPC5_OK) {
            dev_free(s.carry);
            dev_free(s.range);
            return rc;
        }
        it = h->scratch.emplace(st, s).first;
    }
    *out = it->second;
    return SPC5_OK;
}

}  // namespace spc5

using namespace spc5;

extern "C" {

int spc5_version(void) { return 10000; }

const char *spc5_last_error(void) { return g_err.c_str(); }

int spc5_last_launch_count(void) { return g_launches; }

int spc5_device_count(int *count) {
    *count = 0;
    cudaError_t e = cudaGetDeviceCount(count);
    if (e != cudaSuccess) {
        cudaGetLastError();
        *count = 0;
        return cuda_fail(e, "cudaGetDeviceCount");
    }
    return SPC5_OK;
}

int spc5_convert_csr(int64_t num_rows, int64_t num_cols, int64_t nnz, int precision, int r,
                     int vs, const int64_t *d_row_ptr, const int32_t *d_col_idx,
                     const void *d_values, int64_t block_base, void *stream,
                     spc5_matrix_t *out) {
    g_launches = 0;
    *out = nullptr;
    SPC5_TRY(check_shape(r, vs, precision));
    if (num_rows < 0 || num_cols < 0 || nnz < 0)
        return fail(SPC5_EINVAL, "dimensions must be non-negative");
    if (num_cols > (int64_t)INT32_MAX + 1)
        return fail(SPC5_EINVAL, "num_cols exceeds the int32 column index range");
    auto *h = new (std::nothrow) spc5_matrix();
    if (!h) return fail(SPC5_ENOMEM, "out of host memory");
    Matrix &m = h->m;
    init_common(m, num_rows, num_cols, r, vs, precision, block_base);
    m.nnz = nnz;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int s = convert_csr(m, d_row_ptr, d_col_idx, d_values, st);
    if (s == SPC5_OK) {
        cudaEvent_t p0 = nullptr, p1 = nullptr;
        cudaEventCreate(&p0);
        cudaEventCreate(&p1);
        cudaEventRecord(p0, st);
        s = build_plan(m, /*validate=*/false, st);
        cudaEventRecord(p1, st);
        if (s == SPC5_OK && cudaEventSynchronize(p1) == cudaSuccess)
            cudaEventElapsedTime(&m.plan_ms, p0, p1);
        cudaEventDestroy(p0);
        cudaEventDestroy(p1);
    }
    if (s == SPC5_OK) s = ensure_plan(h, st);
    if (s != SPC5_OK) {
        std::string keep = g_err;
        h->free_scratch();
        free_matrix(m);
        delete h;
        g_err = keep;
        return s;
    }
    *out = h;
    return SPC5_OK;
}

int spc5_import(int64_t num_rows, int64_t num_cols, int r, int vs, int precision,
                int64_t num_blocks, int64_t nnz, const int64_t *rowptr, const uint32_t *colidx,
                const void *masks, const void *values, int from_host, int64_t block_base,
                void *stream, spc5_matrix_t *out) {
    g_launches = 0;
    *out = nullptr;
    SPC5_TRY(check_shape(r, vs, precision));
    if (num_rows < 0 || num_cols < 0 || nnz < 0 || num_blocks < 0)
        return fail(SPC5_EINVAL, "dimensions must be non-negative");
    auto *h = new (std::nothrow) spc5_matrix();
    if (!h) return fail(SPC5_ENOMEM, "out of host memory");
    Matrix &m = h->m;
    init_common(m, num_rows, num_cols, r, vs, precision, block_base);
    m.num_blocks = num_blocks;
    m.nnz = nnz;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const cudaMemcpyKind kind = from_host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
    auto body = [&]() -> int {
        SPC5_TRY(dev_alloc(&m.rowptr, (size_t)m.num_panels + 1));
        SPC5_TRY(dev_alloc(&m.colidx, (size_t)num_blocks));
        SPC5_TRY(dev_alloc(reinterpret_cast<uint8_t **>(&m.masks),
                           (size_t)(num_blocks * r * m.mask_bytes())));
        SPC5_TRY(dev_alloc(reinterpret_cast<uint8_t **>(&m.values),
                           (size_t)(nnz * m.value_bytes())));
        SPC5_CUDA(cudaMemcpyAsync(m.rowptr, rowptr, sizeof(int64_t) * (m.num_panels + 1), kind, st));
        if (num_blocks) {
            SPC5_CUDA(cudaMemcpyAsync(m.colidx, colidx, sizeof(uint32_t) * num_blocks, kind, st));
            SPC5_CUDA(cudaMemcpyAsync(m.masks, masks, (size_t)num_blocks * r * m.mask_bytes(),
                                      kind, st));
        }
        if (nnz)
            SPC5_CUDA(cudaMemcpyAsync(m.values, values, (size_t)nnz * m.value_bytes(), kind, st));
        SPC5_CUDA(cudaStreamSynchronize(st));
        return SPC5_OK;
    };
    int s = body();
    if (s != SPC5_OK) {
        std::string keep = g_err;
        free_matrix(m);
        delete h;
        g_err = keep;
        return s;
    }
    *out = h;
    return SPC5_OK;
}

int spc5_info(spc5_matrix_t h, spc5_info_t *info) {
    if (!h || !info) return fail(SPC5_EINVAL, "null handle");
    const Matrix &m = h->m;
    info->num_rows = m.num_rows;
    info->num_cols = m.num_cols;
    info->num_panels = m.num_panels;
    info->num_blocks = m.num_blocks;
    info->nnz = m.nnz;
    info->r = m.r;
    info->vs = m.vs;
    info->precision = m.precision;
    info->mask_bytes = m.mask_bytes();
    info->block_base = m.block_base;
    info->num_chunks = m.plan.num_chunks;
    info->num_split_chunks = m.plan.num_split;
    // blocks.py:180-183 (4-byte declared index width)
    info->footprint_bytes = m.nnz * m.value_bytes() + m.num_blocks * 4 +
                            m.num_blocks * m.r * m.mask_bytes() + (m.num_panels + 1) * 4;
    return SPC5_OK;
}

int spc5_convert_timing(spc5_matrix_t h, double *k1_count_ms, double *k1_fill_ms,
                        double *plan_ms) {
    if (!h) return fail(SPC5_EINVAL, "null handle");
    if (k1_count_ms) *k1_count_ms = h->m.k1_count_ms;
    if (k1_fill_ms) *k1_fill_ms = h->m.k1_fill_ms;
    if (plan_ms) *plan_ms = h->m.plan_ms;
    return SPC5_OK;
}

int spc5_prepare(spc5_matrix_t h, void *stream) {
    if (!h) return fail(SPC5_EINVAL, "null handle");
    g_launches = 0;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    SPC5_TRY(ensure_plan(h, st));
    Scratch sc;  // this stream's scratch now, so its products never allocate
    return scratch_for(h, st, &sc);
}

int spc5_export(spc5_matrix_t h, int64_t *rowptr, uint32_t *colidx, void *masks, void *values,
                int to_host, void *stream) {
    if (!h) return fail(SPC5_EINVAL, "null handle");
    const Matrix &m = h->m;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const cudaMemcpyKind kind = to_host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
    if (rowptr)
        SPC5_CUDA(cudaMemcpyAsync(rowptr, m.rowptr, sizeof(int64_t) * (m.num_panels + 1), kind, st));
    if (colidx && m.num_blocks)
        SPC5_CUDA(cudaMemcpyAsync(colidx, m.colidx, sizeof(uint32_t) * m.num_blocks, kind, st));
    if (masks && m.num_blocks)
        SPC5_CUDA(cudaMemcpyAsync(masks, m.masks, (size_t)m.num_blocks * m.r * m.mask_bytes(),
                                  kind, st));
    if (values && m.nnz)
        SPC5_CUDA(cudaMemcpyAsync(values, m.values, (size_t)m.nnz * m.value_bytes(), kind, st));
    SPC5_CUDA(cudaStreamSynchronize(st));
    return SPC5_OK;
}

int spc5_device_arrays(spc5_matrix_t h, const int64_t **rowptr, const uint32_t **colidx,
                       const void **masks, const void **values) {
    if (!h) return fail(SPC5_EINVAL, "null handle");
    if (rowptr) *rowptr = h->m.rowptr;
    if (colidx) *colidx = h->m.colidx;
    if (masks) *masks = h->m.masks;
    if (values) *values = h->m.values;
    return SPC5_OK;
}

int spc5_spmv(spc5_matrix_t h, const void *d_x, void *d_y, int accumulate, void *stream) {
    g_launches = 0;
    if (!h) return fail(SPC5_EINVAL, "null handle");
    if ((!d_x && h->m.num_cols) || (!d_y && h->m.num_rows))
        return fail(SPC5_EINVAL, "x/y must be non-null");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    SPC5_TRY(ensure_plan(h, st));
    Scratch sc;
    SPC5_TRY(scratch_for(h, st, &sc));
    return launch_spmv(h->m, 0, h->m.num_panels, d_x, d_y, accumulate, st, sc);
}

int spc5_spmv_mirrored(spc5_matrix_t h, const void *d_x, void *d_y, double scale,
                       const void *const *d_peer_bases, int npeers, int64_t row0, void *stream) {
    g_launches = 0;
    if (!h) return fail(SPC5_EINVAL, "null handle");
    if ((!d_x && h->m.num_cols) || (!d_y && h->m.num_rows))
        return fail(SPC5_EINVAL, "x/y must be non-null");
    if (npeers < 0 || npeers > 8 || (npeers && !d_peer_bases))
        return fail(SPC5_EINVAL, "npeers must be in [0, 8] with a peer pointer array");
    Mirror mi;
    mi.n = npeers;
    for (int k = 0; k < npeers; ++k) mi.ptr[k] = const_cast<void *>(d_peer_bases[k]);
    mi.row0 = row0;
    mi.scale = scale;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    SPC5_TRY(ensure_plan(h, st));
    Scratch sc;
    SPC5_TRY(scratch_for(h, st, &sc));
    return launch_spmv(h->m, 0, h->m.num_panels, d_x, d_y, 0, st, sc, &mi);
}

int spc5_spmv_panels(spc5_matrix_t h, int64_t panel_lo, int64_t panel_hi, const void *d_x,
                     void *d_y, int accumulate, void *stream) {
    g_launches = 0;
    if (!h) return fail(SPC5_EINVAL, "null handle");
    if (panel_lo < 0 || panel_hi < panel_lo || panel_hi > h->m.num_panels)
        return fail(SPC5_EINVAL, "panel range out of bounds");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    SPC5_TRY(ensure_plan(h, st));
    if (panel_lo == panel_hi) return SPC5_OK;
    Scratch sc;
    SPC5_TRY(scratch_for(h, st, &sc));
    return launch_spmv(h->m, panel_lo, panel_hi, d_x, d_y, accumulate, st, sc);
}

// End-to-end product on host buffers, pipelined over PCIe: K nnz-balanced
// panel stages; x lands in pieces (stage k starts as soon as the columns it
// reads are on the device), each stage's rows go back while later stages
// compute.  Copies in, products and copies out run on three streams of the
// handle (the copy engines run both directions at once), ordered after the
// caller's stream and joined back into it.  Stages are range products
// (spc5_spmv_panels), so y is bitwise the one-shot product's.  Measured on
// config 2, beta(1,8): 0.55 ms per call against 0.73 ms for copy, product,
// copy in sequence (x lands slower while the products saturate HBM).
// Pageable host buffers (ordinary numpy arrays, what a drop-in caller of
// kernels.py:119-129 passes).  cudaMemcpyAsync from pageable memory goes
// through the driver's single-threaded staging at ~10 GB/s (45 GFLOP/s end to
// end on the 400^3 matrix against 262 from pinned buffers), so large pageable
// x / y are staged here instead: a team of host threads copies each pipeline
// stage's piece of x into a process-wide pinned buffer while the previous
// piece is on the wire, and copies each stage's y rows out of the pinned
// buffer as its device-to-host copy completes.
namespace {
struct PinnedStage {
    std::mutex mu;  // one pageable host product at a time per process
    void *x = nullptr, *y = nullptr;
    size_t xcap = 0, ycap = 0;
    int grow(void **p, size_t *cap, size_t bytes) {
        if (*cap >= bytes) return SPC5_OK;
        if (*p) cudaFreeHost(*p);
        *p = nullptr;
        *cap = 0;
        SPC5_CUDA(cudaHostAlloc(p, bytes, cudaHostAllocDefault));
        *cap = bytes;
        return SPC5_OK;
    }
};
PinnedStage g_stage;

bool is_pageable(const void *p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return true;
    }
    return a.type == cudaMemoryTypeUnregistered;
}

int host_threads() {
    static const int n = [] {
        if (const char *e = getenv("SPC5_HOST_THREADS")) return std::min(32, std::max(1, atoi(e)));
        const unsigned hc = std::thread::hardware_concurrency();
        return (int)std::min(8u, std::max(1u, hc / 2));
    }();
    return n;
}

// thread t of T copies its 64-byte-aligned share of [0, bytes)
void copy_share(char *dst, const char *src, size_t bytes, int t, int T) {
    const size_t lo = (bytes * (size_t)t / T) & ~(size_t)63, hi = t == T - 1 ? bytes
                                                                            : (bytes * (size_t)(t + 1) / T) & ~(size_t)63;
    if (hi > lo) std::memcpy(dst + lo, src + lo, hi - lo);
}
}  // namespace

int spc5_spmv_host(spc5_matrix_t h, const void *h_x, void *h_y, int accumulate, void *stream) {
    g_launches = 0;
    if (!h) return fail(SPC5_EINVAL, "null handle");
    Matrix &m = h->m;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    SPC5_TRY(ensure_plan(h, st));
    const int vb = m.value_bytes();
    const size_t xb = (size_t)m.num_cols * vb, yb = (size_t)m.num_rows * vb;
    HostPipe &hp = h->pipe;
    // one staging buffer pair and stream set per handle: concurrent host
    // products of one handle run one after the other
    std::lock_guard<std::mutex> host_lk(h->host_mu);
    {
        if (!m.dx) SPC5_TRY(dev_alloc(&m.dx, xb));
        if (!m.dy) SPC5_TRY(dev_alloc(&m.dy, yb));
        if (!hp.K) {
            // a few MB per stage at least, else one stage
            int K = std::min<int64_t>(8, std::max<int64_t>(1, (int64_t)(xb + yb) >> 22));
            if (const char *e = getenv("SPC5_HOST_STAGES")) K = std::min(8, std::max(1, atoi(e)));
            SPC5_TRY(host_stages(m, K, hp.p, hp.b, hp.need, st));
            SPC5_CUDA(cudaStreamCreateWithFlags(&hp.h2d, cudaStreamNonBlocking));
            SPC5_CUDA(cudaStreamCreateWithFlags(&hp.d2h, cudaStreamNonBlocking));
            SPC5_CUDA(cudaStreamCreateWithFlags(&hp.comp, cudaStreamNonBlocking));
            SPC5_CUDA(cudaEventCreateWithFlags(&hp.start, cudaEventDisableTiming));
            SPC5_CUDA(cudaEventCreateWithFlags(&hp.done, cudaEventDisableTiming));
            for (int k = 0; k < K; ++k) {
                SPC5_CUDA(cudaEventCreateWithFlags(&hp.xin[k], cudaEventDisableTiming));
                SPC5_CUDA(cudaEventCreateWithFlags(&hp.yout[k], cudaEventDisableTiming));
                SPC5_CUDA(cudaEventCreateWithFlags(&hp.ycopied[k], cudaEventDisableTiming));
            }
            hp.K = K;
        }
    }
    const int R = m.r;
    auto rows = [&](int k, int64_t *r0, int64_t *r1) {
        *r0 = std::min(hp.p[k] * R, m.num_rows);
        *r1 = std::min(hp.p[k + 1] * R, m.num_rows);
    };
    // copies wait for the work already queued on the caller's stream
    SPC5_CUDA(cudaEventRecord(hp.start, st));
    SPC5_CUDA(cudaStreamWaitEvent(hp.h2d, hp.start, 0));
    SPC5_CUDA(cudaStreamWaitEvent(hp.d2h, hp.start, 0));
    SPC5_CUDA(cudaStreamWaitEvent(hp.comp, hp.start, 0));
    cudaStream_t cs = hp.comp;  // products on the pipeline's own stream
    Scratch sc;
    SPC5_TRY(scratch_for(h, cs, &sc));
    int64_t have = 0;  // x columns already queued
    char *dx = static_cast<char *>(m.dx), *dy = static_cast<char *>(m.dy);
    const char *hx = static_cast<const char *>(h_x);
    char *hy = static_cast<char *>(h_y);
    // large pageable buffers go through the pinned staging buffers, copied by a thread team
    const bool big = xb + yb >= ((size_t)8 << 20) && !getenv("SPC5_NO_HOST_STAGING");
    const bool px = big && is_pageable(h_x), py = big && is_pageable(h_y);
    std::unique_lock<std::mutex> stage_lk(g_stage.mu, std::defer_lock);
    const char *ux = hx;  // the caller's buffers
    char *uy = hy;
    const int T = host_threads();
    std::vector<std::thread> team;
    std::vector<std::atomic<int>> x_ready(px || (py && accumulate) ? hp.K : 0);
    int64_t xlo[8], xhi[8];
    if (px || py) {
        stage_lk.lock();
        if (px) SPC5_TRY(g_stage.grow(&g_stage.x, &g_stage.xcap, xb));
        if (py) SPC5_TRY(g_stage.grow(&g_stage.y, &g_stage.ycap, yb));
        if (px) hx = static_cast<const char *>(g_stage.x);
        if (py) hy = static_cast<char *>(g_stage.y);
        int64_t hv = 0;
        for (int k = 0; k < hp.K; ++k) {
            const int64_t want = k == hp.K - 1 ? m.num_cols : hp.need[k];
            xlo[k] = hv;
            xhi[k] = std::max(hv, want);
            hv = xhi[k];
        }
        if (!x_ready.empty()) {
            for (auto &c : x_ready) c.store(0);
            char *sx = static_cast<char *>(g_stage.x), *sy = static_cast<char *>(g_stage.y);
            for (int t = 0; t < T; ++t)
                team.emplace_back([&, t, sx, sy] {
                    for (int k = 0; k < hp.K; ++k) {
                        if (px)
                            copy_share(sx + xlo[k] * vb, ux + xlo[k] * vb,
                                       (size_t)(xhi[k] - xlo[k]) * vb, t, T);
                        if (py && accumulate) {
                            int64_t r0, r1;
                            rows(k, &r0, &r1);
                            copy_share(sy + r0 * vb, uy + r0 * vb, (size_t)(r1 - r0) * vb, t, T);
                        }
                        x_ready[k].fetch_add(1, std::memory_order_release);
                    }
                });
        }
    }
    struct Joiner {  // the team is joined on every exit path
        std::vector<std::thread> &t;
        ~Joiner() {
            for (auto &th : t)
                if (th.joinable()) th.join();
        }
    } joiner{team};
    int launches = 0;
    for (int k = 0; k < hp.K; ++k) {
        if (!x_ready.empty())  // this stage's piece has been staged by every thread
            while (x_ready[k].load(std::memory_order_acquire) < T) std::this_thread::yield();
        const int64_t want = k == hp.K - 1 ? m.num_cols : hp.need[k];
        if (want > have) {
            SPC5_CUDA(cudaMemcpyAsync(dx + have * vb, hx + have * vb, (size_t)(want - have) * vb,
                                      cudaMemcpyHostToDevice, hp.h2d));
            have = want;
        }
        int64_t r0, r1;
        rows(k, &r0, &r1);
        if (accumulate && r1 > r0)
            SPC5_CUDA(cudaMemcpyAsync(dy + r0 * vb, hy + r0 * vb, (size_t)(r1 - r0) * vb,
                                      cudaMemcpyHostToDevice, hp.h2d));
        SPC5_CUDA(cudaEventRecord(hp.xin[k], hp.h2d));
        SPC5_CUDA(cudaStreamWaitEvent(cs, hp.xin[k], 0));
        if (hp.K == 1) {
            SPC5_TRY(launch_spmv(m, 0, m.num_panels, m.dx, m.dy, accumulate, cs, sc));
        } else {
            const int64_t blk[2] = {hp.b[k], hp.b[k + 1]};
            SPC5_TRY(launch_spmv(m, hp.p[k], hp.p[k + 1], m.dx, m.dy, accumulate, cs, sc,
                                 nullptr, blk));
        }
        launches += g_launches;
        g_launches = 0;
        SPC5_CUDA(cudaEventRecord(hp.yout[k], cs));
        SPC5_CUDA(cudaStreamWaitEvent(hp.d2h, hp.yout[k], 0));
        if (r1 > r0)
            SPC5_CUDA(cudaMemcpyAsync(hy + r0 * vb, dy + r0 * vb, (size_t)(r1 - r0) * vb,
                                      cudaMemcpyDeviceToHost, hp.d2h));
        if (py) SPC5_CUDA(cudaEventRecord(hp.ycopied[k], hp.d2h));
    }
    g_launches = launches;
    // the caller's stream completes with the last copy back
    SPC5_CUDA(cudaEventRecord(hp.done, hp.d2h));
    SPC5_CUDA(cudaStreamWaitEvent(st, hp.done, 0));
    if (py) {
        // each stage's rows leave the pinned buffer as soon as they have landed in it
        for (auto &th : team)
            if (th.joinable()) th.join();
        team.clear();
        std::atomic<int> bad{0};
        for (int t = 0; t < T; ++t)
            team.emplace_back([&, t] {
                for (int k = 0; k < hp.K; ++k) {
                    if (cudaEventSynchronize(hp.ycopied[k]) != cudaSuccess) bad.store(1);
                    int64_t r0, r1;
                    rows(k, &r0, &r1);
                    copy_share(uy + r0 * vb, hy + r0 * vb, (size_t)(r1 - r0) * vb, t, T);
                }
            });
        for (auto &th : team) th.join();
        team.clear();
        if (bad.load()) return fail(SPC5_ECUDA, "device-to-host copy of y failed");
    }
    SPC5_CUDA(cudaStreamSynchronize(st));
    return SPC5_OK;
}

int spc5_partition_by_nnz(spc5_matrix_t h, int workers, int64_t *h_ranges, void *stream) {
    g_launches = 0;
    if (!h) return fail(SPC5_EINVAL, "null handle");
    if (workers < 1) return fail(SPC5_EINVAL, "workers must be >= 1");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    SPC5_TRY(ensure_plan(h, st));
    return partition_by_nnz(h->m, workers, h_ranges, st);
}

int spc5_block_value_offsets(spc5_matrix_t h, int64_t *d_offsets, void *stream) {
    if (!h) return fail(SPC5_EINVAL, "null handle");
    return block_value_offsets(h->m, d_offsets, static_cast<cudaStream_t>(stream));
}

int spc5_validate(spc5_matrix_t h, void *stream) {
    if (!h) return fail(SPC5_EINVAL, "null handle");
    return validate_structure(h->m, static_cast<cudaStream_t>(stream));
}

int spc5_to_csr(spc5_matrix_t h, int64_t *d_row_ptr, int32_t *d_col_idx, void *d_values,
                void *stream) {
    if (!h) return fail(SPC5_EINVAL, "null handle");
    return to_csr(h->m, d_row_ptr, d_col_idx, d_values, static_cast<cudaStream_t>(stream));
}

int spc5_free(spc5_matrix_t h) {
    if (!h) return SPC5_OK;
    h->free_scratch();
    free_matrix(h->m);
    delete h;
    return SPC5_OK;
}

int spc5_csr_exact(int64_t num_rows, int precision, const int64_t *d_row_ptr,
                   const int32_t *d_col_idx, const void *d_values, const void *d_x, double *d_y,
                   double *d_abs, void *stream) {
    if (precision != SPC5_F32 && precision != SPC5_F64)
        return fail(SPC5_EINVAL, "precision must be 'f32' or 'f64'");
    return csr_exact(num_rows, precision, d_row_ptr, d_col_idx, d_values, d_x, d_y, d_abs,
                     static_cast<cudaStream_t>(stream));
}

int spc5_gen_stencil27_rowptr(int64_t n, int64_t row_lo, int64_t row_hi, int64_t *d_row_ptr,
                              void *stream) {
    return gen_stencil27_rowptr(n, n, row_lo, row_hi, d_row_ptr,
                                static_cast<cudaStream_t>(stream));
}

int spc5_gen_stencil27_fill(int64_t n, int64_t row_lo, int64_t row_hi, int precision,
                            uint64_t seed, double diag, const int64_t *d_row_ptr,
                            int32_t *d_col_idx, void *d_values, void *stream) {
    return spc5_gen_stencil27_box_fill(n, n, row_lo, row_hi, precision, seed, diag, d_row_ptr,
                                       d_col_idx, d_values, stream);
}

int spc5_gen_stencil27_box_rowptr(int64_t n, int64_t nz, int64_t row_lo, int64_t row_hi,
                                  int64_t *d_row_ptr, void *stream) {
    return gen_stencil27_rowptr(n, nz, row_lo, row_hi, d_row_ptr,
                                static_cast<cudaStream_t>(stream));
}

int spc5_gen_stencil27_box_fill(int64_t n, int64_t nz, int64_t row_lo, int64_t row_hi,
                                int precision, uint64_t seed, double diag,
                                const int64_t *d_row_ptr, int32_t *d_col_idx, void *d_values,
                                void *stream) {
    if (precision != SPC5_F32 && precision != SPC5_F64)
        return fail(SPC5_EINVAL, "precision must be 'f32' or 'f64'");
    return gen_stencil27_fill(n, nz, row_lo, row_hi, precision, seed, diag, d_row_ptr,
                              d_col_idx, d_values, static_cast<cudaStream_t>(stream));
}

int spc5_gen_powerlaw_rowptr(int64_t n, int64_t row_lo, int64_t row_hi, uint64_t seed,
                             const int32_t *d_len_table, int table_bits, int64_t *d_row_ptr,
                             void *stream) {
    return gen_powerlaw_rowptr(n, row_lo, row_hi, seed, d_len_table, table_bits, d_row_ptr,
                               static_cast<cudaStream_t>(stream));
}

int spc5_gen_powerlaw_fill(int64_t n, int64_t row_lo, int64_t row_hi, int precision,
                           uint64_t seed, const int32_t *d_len_table, int table_bits,
                           const int64_t *d_row_ptr, int32_t *d_col_idx, void *d_values,
                           void *stream) {
    if (precision != SPC5_F32 && precision != SPC5_F64)
        return fail(SPC5_EINVAL, "precision must be 'f32' or 'f64'");
    return gen_powerlaw_fill(n, row_lo, row_hi, precision, seed, d_len_table, table_bits,
                             d_row_ptr, d_col_idx, d_values, static_cast<cudaStream_t>(stream));
}

int spc5_gen_fem_rowptr(int64_t nodes, int64_t row_lo, int64_t row_hi, int64_t *d_row_ptr,
                        void *stream) {
    return gen_fem_rowptr(nodes, row_lo, row_hi, d_row_ptr, static_cast<cudaStream_t>(stream));
}

int spc5_gen_fem_fill(int64_t nodes, int64_t row_lo, int64_t row_hi, int precision,
                      uint64_t seed, const int64_t *d_row_ptr, int32_t *d_col_idx,
                      void *d_values, void *stream) {
    if (precision != SPC5_F32 && precision != SPC5_F64)
        return fail(SPC5_EINVAL, "precision must be 'f32' or 'f64'");
    return gen_fem_fill(nodes, row_lo, row_hi, precision, seed, d_row_ptr, d_col_idx, d_values,
                        static_cast<cudaStream_t>(stream));
}

}  // extern "C"
