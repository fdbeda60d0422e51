// mg.cu -- multi-GPU row-panel sharding over NCCL: the spc5_mg_* entry points
// of include/spc5_b200.h, the C-ABI form of distributed.py for callers that do
// not use torch.distributed.
//
// The reference parallelises one product with a thread pool over contiguous
// nnz-balanced panel ranges (parallel.py:31-92).  Here each range is a rank
// (one process per GPU): spc5_mg_partition reproduces partition_by_nnz from
// the CSR row pointers alone, each rank converts only its rows
// (spc5_convert_csr), and spc5_mg_spmv_step runs one product of the iterated
// form -- the local K2 writes the rank's slice of the next x (scaled), then
// the slices are all-gathered (unequal sizes: one NCCL group of point-to-point
// sends and receives, every transfer in flight at once over NVSwitch).
//
// NCCL is loaded with dlopen on first use (libnccl.so.2: the copy torch
// already loaded when there is one, else the system's), so the library has
// no link-time NCCL dependency and the single-GPU entry points never need it.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "common.cuh"

namespace spc5 {
namespace {

struct NcclApi {
    bool ok = false;
    std::string err;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t,
                         cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi load_nccl() {
    NcclApi a;
    void *h = nullptr;
    for (const char *name : {"libnccl.so.2", "libnccl.so"}) {
        h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
        if (h) break;
    }
    if (!h) {
        a.err = std::string("cannot load NCCL (libnccl.so.2): ") + dlerror();
        return a;
    }
    auto sym = [&](const char *n) -> void * {
        void *p = dlsym(h, n);
        if (!p && a.err.empty()) a.err = std::string("NCCL symbol missing: ") + n;
        return p;
    };
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
    a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
    a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
    a.Send = reinterpret_cast<decltype(a.Send)>(sym("ncclSend"));
    a.Recv = reinterpret_cast<decltype(a.Recv)>(sym("ncclRecv"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
    a.ok = a.err.empty();
    return a;
}

NcclApi &nccl() {
    static NcclApi api = load_nccl();
    return api;
}

int nccl_fail(ncclResult_t r, const char *what) {
    return fail(SPC5_ECUDA, std::string("NCCL error ") +
                                (nccl().GetErrorString ? nccl().GetErrorString(r) : "?") +
                                " in " + what);
}

#define SPC5_NCCL(call)                                          \
    do {                                                         \
        ncclResult_t _r = (call);                                \
        if (_r != ncclSuccess) return nccl_fail(_r, #call);      \
    } while (0)

// boundary k of partition_by_nnz over the panels of a CSR (parallel.py:42-50):
// cum[p] = row_ptr[min((p+1)*r, n)]; searchsorted(cum, total*k/P, 'left') + 1
__global__ void mg_partition_kernel(const int64_t *__restrict__ row_ptr, int64_t n, int r,
                                    int workers, int64_t *bounds) {
    const int k = (int)(blockIdx.x * blockDim.x + threadIdx.x) + 1;
    if (k >= workers) return;
    const int64_t np = (n + r - 1) / r;
    const int64_t total = row_ptr[n];
    const double target = (double)total * (double)k / (double)workers;
    int64_t res = 0;
    if (target > 0) {
        int64_t lo = 0, hi = np;
        while (lo < hi) {
            const int64_t mid = lo + (hi - lo) / 2;
            const double cum = (double)row_ptr[min((mid + 1) * r, n)];
            if (cum < target) lo = mid + 1;
            else hi = mid;
        }
        res = lo + 1;
    }
    bounds[k] = res < np ? res : np;
}

}  // namespace
}  // namespace spc5

using namespace spc5;

struct spc5_mg {
    ncclComm_t comm = nullptr;
    int nranks = 0, rank = 0;
    spc5_matrix_t shard = nullptr;  // borrowed: the caller frees it
    spc5_info_t info{};
    std::vector<int64_t> row_lo, row_hi;  // rows of every rank
};

extern "C" {

int spc5_mg_unique_id(void *id) {
    if (!id) return fail(SPC5_EINVAL, "null id buffer");
    if (!nccl().ok) return fail(SPC5_ECUDA, nccl().err);
    ncclUniqueId u;
    SPC5_NCCL(nccl().GetUniqueId(&u));
    memcpy(id, &u, sizeof(u));
    return SPC5_OK;
}

int spc5_mg_init(const void *id, int nranks, int rank, spc5_mg_t *out) {
    if (!out) return fail(SPC5_EINVAL, "null output handle");
    *out = nullptr;
    if (!id || nranks < 1 || rank < 0 || rank >= nranks)
        return fail(SPC5_EINVAL, "bad NCCL id, rank or rank count");
    if (!nccl().ok) return fail(SPC5_ECUDA, nccl().err);
    auto *mg = new (std::nothrow) spc5_mg();
    if (!mg) return fail(SPC5_ENOMEM, "out of host memory");
    ncclUniqueId u;
    memcpy(&u, id, sizeof(u));
    ncclResult_t r = nccl().CommInitRank(&mg->comm, nranks, u, rank);
    if (r != ncclSuccess) {
        delete mg;
        return nccl_fail(r, "ncclCommInitRank");
    }
    mg->nranks = nranks;
    mg->rank = rank;
    *out = mg;
    return SPC5_OK;
}

int spc5_mg_partition(const int64_t *d_row_ptr, int64_t num_rows, int r, int workers,
                      int64_t *h_ranges, void *stream) {
    if (!d_row_ptr || !h_ranges || num_rows < 0 || workers < 1)
        return fail(SPC5_EINVAL, "bad partition arguments");
    if (r != 1 && r != 2 && r != 4 && r != 8)
        return fail(SPC5_EINVAL, "r must be one of (1, 2, 4, 8), got " + std::to_string(r));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t np = (num_rows + r - 1) / r;
    std::vector<int64_t> b(workers + 1, 0);
    b[workers] = np;
    if (workers > 1 && np > 0) {
        int64_t *d = nullptr;
        SPC5_TRY(dev_alloc(&d, (size_t)workers + 1));
        mg_partition_kernel<<<(unsigned)cdiv(workers, 128), 128, 0, st>>>(d_row_ptr, num_rows, r,
                                                                          workers, d);
        SPC5_CUDA(cudaGetLastError());
        SPC5_CUDA(cudaMemcpyAsync(b.data() + 1, d + 1, sizeof(int64_t) * (workers - 1),
                                  cudaMemcpyDeviceToHost, st));
        SPC5_CUDA(cudaStreamSynchronize(st));
        dev_free(d);
    }
    for (int k = 0; k < workers; ++k) {
        h_ranges[2 * k] = std::min(b[k], np);
        h_ranges[2 * k + 1] = std::min(b[k + 1], np);
    }
    return SPC5_OK;
}

int spc5_mg_shard(spc5_mg_t mg, spc5_matrix_t local, const int64_t *h_row_ranges) {
    if (!mg || !local || !h_row_ranges) return fail(SPC5_EINVAL, "null argument");
    spc5_info_t info;
    SPC5_TRY(spc5_info(local, &info));
    std::vector<int64_t> lo(mg->nranks), hi(mg->nranks);
    for (int k = 0; k < mg->nranks; ++k) {
        lo[k] = h_row_ranges[2 * k];
        hi[k] = h_row_ranges[2 * k + 1];
        if (lo[k] < 0 || hi[k] < lo[k] || (k && lo[k] != hi[k - 1]))
            return fail(SPC5_EINVAL, "row ranges must be contiguous and ordered by rank");
    }
    if (hi[mg->rank] - lo[mg->rank] != info.num_rows)
        return fail(SPC5_EINVAL, "the local matrix must hold exactly this rank's rows");
    if (info.num_cols != hi[mg->nranks - 1] || lo[0] != 0)
        return fail(SPC5_EINVAL, "the row ranges must cover the square matrix's columns");
    mg->shard = local;
    mg->info = info;
    mg->row_lo = std::move(lo);
    mg->row_hi = std::move(hi);
    return SPC5_OK;
}

int spc5_mg_spmv_step(spc5_mg_t mg, const void *d_x, void *d_x_next, double scale,
                      void *stream) {
    if (!mg || !mg->shard) return fail(SPC5_EINVAL, "no shard attached (spc5_mg_shard)");
    if (!d_x || !d_x_next) return fail(SPC5_EINVAL, "x buffers must be non-null");
    if (!nccl().ok) return fail(SPC5_ECUDA, nccl().err);
    const int vb = mg->info.precision == SPC5_F64 ? 8 : 4;
    const ncclDataType_t dt = mg->info.precision == SPC5_F64 ? ncclFloat64 : ncclFloat32;
    char *xn = static_cast<char *>(d_x_next);
    const int me = mg->rank;
    // this rank's rows of the next x: scale * A_local . x (spc5_last_launch_count
    // reports these K2 launches; the NCCL kernels are NCCL's)
    SPC5_TRY(spc5_spmv_mirrored(mg->shard, d_x, xn + mg->row_lo[me] * vb, scale, nullptr, 0, 0,
                                stream));
    if (mg->nranks > 1) {  // all-gather-v of the slices: one group, every transfer at once
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        const int64_t n_me = mg->row_hi[me] - mg->row_lo[me];
        ncclResult_t first = ncclSuccess;
        auto keep = [&](ncclResult_t r) {
            if (first == ncclSuccess) first = r;
        };
        SPC5_NCCL(nccl().GroupStart());
        for (int k = 0; k < mg->nranks; ++k) {
            if (k == me) continue;
            const int64_t nk = mg->row_hi[k] - mg->row_lo[k];
            if (n_me) keep(nccl().Send(xn + mg->row_lo[me] * vb, (size_t)n_me, dt, k, mg->comm, st));
            if (nk) keep(nccl().Recv(xn + mg->row_lo[k] * vb, (size_t)nk, dt, k, mg->comm, st));
        }
        keep(nccl().GroupEnd());
        if (first != ncclSuccess) return nccl_fail(first, "all-gather-v group");
    }
    return SPC5_OK;
}

int spc5_mg_free(spc5_mg_t mg) {
    if (!mg) return SPC5_OK;
    if (mg->comm && nccl().ok) nccl().CommDestroy(mg->comm);
    delete mg;
    return SPC5_OK;
}

}  // extern "C"
