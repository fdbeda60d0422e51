// Microbenchmark (experiments, not part of the library): HBM read bandwidth of
// per-warp cp.async.bulk rings vs a plain vectorised-load stream on sm_100a.
//   tma: each warp owns S slots of CB bytes; a chunk = P bulk copies of CB/P
//        bytes taken from P separate arrays (like SPC5's col/mask/value arrays).
//   ldg: every thread reads 16-byte vectors, grid-stride.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_stream tma_stream.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void tma_kernel(const uint8_t *buf, int64_t bytes_per_array, int P, int CB, int S,
                           int64_t nchunks, unsigned long long *sink) {
    extern __shared__ __align__(128) uint8_t smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, wpc = blockDim.x >> 5;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem) + warp * S;
    const uint32_t ring = sa(smem) + 1024 + (uint32_t)(warp * S) * CB;
    if (lane == 0)
        for (int i = 0; i < S; ++i)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(bars + i)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    const int64_t stride = (int64_t)gridDim.x * wpc;
    const int64_t c0 = (int64_t)blockIdx.x * wpc + warp;
    const int piece = (CB / P) & ~15;
    auto issue = [&](int64_t c, int slot) {
        const uint32_t dst = ring + slot * CB;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(bars + slot)),
                     "r"(piece * P) : "memory");
        for (int p = 0; p < P; ++p) {
            const uint8_t *src = buf + p * bytes_per_array + c * piece;
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
                "[%0], [%1], %2, [%3], %4;" ::"r"(dst + p * piece), "l"(src), "r"(piece),
                "r"(sa(bars + slot)), "l"(pol) : "memory");
        }
    };
    if (lane == 0)
        for (int i = 0; i < S; ++i)
            if (c0 + i * stride < nchunks) issue(c0 + i * stride, i);
    unsigned long long acc = 0;
    int it = 0;
    for (int64_t c = c0; c < nchunks; c += stride, ++it) {
        const int slot = it % S;
        const uint32_t par = (it / S) & 1;
        asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n"
                     ::"r"(sa(bars + slot)), "r"(par) : "memory");
        uint32_t v;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(ring + slot * CB + lane * 4));
        acc += v;
        __syncwarp();
        const int64_t cn = c + (int64_t)S * stride;
        if (lane == 0 && cn < nchunks) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(cn, slot);
        }
    }
    if (acc == 0x12345) atomicAdd(sink, acc);
}

__global__ void ldg_kernel(const int4 *buf, int64_t n, unsigned long long *sink) {
    int acc = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int4 v = __ldcs(buf + i);
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x12345) atomicAdd(sink, acc);
}

int main(int argc, char **argv) {
    const int64_t total = 576ll << 20;  // ~ the beta(1,8) matrix stream
    uint8_t *buf;
    unsigned long long *sink;
    cudaMalloc(&buf, total + (1 << 20));
    cudaMalloc(&sink, 8);
    cudaMemset(buf, 1, total);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    // plain load stream
    for (int bpsm : {4, 8, 16}) {
        for (int r = 0; r < 3; ++r) ldg_kernel<<<sms * bpsm, 256>>>((const int4 *)buf, total / 16, sink);
        cudaEventRecord(e0);
        for (int r = 0; r < 10; ++r) ldg_kernel<<<sms * bpsm, 256>>>((const int4 *)buf, total / 16, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("ldg   blocks/sm=%2d              %7.1f GB/s\n", bpsm, total * 10 / (ms * 1e-3) / 1e9);
    }
    // argv: list of "CB,P,wpc,S" configurations
    for (int ai = 1; ai < argc; ++ai) {
        int CB, P, wpc, S;
        if (sscanf(argv[ai], "%d,%d,%d,%d", &CB, &P, &wpc, &S) != 4) continue;
        const size_t smem = 1024 + (size_t)wpc * S * CB;
        if (smem > 227 * 1024) continue;
        cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tma_kernel, wpc * 32, smem);
        if (per_sm < 1) continue;
        const int piece = (CB / P) & ~15;
        const int64_t bpa = (total / P) & ~(int64_t)255;
        const int64_t nchunks = bpa / piece;
        const int grid = sms * per_sm;
        for (int r = 0; r < 2; ++r)
            tma_kernel<<<grid, wpc * 32, smem>>>(buf, bpa, P, CB, S, nchunks, sink);
        cudaEventRecord(e0);
        for (int r = 0; r < 5; ++r)
            tma_kernel<<<grid, wpc * 32, smem>>>(buf, bpa, P, CB, S, nchunks, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("tma   CB=%5d P=%d wpc=%d S=%d ctas/sm=%d warps/sm=%2d ring/sm=%3dKB %7.1f GB/s\n",
               CB, P, wpc, S, per_sm, per_sm * wpc, per_sm * wpc * S * CB / 1024,
               (double)nchunks * piece * P * 5 / (ms * 1e-3) / 1e9);
    }
    cudaError_t err = cudaGetLastError();
    printf("status: %s\n", cudaGetErrorString(err));
    return 0;
}
