// One K2 instance per translation unit (parallel build): see spmv_kernel.cuh.
#include "spmv_kernel.cuh"
namespace spc5 {
int launch_k2_f64_u8_r1(const Matrix &m, const SpmvArgs &a, cudaStream_t st) {
    return launch_typed<double, uint8_t, 1>(m, a, st);
}
}  // namespace spc5
