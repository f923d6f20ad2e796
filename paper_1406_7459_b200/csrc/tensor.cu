// Device tensor setup translation unit (K0a / K0b); see tensor.cuh.
#include "tensor.cuh"
#include "tensor_api.h"

namespace mfd {

void launch_tensor_octant(int nx, int ny, int nz, double dx, double dy, double dz, double* out, cudaStream_t s) {
    const long long n = (long long)nx * ny * nz;
    k_tensor_octant<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(nx, ny, nz, dx, dy, dz, out);
}
void launch_axis_matrix(int H, int n, int P, int odd, double* C, cudaStream_t s) {
    k_axis_matrix<<<(unsigned)(((long long)H * n + 255) / 256), 256, 0, s>>>(H, n, P, odd, C);
}
template <class TO>
static void gemm(const GemmDesc& d, int nbatch, const double* A, const double* B, TO* O, cudaStream_t s) {
    dim3 grid((d.Ndim + 63) / 64, (d.Mdim + 63) / 64, nbatch);
    k_gemm64<TO><<<grid, 256, 0, s>>>(d, A, B, O);
}
void launch_gemm64(const GemmDesc& d, int nb, const double* A, const double* B, double* O, cudaStream_t s) {
    gemm<double>(d, nb, A, B, O, s);
}
void launch_gemm64(const GemmDesc& d, int nb, const double* A, const double* B, float* O, cudaStream_t s) {
    gemm<float>(d, nb, A, B, O, s);
}

} // namespace mfd
