// Host launchers of the device tensor setup (tensor.cu).
#pragma once
#include <cuda_runtime.h>

namespace mfd {

struct GemmDesc {
    int Mdim, Ndim, Kdim;
    long long a_m, a_k, b_k, b_n, o_m, o_n;
    long long a_b1, a_b2, b_b1, b_b2, o_b1, o_b2;
    int nb2;
    double scale;
};

// K0a: K = -N octant planes [k0, k0 + nzc): out = [6][nzc][ny][nx] (fp64).
void launch_tensor_octant(int nx, int ny, int k0, int nzc, double dx, double dy, double dz, double* out,
                          cudaStream_t s);
// Transform matrix [H][n] (cos with weights 1,2,2,.. or 2 sin).
void launch_axis_matrix(int H, int n, int P, int odd, double* C, cudaStream_t s);
// K0b batched fp64 GEMM, output fp64 or fp32.
void launch_gemm64(const GemmDesc& d, int nbatch, const double* A, const double* B, double* O, cudaStream_t s);
void launch_gemm64(const GemmDesc& d, int nbatch, const double* A, const double* B, float* O, cudaStream_t s);

} // namespace mfd
