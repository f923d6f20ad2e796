// Device tensor setup translation unit (K0a / K0b); see tensor.cuh.
#include "tensor.cuh"
#include "tensor_api.h"

namespace mfd {

void launch_tensor_octant(int nx, int ny, int k0, int nzc, double dx, double dy, double dz, double* out,
                          cudaStream_t s) {
    const long long n = (long long)nx * ny * nzc;
    if (n > 0) k_tensor_octant<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(nx, ny, k0, nzc, dx, dy, dz, out);
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

// ---- TMA descriptor creation (driver entry point fetched through the runtime:
// no link-time dependency on libcuda)
#include <cudaTypedefs.h>
#include "tma.cuh"
namespace mfd {
static PFN_cuTensorMapEncodeTiled tmap_encoder() {
    static PFN_cuTensorMapEncodeTiled encode = nullptr;
    if (!encode) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn)
            return nullptr;
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled>(fn);
    }
    return encode;
}
bool make_tmap_2d(CUtensorMap* map, const void* base, unsigned long long cols, unsigned long long rows,
                  unsigned long long pitch_bytes, unsigned box_cols, unsigned box_rows) {
    PFN_cuTensorMapEncodeTiled encode = tmap_encoder();
    if (!encode) return false;
    const cuuint64_t dims[2] = {cols, rows};
    const cuuint64_t strides[1] = {pitch_bytes};
    const cuuint32_t box[2] = {box_cols, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    return encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
} // namespace mfd
