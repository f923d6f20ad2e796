// Throughput of packed FP32x2 (FADD2/FMUL2/FFMA2, sm_100) against scalar FP32 on B200.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 fp2_bench.cu -o fp2_bench
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(float* out, int iters, float s) {
    float2 a[8];
    float b[16];
    for (int i = 0; i < 8; ++i) { a[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f); b[2 * i] = a[i].x; b[2 * i + 1] = a[i].y; }
    const float2 c = make_float2(s, -s), d = make_float2(0.999f, 1.001f);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (MODE == 0) { b[2 * i] = b[2 * i] + s; b[2 * i + 1] = b[2 * i + 1] - s; }
            if (MODE == 1) a[i] = __fadd2_rn(a[i], c);
            if (MODE == 2) { b[2 * i] = fmaf(b[2 * i], 0.999f, s); b[2 * i + 1] = fmaf(b[2 * i + 1], 1.001f, -s); }
            if (MODE == 3) a[i] = __ffma2_rn(a[i], d, c);
        }
    }
    float r = 0;
    for (int i = 0; i < 8; ++i) r += a[i].x + a[i].y + b[2 * i] + b[2 * i + 1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
int main() {
    float* o;
    cudaMalloc(&o, 148 * 8 * 256 * 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 20000;
    const char* names[4] = {"FADD x2 (scalar)", "FADD2", "FFMA x2 (scalar)", "FFMA2"};
    for (int rep = 0; rep < 2; ++rep)
    for (int m = 0; m < 4; ++m) {
        auto run = [&]() {
            if (m == 0) k<0><<<148 * 8, 256>>>(o, iters, 1e-7f);
            if (m == 1) k<1><<<148 * 8, 256>>>(o, iters, 1e-7f);
            if (m == 2) k<2><<<148 * 8, 256>>>(o, iters, 1e-7f);
            if (m == 3) k<3><<<148 * 8, 256>>>(o, iters, 1e-7f);
        };
        run();
        cudaEventRecord(e0);
        run();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double flops = 148.0 * 8 * 256 * iters * 16 * (m >= 2 ? 2 : 1);
        printf("%-18s %8.3f ms  %8.1f TFLOP/s (fp32 element ops x%s)\n", names[m], ms, flops / ms / 1e9, m >= 2 ? "2 (fma)" : "1");
    }
    return 0;
}
