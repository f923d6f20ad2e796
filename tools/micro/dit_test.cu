#include "/root/repo/paper_1406_7459_b200/csrc/common.cuh"
#include <cstdio>
#include <cmath>
using namespace mfd;
template <class T, int R, bool INV, bool ZIN, bool HOUT>
__global__ void kt(const C2<T>* in, C2<T>* out) {
    C2<T> v[R];
    for (int i = 0; i < R; ++i) v[i] = (ZIN && 2 * i >= R) ? mk<T>(0, 0) : in[i];
    dft<T, R, INV, ZIN, HOUT>(v);
    for (int i = 0; i < R; ++i) out[i] = v[i];
}
template <class T, int R, bool INV, bool ZIN, bool HOUT>
double check() {
    C2<T> *in, *out;
    cudaMallocManaged(&in, R * sizeof(C2<T>)); cudaMallocManaged(&out, R * sizeof(C2<T>));
    for (int i = 0; i < R; ++i) { in[i].x = sin(1.3 * i + 0.2); in[i].y = cos(0.7 * i * i); }
    kt<T, R, INV, ZIN, HOUT><<<1, 1>>>(in, out);
    cudaDeviceSynchronize();
    double err = 0, mx = 0;
    for (int k = 0; k < (HOUT ? R / 2 : R); ++k) {
        double re = 0, im = 0;
        for (int n = 0; n < R; ++n) {
            if (ZIN && 2 * n >= R) continue;
            double a = (INV ? 2 : -2) * M_PI * n * k / R;
            re += in[n].x * cos(a) - in[n].y * sin(a);
            im += in[n].x * sin(a) + in[n].y * cos(a);
        }
        err = fmax(err, fmax(fabs(re - out[k].x), fabs(im - out[k].y)));
        mx = fmax(mx, fmax(fabs(re), fabs(im)));
    }
    return err / mx;
}
int main() {
#define C(T, R, I, Z, H) printf("%s R=%2d inv=%d zin=%d hout=%d rel %.2e\n", #T, R, I, Z, H, check<T, R, I, Z, H>());
    C(float, 2, 0, 0, 0) C(float, 4, 0, 0, 0) C(float, 8, 0, 0, 0) C(float, 16, 0, 0, 0) C(float, 32, 0, 0, 0)
    C(float, 32, 1, 0, 0) C(float, 16, 0, 1, 0) C(float, 32, 0, 1, 0) C(float, 16, 1, 0, 1) C(float, 32, 1, 0, 1)
    C(double, 16, 0, 0, 0) C(double, 16, 1, 0, 1) C(double, 8, 0, 1, 0) C(double, 4, 1, 0, 0) C(double, 2, 0, 1, 0)
    return 0;
}
