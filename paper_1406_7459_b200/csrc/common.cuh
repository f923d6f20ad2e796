// Shared device helpers for the magfd-b200 kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <type_traits>

namespace mfd {

// Complex storage type per precision: float2 / double2 give 8 B / 16 B vector
// loads and stores.
template <class T> struct C2t;
template <> struct C2t<float> { using type = float2; };
template <> struct C2t<double> { using type = double2; };
template <class T> using C2 = typename C2t<T>::type;

template <class T> __device__ __forceinline__ C2<T> mk(T x, T y) { C2<T> r; r.x = x; r.y = y; return r; }
template <class T> __device__ __forceinline__ C2<T> cadd(C2<T> a, C2<T> b) { return mk<T>(a.x + b.x, a.y + b.y); }
template <class T> __device__ __forceinline__ C2<T> csub(C2<T> a, C2<T> b) { return mk<T>(a.x - b.x, a.y - b.y); }
template <class T> __device__ __forceinline__ C2<T> cmul(C2<T> a, C2<T> b) {
    return mk<T>(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// a * conj(b)
template <class T> __device__ __forceinline__ C2<T> cmulc(C2<T> a, C2<T> b) {
    return mk<T>(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
template <class T> __device__ __forceinline__ C2<T> cconj(C2<T> a) { return mk<T>(a.x, -a.y); }
template <class T> __device__ __forceinline__ C2<T> cscale(C2<T> a, T s) { return mk<T>(a.x * s, a.y * s); }
// multiply by -i (forward) or +i (inverse)
template <class T, bool INV> __device__ __forceinline__ C2<T> cmul_mi(C2<T> a) {
    return INV ? mk<T>(-a.y, a.x) : mk<T>(a.y, -a.x);
}

// exp(-2 pi i k / 64), k = 0..63, 25 significant digits (generated with mpmath).
__constant__ const double kW64[64][2] = {
    {1.0, 0.0},
    {0.995184726672196886244837, -0.09801714032956060199419556},
    {0.9807852804032304491261822, -0.1950903220161282678482849},
    {0.9569403357322088649357979, -0.2902846772544623676361924},
    {0.9238795325112867561281832, -0.38268343236508977172846},
    {0.8819212643483550297127569, -0.4713967368259976485563876},
    {0.8314696123025452370787884, -0.5555702330196022247428308},
    {0.7730104533627369608109066, -0.6343932841636454982151716},
    {0.7071067811865475244008444, -0.7071067811865475244008444},
    {0.6343932841636454982151716, -0.7730104533627369608109066},
    {0.5555702330196022247428308, -0.8314696123025452370787884},
    {0.4713967368259976485563876, -0.8819212643483550297127569},
    {0.38268343236508977172846, -0.9238795325112867561281832},
    {0.2902846772544623676361924, -0.9569403357322088649357979},
    {0.1950903220161282678482849, -0.9807852804032304491261822},
    {0.09801714032956060199419556, -0.995184726672196886244837},
    {2.06703210982639882364969e-43, -1.0},
    {-0.09801714032956060199419556, -0.995184726672196886244837},
    {-0.1950903220161282678482849, -0.9807852804032304491261822},
    {-0.2902846772544623676361924, -0.9569403357322088649357979},
    {-0.38268343236508977172846, -0.9238795325112867561281832},
    {-0.4713967368259976485563876, -0.8819212643483550297127569},
    {-0.5555702330196022247428308, -0.8314696123025452370787884},
    {-0.6343932841636454982151716, -0.7730104533627369608109066},
    {-0.7071067811865475244008444, -0.7071067811865475244008444},
    {-0.7730104533627369608109066, -0.6343932841636454982151716},
    {-0.8314696123025452370787884, -0.5555702330196022247428308},
    {-0.8819212643483550297127569, -0.4713967368259976485563876},
    {-0.9238795325112867561281832, -0.38268343236508977172846},
    {-0.9569403357322088649357979, -0.2902846772544623676361924},
    {-0.9807852804032304491261822, -0.1950903220161282678482849},
    {-0.995184726672196886244837, -0.09801714032956060199419556},
    {-1.0, -4.134064219652797647299381e-43},
    {-0.995184726672196886244837, 0.09801714032956060199419556},
    {-0.9807852804032304491261822, 0.1950903220161282678482849},
    {-0.9569403357322088649357979, 0.2902846772544623676361924},
    {-0.9238795325112867561281832, 0.38268343236508977172846},
    {-0.8819212643483550297127569, 0.4713967368259976485563876},
    {-0.8314696123025452370787884, 0.5555702330196022247428308},
    {-0.7730104533627369608109066, 0.6343932841636454982151716},
    {-0.7071067811865475244008444, 0.7071067811865475244008444},
    {-0.6343932841636454982151716, 0.7730104533627369608109066},
    {-0.5555702330196022247428308, 0.8314696123025452370787884},
    {-0.4713967368259976485563876, 0.8819212643483550297127569},
    {-0.38268343236508977172846, 0.9238795325112867561281832},
    {-0.2902846772544623676361924, 0.9569403357322088649357979},
    {-0.1950903220161282678482849, 0.9807852804032304491261822},
    {-0.09801714032956060199419556, 0.995184726672196886244837},
    {2.233876440654988324291948e-41, 1.0},
    {0.09801714032956060199419556, 0.995184726672196886244837},
    {0.1950903220161282678482849, 0.9807852804032304491261822},
    {0.2902846772544623676361924, 0.9569403357322088649357979},
    {0.38268343236508977172846, 0.9238795325112867561281832},
    {0.4713967368259976485563876, 0.8819212643483550297127569},
    {0.5555702330196022247428308, 0.8314696123025452370787884},
    {0.6343932841636454982151716, 0.7730104533627369608109066},
    {0.7071067811865475244008444, 0.7071067811865475244008444},
    {0.7730104533627369608109066, 0.6343932841636454982151716},
    {0.8314696123025452370787884, 0.5555702330196022247428308},
    {0.8819212643483550297127569, 0.4713967368259976485563876},
    {0.9238795325112867561281832, 0.38268343236508977172846},
    {0.9569403357322088649357979, 0.2902846772544623676361924},
    {0.9807852804032304491261822, 0.1950903220161282678482849},
    {0.995184726672196886244837, 0.09801714032956060199419556},
};

// Compile-time-indexed radix twiddle W_R^m (forward: exp(-2 pi i m/R)).
template <class T, int R, bool INV>
__device__ __forceinline__ C2<T> wconst(int m) {
    const int k = m * (64 / R);
    const T c = static_cast<T>(kW64[k][0]);
    const T s = static_cast<T>(kW64[k][1]);
    return INV ? mk<T>(c, -s) : mk<T>(c, s);
}

constexpr int ilog2(int n) { return n <= 1 ? 0 : 1 + ilog2(n >> 1); }
constexpr int brev(int v, int bits) {
    int r = 0;
    for (int b = 0; b < bits; ++b)
        if (v & (1 << b)) r |= 1 << (bits - 1 - b);
    return r;
}

// In-register radix-R DFT (R a power of two <= 64), natural order in/out.
// Iterative radix-2 DIT over a fully unrolled register array: after
// unrolling every index and twiddle is a compile-time constant, trivial
// twiddles (1, -i) cost no multiply.
// Decimation-in-frequency recursion on the sub-array v[OFF + k], k < R:
// every index is a template constant, so the array never leaves registers.
// ZIN: the upper half of the input is known to be zero (zero padding: every
//      first forward stage, since n <= P/2), so the first level is a copy /
//      twiddle only.
// HOUT: only outputs k < R/2 are consumed (every last inverse stage: only
//      the [0,n) corner is kept), so the final level skips the differences.
//      Natural k < R/2 sit at even bit-reversed positions.
template <class T, int R, bool INV, int OFF, bool ZIN = false, bool HOUT = false>
struct DifStage {
    static __device__ __forceinline__ void run(C2<T>* v) {
        if constexpr (R > 1) {
            constexpr int H = R / 2;
            bfly<0>(v);
            DifStage<T, H, INV, OFF, false, HOUT>::run(v);
            DifStage<T, H, INV, OFF + H, false, HOUT>::run(v);
        }
    }
    template <int J>
    static __device__ __forceinline__ void bfly(C2<T>* v) {
        if constexpr (J < R / 2) {
            const C2<T> a = v[OFF + J];
            if constexpr (HOUT && R == 2) {
                v[OFF] = cadd<T>(a, v[OFF + 1]);
                return;
            }
            C2<T> d;
            if constexpr (ZIN) {
                d = a;
            } else {
                const C2<T> b = v[OFF + J + R / 2];
                v[OFF + J] = cadd<T>(a, b);
                d = csub<T>(a, b);
            }
            if constexpr (J == 0) {
            } else if constexpr (4 * J == R) {
                d = cmul_mi<T, INV>(d);
            } else {
                d = cmul<T>(d, wconst<T, R, INV>(J));
            }
            v[OFF + J + R / 2] = d;
            bfly<J + 1>(v);
        }
    }
};

template <class T, int R, int I>
__device__ __forceinline__ void unscramble(C2<T>* v) {
    if constexpr (I < R) {
        constexpr int J = brev(I, ilog2(R));
        if constexpr (J > I) {
            const C2<T> t = v[I];
            v[I] = v[J];
            v[J] = t;
        }
        unscramble<T, R, I + 1>(v);
    }
}

template <class T, int R, bool INV, bool ZIN = false, bool HOUT = false>
__device__ __forceinline__ void dft(C2<T>* v) {
    DifStage<T, R, INV, 0, ZIN && (R > 1), HOUT>::run(v);   // output in bit-reversed order
    unscramble<T, R, 0>(v);                                  // compile-time register renaming
}

// Non-contracting arithmetic for the reference-order local-field / LLG code:
// the reference build emits no FMA (x86-64 baseline), so bitwise parity in
// the demag-free path needs separate round-to-nearest multiply and add.
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }

} // namespace mfd
