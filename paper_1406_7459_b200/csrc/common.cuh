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
// The same table as a constant expression (compile-time twiddles of the DIT codelets).
struct W64Table {
    static constexpr double v[64][2] = {
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

// In-register radix-2 decimation-in-time on a bit-reversed register array
// (the permutation is a compile-time renaming), natural order out.  Twiddled
// butterflies use the FMA form a +- w b with w b = c [(b.x - t b.y) + i (b.y +
// t b.x)], t = s / c (or the mirrored form with c / s when |s| > |c|, so |t| <= 1):
// 6 FFMA instead of the 4 FADD + complex multiply (8) of a DIF butterfly.
// ZIN: in bit-reversed order the zero upper half sits at odd positions, so the
// first level is a copy.  HOUT: the last level computes only outputs k < R/2.
template <class T, int R, bool INV, int S, bool ZIN, bool HOUT>
struct DitLevel {
    static __device__ __forceinline__ void run(C2<T>* v) {
        group<0>(v);
        if constexpr (S < R) DitLevel<T, R, INV, 2 * S, false, HOUT>::run(v);
    }
    template <int G>
    static __device__ __forceinline__ void group(C2<T>* v) {
        if constexpr (G < R) {
            bf<G, 0>(v);
            group<G + S>(v);
        }
    }
    template <int G, int J>
    static __device__ __forceinline__ void bf(C2<T>* v) {
        if constexpr (J < S / 2) {
            constexpr int H = S / 2;
            constexpr bool last_half = HOUT && S == R;   // only v[J], J < R/2, is consumed
            C2<T>& a = v[G + J];
            C2<T>& b = v[G + J + H];
            if constexpr (ZIN && S == 2) {
                b = a;
            } else if constexpr (J == 0) {
                const C2<T> x = a;
                a = cadd<T>(x, b);
                if constexpr (!last_half) b = csub<T>(x, b);
            } else if constexpr (4 * J == S) {
                const C2<T> x = a, wb = cmul_mi<T, INV>(b);
                a = cadd<T>(x, wb);
                if constexpr (!last_half) b = csub<T>(x, wb);
            } else {
                constexpr int k = J * (64 / S);
                constexpr double c = W64Table::v[k][0], sn = INV ? -W64Table::v[k][1] : W64Table::v[k][1];
                constexpr bool cf = (c < 0 ? -c : c) >= (sn < 0 ? -sn : sn);
                constexpr double f = cf ? c : sn, t = cf ? sn / c : c / sn;
                const T tf = static_cast<T>(t), ff = static_cast<T>(f);
                T u, w;
                if constexpr (cf) {          // w b = c [(b.x - t b.y) + i (b.y + t b.x)]
                    u = fma(-tf, b.y, b.x);
                    w = fma(tf, b.x, b.y);
                } else {                     // w b = s [(t b.x - b.y) + i (t b.y + b.x)]
                    u = fma(tf, b.x, -b.y);
                    w = fma(tf, b.y, b.x);
                }
                const C2<T> x = a;
                a = mk<T>(fma(ff, u, x.x), fma(ff, w, x.y));
                if constexpr (!last_half) b = mk<T>(fma(-ff, u, x.x), fma(-ff, w, x.y));
            }
            bf<G, J + 1>(v);
        }
    }
};

#ifndef MFD_DIT
#define MFD_DIT 1
#endif
template <class T, int R, bool INV, bool ZIN = false, bool HOUT = false>
__device__ __forceinline__ void dft(C2<T>* v) {
    if constexpr (MFD_DIT && R > 1) {
        unscramble<T, R, 0>(v);                                        // compile-time register renaming
        DitLevel<T, R, INV, 2, ZIN, HOUT>::run(v);
    } else {
        DifStage<T, R, INV, 0, ZIN && (R > 1), HOUT>::run(v);   // output in bit-reversed order
        unscramble<T, R, 0>(v);                                  // compile-time register renaming
    }
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
