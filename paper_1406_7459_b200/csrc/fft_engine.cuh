// Mixed-radix Stockham FFT engine for batches of power-of-two columns held by
// one CTA.  Replaces the reference's iterative radix-2 LineTransform
// (proj/include/magfd/fft.hpp:54-121): same unnormalised DFT convention
// (forward exp(-2 pi i nk/L), inverse conjugate twiddles), but organised as
// 1-3 register-radix stages with the data moved through shared memory (or
// straight from / to HBM on the first / last stage), so a length-1024 column
// costs one global read, one shared-memory round trip and one global write.
//
// Stage s (radix R, sub-length M, Mp = M/R) of the forward (DIT) transform,
// for task (p, n2):   out[p*M + Mp*k + n2] = W_M^{n2 k} * sum_n1 in[p*M + Mp*n1 + n2] W_R^{n1 k}
// After all stages, frequency f = k0 + R0*(k1 + R1*k2) sits at buffer
// position bufpos(f) = k0*Mp0 + k1*Mp1 + k2*Mp2 (mixed-radix digit reversal).
// The inverse runs the transposed stages in reverse order: it consumes
// buffer order and produces natural order, so no explicit reordering pass
// is ever needed.
#pragma once
#include "common.cuh"

namespace mfd {

// Radix plans: at most 32 complex values per task in fp32, 16 in fp64.
template <class T, int L> struct Plan;
#define MFD_PLAN(TT, L_, S_, A_, B_, C_)                                    \
    template <> struct Plan<TT, L_> {                                      \
        static constexpr int S = S_, R0 = A_, R1 = B_, R2 = C_;            \
    };
MFD_PLAN(float, 1, 0, 1, 1, 1)
MFD_PLAN(float, 2, 1, 2, 1, 1)
MFD_PLAN(float, 4, 1, 4, 1, 1)
MFD_PLAN(float, 8, 1, 8, 1, 1)
MFD_PLAN(float, 16, 1, 16, 1, 1)
MFD_PLAN(float, 32, 1, 32, 1, 1)
MFD_PLAN(float, 64, 2, 8, 8, 1)
MFD_PLAN(float, 128, 2, 16, 8, 1)
MFD_PLAN(float, 256, 2, 16, 16, 1)
MFD_PLAN(float, 512, 2, 32, 16, 1)
MFD_PLAN(float, 1024, 2, 32, 32, 1)
MFD_PLAN(float, 2048, 3, 16, 16, 8)
MFD_PLAN(double, 1, 0, 1, 1, 1)
MFD_PLAN(double, 2, 1, 2, 1, 1)
MFD_PLAN(double, 4, 1, 4, 1, 1)
MFD_PLAN(double, 8, 1, 8, 1, 1)
MFD_PLAN(double, 16, 1, 16, 1, 1)
MFD_PLAN(double, 32, 2, 8, 4, 1)
MFD_PLAN(double, 64, 2, 8, 8, 1)
MFD_PLAN(double, 128, 2, 16, 8, 1)
MFD_PLAN(double, 256, 2, 16, 16, 1)
MFD_PLAN(double, 512, 3, 16, 8, 4)
MFD_PLAN(double, 1024, 3, 16, 8, 8)
MFD_PLAN(double, 2048, 3, 16, 16, 8)
#undef MFD_PLAN

template <class T, int L, int s> struct StageInfo {
    using P = Plan<T, L>;
    static constexpr int R = s == 0 ? P::R0 : s == 1 ? P::R1 : P::R2;
    static constexpr int PRE = s == 0 ? 1 : s == 1 ? P::R0 : P::R0 * P::R1;
    static constexpr int M = L / PRE;
    static constexpr int MP = M / R;
};

// Buffer position of natural frequency f after the forward stages.
template <class T, int L>
__device__ __forceinline__ int bufpos(int f) {
    using P = Plan<T, L>;
    if constexpr (P::S == 0) {
        return 0;
    } else if constexpr (P::S == 1) {
        return f;
    } else if constexpr (P::S == 2) {
        const int k0 = f % P::R0, k1 = f / P::R0;
        return k0 * StageInfo<T, L, 0>::MP + k1;
    } else {
        const int k0 = f % P::R0, r = f / P::R0;
        const int k1 = r % P::R1, k2 = r / P::R1;
        return k0 * StageInfo<T, L, 0>::MP + k1 * StageInfo<T, L, 1>::MP + k2;
    }
}

// Natural frequency of output k of last-stage task p (the last stage has
// MP = 1): f = k0 + R0*k1 + R0*R1*k2 with the leading digits encoded in p.
template <class T, int L>
__device__ __forceinline__ int natfreq(int p, int k) {
    using P = Plan<T, L>;
    if constexpr (P::S <= 1) return k;
    else if constexpr (P::S == 2) return p + P::R0 * k;
    else return (p / P::R1) + P::R0 * (p % P::R1) + P::R0 * P::R1 * k;
}

// Twiddle tables (one allocation): [0, TWN) W_TWN^e; then for every power of
// two LT <= TWN a dense copy of the LT twiddles W_LT^e at [TWN + LT, TWN + 2 LT)
// (same values: W_LT^e = W_TWN^(e TWN/LT)).  A transform of length L reads
// only its dense L-entry table, so the lines it touches stay few and
// L1-resident (the TWN-strided reads of a length-1024 transform touched every
// line of the 32 KB table and mostly missed L1).
constexpr int TWN = 4096;
constexpr int TW_ALLOC = 3 * TWN;
template <class T, int LT>
__device__ __forceinline__ const C2<T>* tw_dense(const C2<T>* tw) { return tw + TWN + LT; }
// W_M^e for a stage of a length-L transform (M divides L).
template <class T, int L, int M>
__device__ __forceinline__ C2<T> tw_lookup(const C2<T>* __restrict__ tw, int e) {
    static_assert(L % M == 0, "stage length must divide the transform length");
    return __ldg(tw_dense<T, L>(tw) + e * (L / M));
}

// One stage over NCOL columns with NT threads.
//   INV=false: forward DIT stage (gather in-positions, DFT, twiddle, scatter out-positions)
//   INV=true : transposed inverse stage (gather out-positions, conj twiddle, IDFT, scatter in-positions)
// COLFAST: consecutive threads take consecutive columns (y/z passes: columns
// are contiguous in HBM); otherwise consecutive threads take consecutive
// tasks of one column (x pass: positions contiguous in HBM).
// SYNC_MID inserts a barrier between the gather and scatter phases, required
// when source and destination are the same shared buffer.
// ZIN (first forward stage only): inputs n1 >= R/2 are zero padding, not loaded.
// HOUT (last inverse stage only): outputs n1 >= R/2 are outside the kept corner.
struct NoHook { __device__ void operator()() const {} };
// mid: called after the SYNC_MID barrier (every gather of the stage is done)
template <class T, int L, int s, bool INV, int NCOL, int NT, bool COLFAST, bool SYNC_MID, bool ZIN = false,
          bool HOUT = false, bool NAT = false, int TWL = L, class LD, class ST, class MID = NoHook>
__device__ __forceinline__ void fft_stage(LD&& ld, ST&& st, const C2<T>* __restrict__ tw, MID&& mid = MID{}) {
    using SI = StageInfo<T, L, s>;
    constexpr int R = SI::R, M = SI::M, MP = SI::MP;
    constexpr int TPC = L / R;
    constexpr int TOTAL = NCOL * TPC;
    constexpr int TPT = (TOTAL + NT - 1) / NT;
    // NAT on the last stage: the frequency side (forward output / inverse
    // input) uses natural order instead of buffer order.
    constexpr bool NATF = NAT && s == Plan<T, L>::S - 1;
    C2<T> v[TPT][R];
    int colv[TPT], basev[TPT], n2v[TPT], pv[TPT];
#pragma unroll
    for (int i = 0; i < TPT; ++i) {
        const int q = threadIdx.x + i * NT;
        int col, t;
        if (COLFAST) { col = q % NCOL; t = q / NCOL; }
        else { t = q % TPC; col = q / TPC; }
        const int p = t / MP, n2 = t % MP;
        colv[i] = col;
        basev[i] = p * M + n2;
        n2v[i] = n2;
        pv[i] = p;
        if (TOTAL % NT == 0 || q < TOTAL) {
#pragma unroll
            for (int j = 0; j < R; ++j)
                v[i][j] = (ZIN && R > 1 && 2 * j >= R)
                              ? mk<T>(0, 0)
                              : ld(col, (NATF && INV) ? natfreq<T, L>(p, j) : basev[i] + MP * j);
        }
    }
    if (SYNC_MID) {
        __syncthreads();
        mid();
    }
#pragma unroll
    for (int i = 0; i < TPT; ++i) {
        const int q = threadIdx.x + i * NT;
        if (TOTAL % NT == 0 || q < TOTAL) {
            if (!INV) {
                dft<T, R, false, ZIN>(v[i]);
                if (MP > 1) {
#pragma unroll
                    for (int k = 1; k < R; ++k) v[i][k] = cmul<T>(v[i][k], tw_lookup<T, TWL, M>(tw, n2v[i] * k));
                }
            } else {
                if (MP > 1) {
#pragma unroll
                    for (int k = 1; k < R; ++k) v[i][k] = cmulc<T>(v[i][k], tw_lookup<T, TWL, M>(tw, n2v[i] * k));
                }
                dft<T, R, true, false, HOUT>(v[i]);
            }
#pragma unroll
            for (int j = 0; j < R; ++j)
                if (!(HOUT && R > 1 && 2 * j >= R))
                    st(colv[i], (NATF && !INV) ? natfreq<T, L>(pv[i], j) : basev[i] + MP * j, v[i][j]);
        }
    }
}

// Full forward transform: stage 0 reads via ld0, the last stage writes via
// stN, intermediate stages go through shared memory via (lds, sts).
// FIRST_SMEM / LAST_SMEM say whether ld0 / stN touch that same shared buffer,
// in which case the stage gathers everything before a barrier and scatters
// after it (in-place Stockham).  A barrier follows every shared-memory write.
// PRUNE: the upper half of every input column is zero padding (n <= P/2 on
// every axis), so the first stage skips those loads and the first DIF level.
// NAT: the last stage writes natural frequency order (instead of buffer order).
template <class T, int L, int NCOL, int NT, bool COLFAST, bool FIRST_SMEM, bool LAST_SMEM, bool PRUNE = true,
          bool NAT = false, int TWL = L, class LD0, class LDS, class STS, class STN>
__device__ __forceinline__ void fft_forward(LD0&& ld0, LDS&& lds, STS&& sts, STN&& stn,
                                            const C2<T>* __restrict__ tw) {
    constexpr int S = Plan<T, L>::S;
    if constexpr (S == 1) {
        fft_stage<T, L, 0, false, NCOL, NT, COLFAST, FIRST_SMEM && LAST_SMEM, PRUNE, false, NAT, TWL>(ld0, stn, tw);
    } else if constexpr (S == 2) {
        fft_stage<T, L, 0, false, NCOL, NT, COLFAST, FIRST_SMEM, PRUNE, false, false, TWL>(ld0, sts, tw);
        __syncthreads();
        fft_stage<T, L, 1, false, NCOL, NT, COLFAST, LAST_SMEM, false, false, NAT, TWL>(lds, stn, tw);
    } else if constexpr (S == 3) {
        fft_stage<T, L, 0, false, NCOL, NT, COLFAST, FIRST_SMEM, PRUNE, false, false, TWL>(ld0, sts, tw);
        __syncthreads();
        fft_stage<T, L, 1, false, NCOL, NT, COLFAST, true, false, false, false, TWL>(lds, sts, tw);
        __syncthreads();
        fft_stage<T, L, 2, false, NCOL, NT, COLFAST, LAST_SMEM, false, false, NAT, TWL>(lds, stn, tw);
    }
}

// Full inverse (transposed) transform: consumes buffer order via ld0,
// produces natural order via stN.
// PRUNE: only the lower half of every output column is kept (the [0,n)
// corner), so the last stage skips the other half.
// NAT: the first stage reads natural frequency order (instead of buffer order).
template <class T, int L, int NCOL, int NT, bool COLFAST, bool FIRST_SMEM, bool LAST_SMEM, bool PRUNE = true,
          bool NAT = false, int TWL = L, class LD0, class LDS, class STS, class STN>
__device__ __forceinline__ void fft_inverse(LD0&& ld0, LDS&& lds, STS&& sts, STN&& stn,
                                            const C2<T>* __restrict__ tw) {
    constexpr int S = Plan<T, L>::S;
    if constexpr (S == 1) {
        fft_stage<T, L, 0, true, NCOL, NT, COLFAST, FIRST_SMEM && LAST_SMEM, false, PRUNE, NAT, TWL>(ld0, stn, tw);
    } else if constexpr (S == 2) {
        fft_stage<T, L, 1, true, NCOL, NT, COLFAST, FIRST_SMEM, false, false, NAT, TWL>(ld0, sts, tw);
        __syncthreads();
        fft_stage<T, L, 0, true, NCOL, NT, COLFAST, LAST_SMEM, false, PRUNE, false, TWL>(lds, stn, tw);
    } else if constexpr (S == 3) {
        fft_stage<T, L, 2, true, NCOL, NT, COLFAST, FIRST_SMEM, false, false, NAT, TWL>(ld0, sts, tw);
        __syncthreads();
        fft_stage<T, L, 1, true, NCOL, NT, COLFAST, true, false, false, false, TWL>(lds, sts, tw);
        __syncthreads();
        fft_stage<T, L, 0, true, NCOL, NT, COLFAST, LAST_SMEM, false, PRUNE, false, TWL>(lds, stn, tw);
    }
}

} // namespace mfd
