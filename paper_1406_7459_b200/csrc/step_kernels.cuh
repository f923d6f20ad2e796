// Per-step kernels of the demag convolution + fused LLG update.
//
//   K1 k_r2c_x        M rows -> half spectrum along x        (pad fused; demag.hpp:204-228, fft.hpp:201-210)
//   K2 k_fft_y_fwd    y transform of the ny active rows       (fft.hpp:213-220)
//   K3 k_fft_z_conv   z transform -> K~ . M~ -> inverse z     (fft.hpp:223-237, demag.hpp:150-171)
//   K4 k_fft_y_inv    inverse y, keep ny rows                 (fft.hpp:181-186)
//   K5 k_c2r_x_llg    inverse x -> H_demag -> H_eff -> LLG -> Euler -> reductions
//                     (demag.hpp:237-249, fields.hpp:220-253, dynamics.hpp:49-121)
//
// HBM layout (T = float or double, C2<T> = complex):
//   M      3 x N  SoA, x fastest (grid.hpp:30-34), double-buffered
//   A      [3][nz][ny][Hp]  complex   x-spectrum of the active rows (Hp >= Px/2+1)
//   B      [3][nz][Py][Hp]  complex   x,y-spectrum, y in buffer (digit-reversed) order
//   Kt     [Py/2+1][Pz/2+1][Hp][6] T  real tensor spectrum octant, components (xx,yy,zz,xy,xz,yz)
//                                     interleaved per bin
#pragma once
#include "fft_engine.cuh"
#include "tma.cuh"

namespace mfd {

constexpr bool kK2StridedTw = true;
template <class T> constexpr int regE() { return sizeof(T) == 4 ? 32 : 16; }
constexpr int cmin(int a, int b) { return a < b ? a : b; }
constexpr int cmax(int a, int b) { return a > b ? a : b; }
constexpr int clampNT(int n) { return n < 32 ? 32 : n > 1024 ? 1024 : n; }
// x-pass shared layout [col][pos] with one pad element every 128 B.
template <class T> constexpr int padShift() { return sizeof(T) == 4 ? 4 : 3; }
template <class T> __device__ __forceinline__ int xpad(int pos) { return pos + (pos >> padShift<T>()); }
template <class T, int L> constexpr int xpitch() { return L + (L >> padShift<T>()) + 1; }

// -------------------------------------------------------------- configs
// RS > 0: small-grid variant with RS rows per CTA, so grids of a few dozen
// rows (SP4: 32) still spread over the SMs instead of running 1-3 CTAs.
#ifndef MFD_K1_F64_ROWS
#define MFD_K1_F64_ROWS 0   // f64 K1 rows per CTA override (0: the formula below)
#endif
template <class T, int N, int RS = 0> struct XCfg {   // K1
    static constexpr int E = regE<T>();
    static constexpr int ROWS = RS > 0                                ? RS
                                : sizeof(T) == 8 && MFD_K1_F64_ROWS > 0 ? MFD_K1_F64_ROWS
                                                                      : cmax(1, cmin(64, 128 * E / N));   // small CTAs: many phase schedules per SM
    static constexpr int NT = RS > 0 ? clampNT(ROWS * N / E) : clampNT(cmax(128, ROWS * N / E));
    static constexpr int SMEM = ROWS * xpitch<T, N>() * (int)sizeof(C2<T>);
};
#ifndef MFD_Y_TILE_MAX
// bytes of the K2/K4 shared tile (W columns x L).  64 KB keeps 2+ CTAs/SM;
// the three-stage Py = 2048 pass (C5) is faster with 128 KB tiles, i.e.
// 64-byte (f32) column groups at 1 CTA/SM: K2 3.72 -> 2.90 ms, K4 4.08 -> 2.76 ms
#define MFD_Y_TILE_MAX(L) ((L) >= 2048 ? 131072 : 65536)
#endif
#ifndef MFD_Z2_W
#define MFD_Z2_W 0             // K3 (two-stage) columns per CTA override (0: default)
#endif
#ifndef MFD_K3_KEARLY
#define MFD_K3_KEARLY 1   // K3: first register phase's tensor loads issued during stage 0 (C4 f32 K3 0.539 -> 0.528 ms)
#endif
#ifndef MFD_YFWD_F64_MINB
#define MFD_YFWD_F64_MINB 2   // f64 K2 (non-TMA y forward): 128 registers, 2 CTAs/SM (C4 f64 K2 0.713 -> 0.631 ms)
#endif
#ifndef MFD_YINV_F64_MINB
#define MFD_YINV_F64_MINB 2   // f64 K4 (non-TMA y inverse): resident CTAs/SM its register budget assumes
#endif
#ifndef MFD_K5_F64_MINB
#define MFD_K5_F64_MINB 2   // f64 K5: 128 registers, 2 CTAs/SM (C4 f64 K5 1.196 -> 0.949 ms despite a 144-byte spill)
#endif
#ifndef MFD_K5_F64_ROWS
#define MFD_K5_F64_ROWS 2   // f64 K5: 2 rows per CTA (72 instead of 144 load registers): C4 f64 K5 0.960 -> 0.862 ms
#endif
#ifndef MFD_K5_F64_FMA
#define MFD_K5_F64_FMA 1   // f64 K5 epilogue with FMA + rsqrt: C4 f64 K5 0.860 -> 0.843 ms
#endif
#ifndef MFD_Z2_F64_W
#define MFD_Z2_F64_W 0      // f64 K3 columns per CTA override (0: default)
#endif
#ifndef MFD_K3_F64_KPRE
#define MFD_K3_F64_KPRE 1   // f64 K3: tensor bins one register phase ahead
#endif
#ifndef MFD_K5_F64_T1
// f64 K5 sized for one first-stage FFT task per thread: ROWS = max(1, 512/N) rows,
// NT = 3 ROWS N / R0 threads (96 at N = 512) at 5 CTAs/SM (128 registers, no spill).
// C4 f64 K5 0.837 -> 0.725 ms against 2 rows x 256 threads at 2 CTAs/SM, where a
// quarter of the threads idled through every FFT stage.  0: the 2 x 256 layout
#define MFD_K5_F64_T1 1
#endif
#ifndef MFD_K5_F32_MINB
#define MFD_K5_F32_MINB 3   // f32 K5 (RS = 0): resident CTAs/SM its register budget assumes
#endif
#ifndef MFD_K5_DEFER_HALT
#define MFD_K5_DEFER_HALT 1   // 1-2-row K5 variants: halt flag checked at the first barrier (A/B switch)
#endif
#ifndef MFD_K5_RS_NT
#define MFD_K5_RS_NT 64   // threads of the 1-2-row K5 variants (small grids)
#endif
#ifndef MFD_K5_F32_T1
#define MFD_K5_F32_T1 0        // the same layout for f32 K5 (A/B switch)
#endif
#ifndef MFD_K5_F32_T1_ROWS
#define MFD_K5_F32_T1_ROWS 4   // f32 T1: rows per CTA at N = 512
#endif
#ifndef MFD_K5_F32_T1_REGS
#define MFD_K5_F32_T1_REGS 80  // f32 T1: register budget per thread
#endif
template <class T, int N, int RS = 0> struct LCfg {   // K5
    static constexpr bool T1 = RS == 0 && (sizeof(T) == 8 ? MFD_K5_F64_T1 : MFD_K5_F32_T1) && N >= 64 &&
                               Plan<T, N>::S >= 2;
    static constexpr int T1REGS = sizeof(T) == 8 ? 128 : MFD_K5_F32_T1_REGS;
    static constexpr int ROWS = RS > 0 ? RS
                                : T1   ? cmax(1, (sizeof(T) == 8 ? 1 : MFD_K5_F32_T1_ROWS) * 512 / N)
                                       : (sizeof(T) == 8 && MFD_K5_F64_ROWS > 0 ? cmin(MFD_K5_F64_ROWS, cmax(1, cmin(32, 2048 / cmax(N, 1))))
                                                                               : cmax(1, cmin(32, 2048 / cmax(N, 1))));
    static constexpr int NT = RS > 0 ? MFD_K5_RS_NT : T1 ? clampNT(3 * ROWS * N / Plan<T, N>::R0) : 256;
    static constexpr int SMEM = 3 * ROWS * xpitch<T, N>() * (int)sizeof(C2<T>);
    static constexpr int MINB = T1 ? cmax(1, cmin(cmin(sizeof(T) == 8 ? 5 : 8, 65536 / (NT * T1REGS)), (220 * 1024) / SMEM))
                                : sizeof(T) == 4 ? cmax(1, cmin(MFD_K5_F32_MINB, (200 * 1024) / SMEM))
                                           : (MFD_K5_F64_MINB > 1 && MFD_K5_F64_MINB * SMEM <= 226 * 1024 ? MFD_K5_F64_MINB : 1);
};
// dynamic shared memory of a K5 variant
template <class T, int N, int RS, bool FWD> constexpr int k5_smem() { return LCfg<T, N, RS>::SMEM; }
template <class T, int L> struct YCfg {   // K2 / K4
    static constexpr int CS = sizeof(C2<T>);
    static constexpr int W = cmax(1, cmin(128 / CS, MFD_Y_TILE_MAX(L) / (L * CS)));   // <= 64 KB tile: 2+ CTAs/SM
    static constexpr int NT = clampNT(W * L / regE<T>());
    static constexpr int SMEM = Plan<T, L>::S >= 2 ? W * L * CS : 0;
    // resident CTAs per SM the register budget is sized for (shared memory permitting)
    static constexpr int MINB = cmax(1, cmin(3, SMEM > 0 ? (200 * 1024) / SMEM : 3));
    // K4 in f64: at 3 CTAs/SM (80 registers) the inverse spills 456 bytes per thread
    static constexpr int MINB_INV = sizeof(T) == 8 && MFD_YINV_F64_MINB > 0 ? cmin(MINB, MFD_YINV_F64_MINB) : MINB;
    static constexpr int MINB_FWD = sizeof(T) == 8 && MFD_YFWD_F64_MINB > 0 ? cmin(MINB, MFD_YFWD_F64_MINB) : MINB;
};
template <class T, int L> struct ZCfg {   // K3
    static constexpr int CS = sizeof(C2<T>);
    static constexpr int W = cmax(1, cmin(128 / CS, 98304 / (6 * L * CS)));
    static constexpr int NCOL = 6 * W;
    static constexpr int NT = clampNT(NCOL * L / regE<T>());
    static constexpr int SMEM = NCOL * L * CS;
};

// Geometry of one rank's share of the problem.  Single GPU: G = 1, the slab
// is the whole grid, A is [3][nz][ny][Hp] and B is [3][nz][Py][Hp].
// z-slab decomposition over G ranks: the rank owns
// planes [k0, k0+nz) of nzg for the x passes (K1, K5) and the LLG update, and
// x-bin block `ublk` (width Wb, Hv valid) of every plane for the y and z
// passes (K2-K4).  The transposes sit right after K1 / before K5, where the
// spectrum has ny (not Py) rows, so they move half the bytes of a transpose
// after the y pass.  A is laid out [block][3][nz][ny][Wb] (row pitch Hp = Wb):
// block b of the send side goes to rank b, block g of the receive side came
// from rank g (planes g*nz ...), so both all-to-alls move contiguous blocks and
// no pack kernel exists.  B = [3][nzg][Py][Wb] is then rank-local.
struct Geo {
    int nx, ny, nz;       // nz: planes of this rank's slab
    int Px, Py, Pz;       // Pz from the global nzg
    int N;                // Px/2 complex points per x row
    int Hx;               // N + 1 bins
    int Hp;               // pitch of A rows (= Wb when G > 1)
    long long ncell;      // cells of the slab
    int nzg, k0;          // global planes, first plane of the slab
    int G, ublk, Wb, Hv;  // ranks, this rank's x-bin block, block width, valid bins in it
    long long SA;         // A block stride (3 nz ny Hp; one block when G == 1)
    unsigned binv;        // ceil(2^24 / Wb): x-bin u -> block (u * binv) >> 24
    long long S_c, S_k;   // B strides: component (nzg planes), plane (row stride Wb)
    int pf1, pf5;         // L2 prefetch distance of K1 / K5 in CTAs (~resident CTAs; 0 = off)
    int pfm;              // prefetch mask: 1 K1 ahead, 2 K5 own M rows, 4 K5 spectrum ahead
};

// Round a shared-memory pointer up to 128 bytes (TMA destinations).  The offset
// is added to the shared pointer itself, so the compiler keeps shared-space
// addressing (LDS/STS); an integer round trip would degrade it to generic LD/ST.
template <class P>
__device__ __forceinline__ P* align128(P* p) {
    const unsigned pad = (128u - (smem_u32(p) & 127u)) & 127u;
    return reinterpret_cast<P*>(reinterpret_cast<unsigned char*>(p) + pad);
}

// Asynchronous L2 prefetch of [p, p + bytes) (cp.async.bulk.prefetch, TMA
// unit: no registers, no shared memory).  Trimmed inward to 16-byte bounds.
__device__ __forceinline__ void l2_prefetch(const void* p, long long bytes) {
    const unsigned long long a = (reinterpret_cast<unsigned long long>(p) + 15) & ~15ull;
    const unsigned long long e = (reinterpret_cast<unsigned long long>(p) + bytes) & ~15ull;
    if (e <= a) return;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"((unsigned)(e - a)) : "memory");
}
// Element of x-bin u in the A row at in-block offset rowoff.  Single GPU: one
// block.  Slab decomposition (MULTI): bin u sits in the block of rank u / Wb at
// column u % Wb (the division as a 24-bit reciprocal multiply, exact for u < 2^12).
// rowp = A + rowoff (the row in block 0).
template <bool MULTI, class P>
__device__ __forceinline__ P* abin(const Geo& g, P* rowp, int u) {
    if constexpr (!MULTI) {
        return rowp + u;
    } else {
        const int b = (int)(((unsigned)u * g.binv) >> 24);
        return rowp + (b * g.SA + (u - b * g.Wb));
    }
}
// Offset of the A row (component comp, global plane k, row j) seen by the y
// passes on the receive side: plane k came from rank k / nz.
__device__ __forceinline__ long long arow_y(const Geo& g, int comp, int k, int j) {
    const int kb = k / g.nz, kl = k - kb * g.nz;
    return kb * g.SA + ((long long)(comp * g.nz + kl) * g.ny + j) * g.Hp;
}
// One-plane M halos below / above the slab ([3][ny][nx] each; null at the
// global boundary or on a single GPU).
template <class T> struct Halo { const T* lo; const T* hi; };

// Step control: early exit after a non-finite update (error) or, in relax
// mode, once the previous iteration met the torque criterion
// (dynamics.hpp:180-188).  Only K1 and K5 check it: the y / z passes (K2-K4)
// read and write nothing but the A / B spectrum scratch, so running them on a
// halted iteration is harmless, and skipping the dependent flag load at the
// entry of every K2-K4 CTA saves ~1 % of the step (C4 f32: K3 0.555 -> 0.541 ms).
struct Ctl {
    int* err;                                   // 0 ok, else failing iteration + 1
    const unsigned long long* prev_torque;      // null: no convergence check
    double Ms, tol, rad2deg;
};
__device__ __forceinline__ bool halted(const Ctl& c) {
    if (*(volatile int*)c.err) return true;
    if (c.prev_torque) {
        const double r = __longlong_as_double((long long)*(volatile unsigned long long*)c.prev_torque);
        if (sqrt(r) / c.Ms * c.rad2deg <= c.tol) return true;
    }
    return false;
}
// The same test split in two: the raw loads (issued early, nothing waits on
// them) and the decision (taken where the values are needed).
struct HaltRaw {
    int err;
    unsigned long long tq;
};
__device__ __forceinline__ HaltRaw halted_load(const Ctl& c) {
    HaltRaw h;
    h.err = *(volatile int*)c.err;
    h.tq = c.prev_torque ? *(volatile unsigned long long*)c.prev_torque : 0ull;
    return h;
}
__device__ __forceinline__ int halted_test(const Ctl& c, const HaltRaw& h) {
    return h.err != 0 || (c.prev_torque && sqrt(__longlong_as_double((long long)h.tq)) / c.Ms * c.rad2deg <= c.tol);
}

// Real-to-complex post-process of one pair (k, N-k) of a row whose N-point
// complex FFT of (x[2n], x[2n+1]) sits in scol (natural order):
// X[k] = E + W^k O, X[N-k] = conj(E - W^k O), E/O the even/odd spectra.
template <class T, int N>
__device__ __forceinline__ void r2c_post(const C2<T>* scol, C2<T>* dst, int k, C2<T> w) {
    const C2<T> zk = scol[xpad<T>(k & (N - 1))];
    const C2<T> zn = cconj<T>(scol[xpad<T>((N - k) & (N - 1))]);
    const C2<T> E = cscale<T>(cadd<T>(zk, zn), T(0.5));
    const C2<T> d = csub<T>(zk, zn);
    const C2<T> O = mk<T>(T(0.5) * d.y, T(-0.5) * d.x);   // -i/2 (zk - zn)
    const C2<T> wo = cmul<T>(w, O);
    dst[k] = cadd<T>(E, wo);
    if (N - k != k) dst[N - k] = cconj<T>(csub<T>(E, wo));
}

// ------------------------------------------------------------------ K1
// Body of one CTA (row group bx, component comp).
template <class T, int N, int RS = 0, bool MULTI = false>
__device__ __forceinline__ void k1_body(const Geo& g, const T* __restrict__ M, C2<T>* __restrict__ A,
                                        const C2<T>* __restrict__ tw, long long bx, int comp,
                                        unsigned char* smem_raw) {
    using CF = XCfg<T, N, RS>;
    constexpr int ROWS = CF::ROWS, NT = CF::NT, LP = xpitch<T, N>();
    C2<T>* sm = reinterpret_cast<C2<T>*>(smem_raw);
    const long long nrows = (long long)g.ny * g.nz;
    const long long row0 = bx * ROWS;
    const T* Mc = M + comp * g.ncell;
    const int nx = g.nx;
    const bool even = (nx & 1) == 0;
    // rows of the CTA ~one resident wave later: in L2 by the time it starts
    if ((g.pfm & 1) && threadIdx.x == 0) {
        const long long lin = (long long)blockIdx.y * gridDim.x + blockIdx.x + g.pf1;
        if (lin < (long long)gridDim.x * gridDim.y) {
            const long long r1 = (lin % gridDim.x) * ROWS;
            const long long nr = nrows - r1 < ROWS ? nrows - r1 : ROWS;
            l2_prefetch(M + (lin / gridDim.x) * g.ncell + r1 * nx, nr * nx * (long long)sizeof(T));
        }
    }

    auto ld0 = [&](int col, int pos) -> C2<T> {
        const long long row = row0 + col;
        const int i0 = 2 * pos;
        if (row >= nrows || i0 >= nx) return mk<T>(0, 0);
        const T* src = Mc + row * nx + i0;
        if (even) {
            return *reinterpret_cast<const C2<T>*>(src);
        }
        return mk<T>(src[0], i0 + 1 < nx ? src[1] : T(0));
    };
    auto lds = [&](int col, int pos) -> C2<T> { return sm[col * LP + xpad<T>(pos)]; };
    auto sts = [&](int col, int pos, C2<T> v) { sm[col * LP + xpad<T>(pos)] = v; };
    if constexpr (Plan<T, N>::S == 0) {
        for (int c = threadIdx.x; c < ROWS; c += NT) sts(c, 0, ld0(c, 0));
    } else {
        // last stage writes natural frequency order: the post-process needs no index reversal
        fft_forward<T, N, ROWS, NT, false, false, true, true, true>(ld0, lds, sts, sts, tw);
    }
    __syncthreads();
    // Real-to-complex post-process on pairs (k, N-k): X[k] = E + W^k O,
    // X[N-k] = conj(E - W^k O).  A thread owns pair index k (its twiddle is
    // loaded once) across all ROWS rows; the k = 0 owner also emits the
    // self-paired k = N/2.
    auto post = [&](int col, int k, C2<T> w) {
        const C2<T> zk = sm[col * LP + xpad<T>(k & (N - 1))];
        const C2<T> zn = cconj<T>(sm[col * LP + xpad<T>((N - k) & (N - 1))]);
        const C2<T> E = cscale<T>(cadd<T>(zk, zn), T(0.5));
        const C2<T> d = csub<T>(zk, zn);
        const C2<T> O = mk<T>(T(0.5) * d.y, T(-0.5) * d.x);   // -i/2 (zk - zn)
        const C2<T> wo = cmul<T>(w, O);
        C2<T>* dst = A + ((long long)comp * nrows + row0 + col) * g.Hp;
        *abin<MULTI>(g, dst, k) = cadd<T>(E, wo);
        if (N - k != k) *abin<MULTI>(g, dst, N - k) = cconj<T>(csub<T>(E, wo));
    };
    constexpr int HP = N / 2 > 0 ? N / 2 : 1;
    const int rows = (int)(nrows - row0 < ROWS ? nrows - row0 : ROWS);
    if constexpr (HP >= NT) {
        for (int k = threadIdx.x; k < HP; k += NT) {
            const C2<T> w = __ldg(tw_dense<T, 2 * N>(tw) + k);     // W_Px^k
            const C2<T> wh = __ldg(tw_dense<T, 2 * N>(tw) + N / 2);
#pragma unroll 4
            for (int col = 0; col < rows; ++col) {
                post(col, N / 2 > 0 ? k : 0, w);
                if (k == 0 && N > 1) post(col, N / 2, wh);
            }
        }
    } else {
        for (int e = threadIdx.x; e < ROWS * HP; e += NT) {
            const int col = e / HP, k = N / 2 > 0 ? e % HP : 0;
            if (col >= rows) continue;
            post(col, k, __ldg(tw_dense<T, 2 * N>(tw) + k));
            if (k == 0 && N > 1) post(col, N / 2, __ldg(tw_dense<T, 2 * N>(tw) + N / 2));
        }
    }
}

#ifndef MFD_K1_F64_MINB
// f64 K1 (RS = 0): resident CTAs/SM its register budget assumes (0: unconstrained, 92
// registers, 5 CTAs/SM).  4 (128 registers): C4 f64 K1 0.347 -> 0.335 ms; 6 spills
#define MFD_K1_F64_MINB 4
#endif
#ifndef MFD_K1_MINB
// f32 K1 (RS = 0): resident CTAs/SM its register budget assumes (0: unconstrained, 141
// registers at N = 512, 3 CTAs/SM).  4 (128 registers, no spill): C4 K1 0.160 -> 0.142 ms,
// C5 1.271 -> 1.122 ms; 5 (96 registers) spills at N = 1024; 6-7 spill everywhere
#define MFD_K1_MINB 4
#endif
template <class T, int N, int RS = 0, bool MULTI = false>
__global__ void __launch_bounds__(XCfg<T, N, RS>::NT, (sizeof(T) == 4 && RS == 0 && MFD_K1_MINB > 0)   ? MFD_K1_MINB
                                                       : (sizeof(T) == 8 && RS == 0 && MFD_K1_F64_MINB > 0) ? MFD_K1_F64_MINB
                                                                                                           : 1)
k_r2c_x(Geo g, const T* __restrict__ M, C2<T>* __restrict__ A, const C2<T>* __restrict__ tw, Ctl ctl) {
    if (halted(ctl)) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    k1_body<T, N, RS, MULTI>(g, M, A, tw, blockIdx.x, blockIdx.y, smem_raw);
}

// Measured on B200 (512x512x64 f32): the swizzle removes the conflicts but the
// extra integer work made K2 slower (0.32 -> 0.40 ms), so it is off.
constexpr bool kYSwizzle = false;   // re-measured with the TMA K2: 0.238 -> 0.242 ms (C4), C5 +0.6 %
// y-pass shared tile [pos][W]: with 64-byte position rows, the last stage's
// tasks (stride R_last positions apart) would land two per bank group; XOR the
// row parity with the stride bit so a half-warp covers both 64-byte halves.
template <class T, int L, int W>
__device__ __forceinline__ int yswz(int pos) {
    constexpr int S = Plan<T, L>::S;
    constexpr int RL = S == 3 ? Plan<T, L>::R2 : S == 2 ? Plan<T, L>::R1 : 1;
    if constexpr (kYSwizzle && W * (int)sizeof(C2<T>) == 64 && S >= 2) return pos ^ ((pos / RL) & 1);
    else return pos;
}

// ---------------------------------------------------- async copy helpers
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}
// one complex element, global -> shared, asynchronously
template <class T>
__device__ __forceinline__ void cp_async_c2(C2<T>* smem, const C2<T>* gmem) {
    if constexpr (sizeof(C2<T>) == 16) cp_async16(smem, gmem);
    else cp_async8(smem, gmem);
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int K>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(K) : "memory"); }

// ------------------------------------------------------------------ K2
// Tiles of W x-bins never leave the padded pitch (Hp and Wb are multiples of
// 16 >= W), so x-bins >= Hx are computed as harmless padding columns instead
// of being masked per element.  FY: ny == Py/2 (power-of-two ny), so the
// pruned first stage never meets a row >= ny and the row test disappears.
template <class T, int L, bool FY>
__global__ void __launch_bounds__(YCfg<T, L>::NT, YCfg<T, L>::MINB_FWD)
k_fft_y_fwd(Geo g, const C2<T>* __restrict__ A, C2<T>* __restrict__ B, const C2<T>* __restrict__ tw, Ctl ctl,
            int comp0) {
    using CF = YCfg<T, L>;
    constexpr int W = CF::W, NT = CF::NT;
    // no halt check: K2-K4 touch only spectrum scratch (see Ctl)
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C2<T>* sm = reinterpret_cast<C2<T>*>(smem_raw);
    const int u0 = blockIdx.x * W;
    const int k = blockIdx.y, comp = comp0 + (int)blockIdx.z;   // k: global plane
    const C2<T>* src = A + arow_y(g, comp, k, 0) + u0;
    C2<T>* dst = B + comp * g.S_c + k * g.S_k + u0;
    const int ny = g.ny, Hp = g.Hp, Wb = g.Wb;
    auto ld0 = [&](int col, int pos) -> C2<T> {
        if (!FY && pos >= ny) return mk<T>(0, 0);
        return src[pos * Hp + col];
    };
    auto lds = [&](int col, int pos) -> C2<T> { return sm[yswz<T, L, W>(pos) * W + col]; };
    auto sts = [&](int col, int pos, C2<T> v) { sm[yswz<T, L, W>(pos) * W + col] = v; };
    auto stn = [&](int col, int pos, C2<T> v) { dst[pos * Wb + col] = v; };
    // twiddles from the TWN-strided copy: measured faster for this pass than the
    // dense L table (0.314 vs 0.342 ms, 512x512x64 f32), unlike every other pass
    fft_forward<T, L, W, NT, true, false, false, true, false, kK2StridedTw ? TWN : L>(ld0, lds, sts, stn, tw);
}

// K2 with TMA-staged input (two-stage plans): persistent CTAs; the A tile of
// the next (x-bin block, plane, component) streams into a shared staging
// buffer (cp.async.bulk.tensor, mbarrier-completed) while the current tile runs
// its second FFT stage, so no warp waits on global loads.  Same arithmetic as
// k_fft_y_fwd.
#ifndef MFD_K2_REV
#define MFD_K2_REV 1   // TMA K2 tiles in reverse order (C5 K2 2.32 -> 2.27 ms; C4 neutral)
#endif
#ifndef MFD_K2_TMA3
#define MFD_K2_TMA3 1   // TMA-staged K2 also for three-stage plans (f32 Py = 2048, f64 Py = 1024)
#endif
#ifndef MFD_K2_T3_ROWB
// three-stage TMA K2: 128-byte tile rows where work + staging fit 220 KB (f64 Py = 1024:
// 0.610 -> 0.589 ms against the plain K2's 64-byte rows); 0: the plain K2's rows
#define MFD_K2_T3_ROWB 128
#endif
template <class T, int L> struct YTCfg {
    static constexpr int CS = sizeof(C2<T>);
    static constexpr bool WIDE = Plan<T, L>::S == 3 && MFD_K2_T3_ROWB > 0 &&
                                 (MFD_K2_T3_ROWB / CS) * L * CS * 3 / 2 + 128 <= 220 * 1024;
    static constexpr int W = WIDE ? MFD_K2_T3_ROWB / CS : YCfg<T, L>::W;
    static constexpr int NT = clampNT(W * L / regE<T>());
    static constexpr int SMEM = W * L * CS + W * (L / 2) * CS + 128;   // work + staging (ny <= L/2 rows) + align
    static constexpr int MINB = 2 * SMEM <= 220 * 1024 ? 2 : 1;
    // Measured (f32): Py = 1024 0.317 -> 0.243 ms (512x512x64); at Py = 256 the
    // plain kernel is ~10 % faster (short tiles), so staging starts at 512
    static constexpr bool OK = (Plan<T, L>::S == 2 && SMEM <= 110 * 1024 && L >= 512) ||
                               (MFD_K2_TMA3 && Plan<T, L>::S == 3 && SMEM <= 220 * 1024);
};

template <class T, int L, bool FY>
__global__ void __launch_bounds__(YTCfg<T, L>::NT, YTCfg<T, L>::MINB)
k_fft_y_fwd_tma(Geo g, const __grid_constant__ CUtensorMap tmA, C2<T>* __restrict__ B,
                const C2<T>* __restrict__ tw, Ctl ctl, int ntx, int box_rows, int comp0, int ncomp) {
    using CF = YTCfg<T, L>;
    constexpr int W = CF::W, NT = CF::NT;
    // dense L-entry twiddle table for two-stage plans (C4 f32: K2 0.238 -> 0.233 ms), the
    // TWN-strided copy for three-stage ones (C5: 2.32 vs 2.37 ms with the dense table)
    constexpr int TWL = kK2StridedTw && Plan<T, L>::S == 3 ? TWN : L;
    // no halt check: K2-K4 touch only spectrum scratch (see Ctl)
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C2<T>* work = reinterpret_cast<C2<T>*>(smem_raw);
    // TMA destinations must be 128-byte aligned
    C2<T>* stage = align128(work + W * L);
    __shared__ uint64_t bar;
    const int ny = g.ny, nz = g.nzg, Wb = g.Wb;   // all planes of this rank's x-bin block
    const int ntiles = ntx * nz * ncomp;          // components [comp0, comp0 + ncomp)
    int t = blockIdx.x;
    if (t >= ntiles) return;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_fence_init();
        tma_prefetch_desc(&tmA);
    }
    __syncthreads();
    // MFD_K2_REV: tiles in reverse order, so the first ones read the A rows K1 wrote
    // last (still in L2)
    auto tmap = [&](int tt) { return MFD_K2_REV ? ntiles - 1 - tt : tt; };
    auto issue = [&](int t0) {   // one thread
        const int tt = tmap(t0);
        const int bx = tt % ntx, k = (tt / ntx) % nz, comp = comp0 + tt / (ntx * nz);
        const int kb = k / g.nz, kl = k - kb * g.nz;   // plane k came from rank kb
        const int row0 = ((kb * 3 + comp) * g.nz + kl) * ny;
        mbar_arrive_expect_tx(&bar, (unsigned)(ny * W * CF::CS));
        for (int r = 0; r < ny; r += box_rows)
            tma_load_2d(stage + r * W, &tmA, bx * W * (CF::CS / 8), row0 + r, &bar);
    };
    if (threadIdx.x == 0) issue(t);
    unsigned parity = 0;
    auto lds = [&](int col, int pos) -> C2<T> { return work[yswz<T, L, W>(pos) * W + col]; };
    auto sts = [&](int col, int pos, C2<T> v) { work[yswz<T, L, W>(pos) * W + col] = v; };
    auto ld0 = [&](int col, int pos) -> C2<T> {
        if (!FY && pos >= ny) return mk<T>(0, 0);
        return stage[pos * W + col];
    };
#pragma unroll 1
    for (; t < ntiles; t += gridDim.x) {
        const int tt = tmap(t);
        const int bx = tt % ntx, k = (tt / ntx) % nz, comp = comp0 + tt / (ntx * nz);
        const int u0 = bx * W;
        C2<T>* dst = B + comp * g.S_c + k * g.S_k + u0;
        auto stn = [&](int col, int pos, C2<T> v) { dst[pos * Wb + col] = v; };
        mbar_wait(&bar, parity);
        parity ^= 1;
        fft_stage<T, L, 0, false, W, NT, true, false, true, false, false, TWL>(ld0, sts, tw);
        __syncthreads();   // staging consumed, stage-0 output visible
        if (threadIdx.x == 0 && t + (int)gridDim.x < ntiles) {
            fence_proxy_async_smem();
            issue(t + gridDim.x);
        }
        if constexpr (Plan<T, L>::S == 3) {
            fft_stage<T, L, 1, false, W, NT, true, true, false, false, false, TWL>(lds, sts, tw);
            __syncthreads();
            fft_stage<T, L, 2, false, W, NT, true, false, false, false, false, TWL>(lds, stn, tw);
        } else {
            fft_stage<T, L, 1, false, W, NT, true, false, false, false, false, TWL>(lds, stn, tw);
        }
        __syncthreads();   // work buffer free for the next tile
    }
}

// ------------------------------------------------------------------ K4
template <class T, int L, bool FY>
__global__ void __launch_bounds__(YCfg<T, L>::NT, YCfg<T, L>::MINB_INV)
k_fft_y_inv(Geo g, const C2<T>* __restrict__ B, C2<T>* __restrict__ A, const C2<T>* __restrict__ tw, Ctl ctl,
            int comp0) {
    using CF = YCfg<T, L>;
    constexpr int W = CF::W, NT = CF::NT;
    // no halt check: K2-K4 touch only spectrum scratch (see Ctl)
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C2<T>* sm = reinterpret_cast<C2<T>*>(smem_raw);
    const int u0 = blockIdx.x * W;
    const int k = blockIdx.y, comp = comp0 + (int)blockIdx.z;   // k: global plane
    const C2<T>* src = B + comp * g.S_c + k * g.S_k + u0;
    C2<T>* dst = A + arow_y(g, comp, k, 0) + u0;
    const int ny = g.ny, Hp = g.Hp, Wb = g.Wb;
    auto ld0 = [&](int col, int pos) -> C2<T> { return src[pos * Wb + col]; };
    auto lds = [&](int col, int pos) -> C2<T> { return sm[yswz<T, L, W>(pos) * W + col]; };
    auto sts = [&](int col, int pos, C2<T> v) { sm[yswz<T, L, W>(pos) * W + col] = v; };
    auto stn = [&](int col, int pos, C2<T> v) {
        if (FY || pos < ny) dst[pos * Hp + col] = v;   // pruned last stage: pos < Py/2 == ny when FY
    };
    fft_inverse<T, L, W, NT, true, false, false>(ld0, lds, sts, stn, tw);
}

// K4 with TMA-staged input (two-stage plans): persistent CTAs over a ring of
// three half-tile slots.  Tile i (L rows x W bins of B) lands as two halves in
// slots (2i) % 3 and (2i+1) % 3.  The transposed first inverse stage (stage 1,
// MP = 1) reads and writes the R1 contiguous rows of its task in place, so it
// needs no second buffer; once the last stage has gathered the tile into
// registers both its slots are free and the next tile's second half and the
// tile after that's first half are issued into them, so every load is in
// flight for at least one stage of compute.  Tiles are 128 bytes wide (16 f32
// bins): a stage-1 task row then spans all 32 banks, so the tasks of a warp
// never share a bank wavefront (with 64-byte rows the tasks, R1 rows apart,
// collide 2-way and TMA destinations cannot be padded off the 128-byte grid).
// Same arithmetic as k_fft_y_inv.
#ifndef MFD_K4_COMPFAST
// three-stage TMA K4: tiles with the component fastest (then x-bin block, then plane)
// instead of x-bin block fastest: C4 f64 K4 0.535 -> 0.516 ms, C5 2.59 -> 2.56 ms
// (two-stage plans: neutral, unchanged)
#define MFD_K4_COMPFAST 1
#endif
#ifndef MFD_K4_TMA3
#define MFD_K4_TMA3 1   // TMA-staged K4 also for three-stage plans (f32 Py = 2048, f64 Py = 1024)
#endif
template <class T, int L> struct YICfg {
    static constexpr int CS = sizeof(C2<T>);
    // 128-byte tile rows; 64-byte rows where three 128-byte half-tile slots exceed 200 KB (f32 Py = 2048)
    static constexpr int W = (3 * (L / 2) * 128 <= 200 * 1024 ? 128 : 64) / CS;
    static constexpr int NT = clampNT(W * L / regE<T>());
    static constexpr int MINB = NT >= 512 ? 1 : 2;
    static constexpr int R0 = Plan<T, L>::R0, R1 = Plan<T, L>::R1;
    static constexpr int HALF = L / 2;                        // rows per slot
    static constexpr int SLOTE = HALF * W;                    // slot size in elements
    static constexpr int SLOT = SLOTE * CS;                   // bytes per slot
    static constexpr int BOX = HALF < 256 ? HALF : 256;       // TMA box rows (<= 256)
    static constexpr int SMEM = 3 * SLOT + 128;               // + TMA alignment
    static constexpr bool OK = (Plan<T, L>::S == 2 || (MFD_K4_TMA3 && Plan<T, L>::S == 3)) && SMEM <= 200 * 1024 &&
                               L >= 256;
};

template <class T, int L, bool FY>
__global__ void __launch_bounds__(YICfg<T, L>::NT, YICfg<T, L>::MINB)
k_fft_y_inv_tma(Geo g, const __grid_constant__ CUtensorMap tmB, C2<T>* __restrict__ A,
                const C2<T>* __restrict__ tw, Ctl ctl, int ntx, int comp0, int ncomp) {
    using CF = YICfg<T, L>;
    constexpr int W = CF::W, NT = CF::NT, R0 = CF::R0, R1 = CF::R1, HALF = CF::HALF;
    constexpr bool CFAST = MFD_K4_COMPFAST && Plan<T, L>::S == 3;   // tile order (see MFD_K4_COMPFAST)
    // no halt check: K2-K4 touch only spectrum scratch (see Ctl)
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C2<T>* slot0 = align128(reinterpret_cast<C2<T>*>(smem_raw));
    __shared__ uint64_t bar[3];
    const int ny = g.ny, nz = g.nzg, Hp = g.Hp;   // all planes of this rank's x-bin block
    const int ntiles = ntx * nz * ncomp;          // components [comp0, comp0 + ncomp)
    if ((int)blockIdx.x >= ntiles) return;
    // fill f = 2 i + h (tile i of this CTA, half h) -> slot f % 3, phase (f / 3) & 1
    auto issue = [&](int i, int h) {   // one thread
        const int tt = blockIdx.x + i * gridDim.x;
        if (tt >= ntiles) return;
        const int bx = CFAST ? (tt / ncomp) % ntx : tt % ntx;
        const int k = CFAST ? tt / (ncomp * ntx) : (tt / ntx) % nz;
        const int comp = comp0 + (CFAST ? tt % ncomp : tt / (ntx * nz));
        const int u0 = bx * W;
        const int row0 = (comp * nz + k) * L + h * CF::HALF;
        const int s = (2 * i + h) % 3;
        mbar_arrive_expect_tx(&bar[s], (unsigned)CF::SLOT);
        for (int r = 0; r < HALF; r += CF::BOX)
            tma_load_2d(slot0 + s * CF::SLOTE + r * W, &tmB, u0 * (CF::CS / 8), row0 + r, &bar[s]);
    };
    if (threadIdx.x == 0) {
        for (int s = 0; s < 3; ++s) mbar_init(&bar[s], 1);
        mbar_fence_init();
        tma_prefetch_desc(&tmB);
    }
    __syncthreads();
    if (threadIdx.x == 0) { issue(0, 0); issue(0, 1); issue(1, 0); }
#pragma unroll 1
    for (int i = 0;; ++i) {
        const int t = blockIdx.x + i * gridDim.x;
        if (t >= ntiles) break;
        const int bx = CFAST ? (t / ncomp) % ntx : t % ntx;
        const int k = CFAST ? t / (ncomp * ntx) : (t / ntx) % nz;
        const int comp = comp0 + (CFAST ? t % ncomp : t / (ntx * nz));
        const int u0 = bx * W;
        C2<T>* sa = slot0 + ((2 * i) % 3) * CF::SLOTE;
        C2<T>* sb = slot0 + ((2 * i + 1) % 3) * CF::SLOTE;
        C2<T>* dst = A + arow_y(g, comp, k, 0) + u0;
        auto stn = [&](int col, int pos, C2<T> v) {
            if (FY || pos < ny) dst[pos * Hp + col] = v;
        };
        mbar_wait(&bar[(2 * i) % 3], ((2 * i) / 3) & 1);
        mbar_wait(&bar[(2 * i + 1) % 3], ((2 * i + 1) / 3) & 1);
        // transposed stage 1 (MP = 1, no twiddles): task p owns rows p*R1 ..
        // p*R1+R1-1, all in one slot; in place, so no barrier between gather and scatter
        if constexpr (Plan<T, L>::S == 3) {
            // three-stage plans: the transposed stages 2 (MP = 1) and 1 (MP = R2)
            // through the generic stage over the two slots; every task scatters to
            // the positions it gathered, so both run in place without a mid barrier
            auto lds = [&](int col, int pos) -> C2<T> {
                return pos < HALF ? sa[pos * W + col] : sb[(pos - HALF) * W + col];
            };
            auto sts = [&](int col, int pos, C2<T> v) {
                if (pos < HALF) sa[pos * W + col] = v;
                else sb[(pos - HALF) * W + col] = v;
            };
            fft_stage<T, L, 2, true, W, NT, true, false>(lds, sts, tw);
            __syncthreads();
            fft_stage<T, L, 1, true, W, NT, true, false>(lds, sts, tw);
        } else {
            constexpr int TPT1 = (W * R0 + NT - 1) / NT;
            static_assert((W * R0) % NT == 0 && R0 * R1 == L, "two-stage plan, whole tasks per thread");
#pragma unroll
            for (int q = 0; q < TPT1; ++q) {
                const int e = threadIdx.x + q * NT, col = e % W, p = e / W;
                C2<T>* b = (2 * p < R0 ? sa + p * R1 * W : sb + (p * R1 - HALF) * W) + col;
                C2<T> x[R1];
#pragma unroll
                for (int j = 0; j < R1; ++j) x[j] = b[j * W];
                dft<T, R1, true>(x);
#pragma unroll
                for (int j = 0; j < R1; ++j) b[j * W] = x[j];
            }
        }
        __syncthreads();
        // transposed stage 0: task n2 gathers rows n2 + MP*j (j < R0/2 in the
        // first slot, resolved at compile time), barrier, refill both slots
        // while this tile's DFTs and HBM stores run
        constexpr int MP = L / R0, TPT = (W * MP + NT - 1) / NT;
        static_assert((W * MP) % NT == 0, "whole tasks per thread");
        C2<T> v[TPT][R0];
#pragma unroll
        for (int q = 0; q < TPT; ++q) {
            const int e = threadIdx.x + q * NT, col = e % W, n2 = e / W;
#pragma unroll
            for (int j = 0; j < R0; ++j)
                v[q][j] = 2 * j < R0 ? sa[(n2 + MP * j) * W + col] : sb[(n2 + MP * j - HALF) * W + col];
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            fence_proxy_async_smem();
            issue(i + 1, 1);
            issue(i + 2, 0);
        }
#pragma unroll
        for (int q = 0; q < TPT; ++q) {
            const int e = threadIdx.x + q * NT, col = e % W, n2 = e / W;
#pragma unroll
            for (int k = 1; k < R0; ++k) v[q][k] = cmulc<T>(v[q][k], tw_lookup<T, L, L>(tw, n2 * k));
            dft<T, R0, true, false, true>(v[q]);
#pragma unroll
            for (int j = 0; 2 * j < R0; ++j) stn(col, n2 + MP * j, v[q][j]);
        }
    }
}

// ------------------------------------------------------------------ K3
// One CTA: W x-bins, the y-frequency pair {v, Py-v}, all three components,
// full z columns.  Forward z (nz active inputs) -> per-bin symmetric real
// 3x3 product with the tensor octant (mirror signs applied on the fly) ->
// inverse z (nz outputs kept).  Nothing padded in z touches HBM.
template <class T, int L>
__global__ void __launch_bounds__(ZCfg<T, L>::NT)
k_fft_z_conv(Geo g, C2<T>* __restrict__ B, const T* __restrict__ Kt, const C2<T>* __restrict__ tw,
             const int* __restrict__ ybuf, Ctl ctl) {
    using CF = ZCfg<T, L>;
    constexpr int W = CF::W, NCOL = CF::NCOL, NT = CF::NT;
    // no halt check: K2-K4 touch only spectrum scratch (see Ctl)
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C2<T>* sm = reinterpret_cast<C2<T>*>(smem_raw);
    const int u0 = blockIdx.x * W;               // x-bin within this rank's block
    const int v = blockIdx.y;                    // 0..Py/2
    const int Py = g.Py, nz = g.nzg, Wb = g.Wb, Hv = g.Hv;
    const int vp = (Py - v) & (Py - 1);
    const bool pair = vp != v;
    const long long rowA = ybuf[v], rowB = ybuf[vp];   // buffer rows of v and Py-v
    // column c = comp*2W + r*W + w  (r: 0 -> v, 1 -> Py-v)
    auto gaddr = [&](int col, int pos) -> long long {
        const int comp = col / (2 * W), r = (col / W) & 1, w = col % W;
        return comp * g.S_c + (long long)pos * g.S_k + (r ? rowB : rowA) * Wb + u0 + w;
    };
    auto valid = [&](int col) { return u0 + (col % W) < Hv && (pair || ((col / W) & 1) == 0); };
    auto ld0 = [&](int col, int pos) -> C2<T> {
        if (pos >= nz || !valid(col)) return mk<T>(0, 0);
        return B[gaddr(col, pos)];
    };
    auto lds = [&](int col, int pos) -> C2<T> { return sm[pos * NCOL + col]; };
    auto sts = [&](int col, int pos, C2<T> val) { sm[pos * NCOL + col] = val; };
    auto stn = [&](int col, int pos, C2<T> val) {
        if (pos < nz && valid(col)) B[gaddr(col, pos)] = val;
    };
    fft_forward<T, L, NCOL, NT, true, false, true>(ld0, lds, sts, sts, tw);
    __syncthreads();
    // K~ . M~ : thread task (w, wq) covers z-frequencies {wq, Pz-wq} and both y rows.
    const int Hz = L / 2 + 1;
    const T* kbase = Kt + (((long long)v * Hz) * Wb + u0) * 6;
    for (int e = threadIdx.x; e < W * Hz; e += NT) {
        const int w = e % W, wq = e / W;
        if (u0 + w >= Hv) continue;
        const T* kp = kbase + ((long long)wq * Wb + w) * 6;
        const T kxx = __ldg(kp), kyy = __ldg(kp + 1), kzz = __ldg(kp + 2);
        const T kxy = __ldg(kp + 3), kxz = __ldg(kp + 4), kyz = __ldg(kp + 5);
        const int wpart = (L - wq) & (L - 1);
        const int nzf = wpart != wq ? 2 : 1;
        const int nr = pair ? 2 : 1;
        for (int zi = 0; zi < nzf; ++zi) {
            const int wf = zi ? wpart : wq;
            const T sz = zi ? T(-1) : T(1);
            const int pos = bufpos<T, L>(wf);
            for (int r = 0; r < nr; ++r) {
                const T sy = r ? T(-1) : T(1);
                C2<T>* s = sm + pos * NCOL + r * W + w;
                const C2<T> mx = s[0], my = s[2 * W], mz = s[4 * W];
                const T cxy = sy * kxy, cxz = sz * kxz, cyz = sy * sz * kyz;
                s[0] = mk<T>(kxx * mx.x + cxy * my.x + cxz * mz.x, kxx * mx.y + cxy * my.y + cxz * mz.y);
                s[2 * W] = mk<T>(cxy * mx.x + kyy * my.x + cyz * mz.x, cxy * mx.y + kyy * my.y + cyz * mz.y);
                s[4 * W] = mk<T>(cxz * mx.x + cyz * my.x + kzz * mz.x, cxz * mx.y + cyz * my.y + kzz * mz.y);
            }
        }
    }
    __syncthreads();
    fft_inverse<T, L, NCOL, NT, true, true, false>(lds, lds, sts, stn, tw);
}

// Tensor product at one z-frequency for the three components of one y row.
// Kt octant entry at (u, v', w'); sy / sz are the mirror signs of the
// partner row Py-v / partner plane Pz-w (odd components flip).
// kp points at the bin's six interleaved components (Kt layout [v][w][u][6]),
// read as three 8/16-byte vectors.
template <class T>
struct KBin { C2<T> k01, k23, k45; };
template <class T>
__device__ __forceinline__ KBin<T> kload(const T* __restrict__ kp) {
    KBin<T> k;
    k.k01 = __ldg(reinterpret_cast<const C2<T>*>(kp));
    k.k23 = __ldg(reinterpret_cast<const C2<T>*>(kp) + 1);
    k.k45 = __ldg(reinterpret_cast<const C2<T>*>(kp) + 2);
    return k;
}
template <class T>
__device__ __forceinline__ void kmul(C2<T>& mx, C2<T>& my, C2<T>& mz, const KBin<T>& kb, T sy, T sz) {
    const C2<T> k01 = kb.k01, k23 = kb.k23, k45 = kb.k45;
    const T kxx = k01.x, kyy = k01.y, kzz = k23.x;
    const T cxy = sy * k23.y, cxz = sz * k45.x;
    const T cyz = sy * sz * k45.y;
    const C2<T> a = mx, b = my, c = mz;
    mx = mk<T>(kxx * a.x + cxy * b.x + cxz * c.x, kxx * a.y + cxy * b.y + cxz * c.y);
    my = mk<T>(cxy * a.x + kyy * b.x + cyz * c.x, cxy * a.y + kyy * b.y + cyz * c.y);
    mz = mk<T>(cxz * a.x + cyz * b.x + kzz * c.x, cxz * a.y + cyz * b.y + kzz * c.y);
}
template <class T>
__device__ __forceinline__ void kmul(C2<T>& mx, C2<T>& my, C2<T>& mz, const T* __restrict__ kp, T sy, T sz) {
    const C2<T> k01 = __ldg(reinterpret_cast<const C2<T>*>(kp));
    const C2<T> k23 = __ldg(reinterpret_cast<const C2<T>*>(kp) + 1);
    const C2<T> k45 = __ldg(reinterpret_cast<const C2<T>*>(kp) + 2);
    const T kxx = k01.x, kyy = k01.y, kzz = k23.x;
    const T cxy = sy * k23.y, cxz = sz * k45.x;
    const T cyz = sy * sz * k45.y;
    const C2<T> a = mx, b = my, c = mz;
    mx = mk<T>(kxx * a.x + cxy * b.x + cxz * c.x, kxx * a.y + cxy * b.y + cxz * c.y);
    my = mk<T>(cxy * a.x + kyy * b.x + cyz * c.x, cxy * a.y + kyy * b.y + cyz * c.y);
    mz = mk<T>(cxz * a.x + cyz * b.x + kzz * c.x, cxz * a.y + cyz * b.y + kzz * c.y);
}

// K3, two-stage plans (Pz = R0*R1).  Thread (x-bin w, stage-0 task n2, y-row
// r) runs forward stage 0 for the three components with one set of twiddles
// (HBM -> shared); then one thread per (w, k0, r) holds the three components
// of its R1 frequencies f = k0 + R0*k1 in registers through forward stage 1,
// the tensor product and the transposed inverse stage 1 (same positions), so
// the product costs no extra shared-memory round trip; the inverse stage 0
// goes shared -> HBM keeping the nz planes.
// SROW: one y row per CTA (the CTAs of rows v and Py-v are launched next to
// each other, so the second one's tensor bins come from L2) instead of the
// pair {v, Py-v}: half the shared memory and threads, twice the CTAs per SM.
#ifndef MFD_K3_R1_256
// f32 K3 at Pz = 256: radix 32 x 8 instead of the shared plan's 16 x 16 (stage 1 as at
// Pz = 128, tensor bins prefetched; 128 threads, 252 registers, 2 CTAs/SM):
// C5 K3 5.69 -> 5.35 ms, C3 0.113 -> 0.108 ms.  0: the shared plan
#define MFD_K3_R1_256 8
#endif
template <class T, int L, bool SROW = false> struct Z2Cfg {
    static constexpr int R1 = sizeof(T) == 4 && L == 256 && MFD_K3_R1_256 > 0 ? MFD_K3_R1_256 : Plan<T, L>::R1;
    static constexpr int R0 = L / R1;
    static constexpr int CS = sizeof(C2<T>);
    // f32: 16 columns (128-byte rows) also at R1 = 16 (Pz = 256, C5: 7.68 -> 7.07 ms)
    static constexpr int W = MFD_Z2_W > 0 && sizeof(T) == 4 ? MFD_Z2_W
                             : sizeof(T) == 4 ? 16
                             : MFD_Z2_F64_W > 0 ? MFD_Z2_F64_W : 8 / (R1 >= 16 ? 2 : 1);
    static constexpr int NROW = SROW ? 1 : 2;
    static constexpr int NCOL = 3 * NROW * W;
    static constexpr int NT = W * R1 * NROW;
    static constexpr int SMEM = NCOL * L * CS;
    // resident CTAs per SM the register budget is sized for (shared memory permitting)
    // tensor bins loaded one phase ahead (register budget: R1 <= 8 only)
    static constexpr bool KPRE = R1 <= 8 && (sizeof(T) == 4 || MFD_K3_F64_KPRE);
    // R1 = 16 (Pz = 256), f32: a 128-register budget for 2 CTAs/SM instead of
    // 254 registers at 1 CTA/SM (8 warps): C5 K3 7.14 -> 6.06 ms, C3 0.134 -> 0.121 ms
    static constexpr int MINB = KPRE ? cmax(1, cmin(2 * (3 - NROW), (200 * 1024) / SMEM))
                                     : (sizeof(T) == 4 && 2 * SMEM <= 200 * 1024 ? 2 : 1);
};

// FZ: nz == Pz/2, so the pruned first/last stages never meet a plane >= nz.
// Padding x-bins (>= Hv, inside the block pitch) are computed, not masked.
template <class T, int L, bool FZ, bool SROW = false>
__global__ void __launch_bounds__(Z2Cfg<T, L, SROW>::NT, Z2Cfg<T, L, SROW>::MINB)
k_fft_z_conv2(Geo g, C2<T>* __restrict__ B, const T* __restrict__ Kt, const C2<T>* __restrict__ tw,
              const int* __restrict__ ybuf, Ctl ctl) {
    using CF = Z2Cfg<T, L, SROW>;
    constexpr int W = CF::W, NCOL = CF::NCOL, R0 = CF::R0, R1 = CF::R1;
    constexpr int CO = CF::NROW * W;   // column stride of the components
    static_assert(Plan<T, L>::S == 2 && R0 % R1 == 0 && R0 <= 32, "two-stage plans with R0 % R1 == 0 only");
    // no halt check: K2-K4 touch only spectrum scratch (see Ctl)
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C2<T>* sm = reinterpret_cast<C2<T>*>(smem_raw);
    const int u0 = blockIdx.x * W;               // x-bin within this rank's block
    const int Py = g.Py, nz = g.nzg, Wb = g.Wb;
    // SROW: y block b -> frequency pair v = (b+1)/2, row v (r = 0) or Py-v (r = 1)
    const int v = SROW ? ((int)blockIdx.y + 1) / 2 : (int)blockIdx.y;
    const int vp = (Py - v) & (Py - 1);
    const bool pair = vp != v;
    const int w = threadIdx.x % W, n2 = (threadIdx.x / W) % R1;
    const int r = SROW ? (pair ? (int)(blockIdx.y & 1) : 0) : (int)threadIdx.x / (W * R1);
    const bool live = SROW || pair || r == 0;
    const long long cstride = g.S_c;
    C2<T>* gcol = B + (long long)(r ? ybuf[vp] : ybuf[v]) * Wb + u0 + w;   // + comp*S_c + k*S_k
    // smem column of (comp c, row r, bin w): c*CO + r*W + w; layout [pos][NCOL]
    C2<T>* scol = sm + (SROW ? 0 : r * W) + w;
    // tensor bins of the register phases (see stage 1 below)
    const int Hz = L / 2 + 1;
    const T sy = r ? T(-1) : T(1);
    const T* kb = Kt + ((long long)v * Hz * Wb + u0 + w) * 6;
    KBin<T> kv[CF::KPRE ? R1 : 1];
    auto kfetch = [&](int it) {
#pragma unroll
        for (int k1 = 0; k1 < R1; ++k1) {
            const int f = n2 + R1 * it + R0 * k1;
            kv[k1] = kload<T>(kb + (long long)(2 * f > L ? L - f : f) * Wb * 6);
        }
    };
    // ---- forward stage 0: x[R1*j + n2], j < R0/2 (upper half is padding).
    {
        // All three components' inputs go into flight at kernel entry as
        // cp.async copies into the thread's own shared-memory slots (the
        // positions R1*j + n2 its stage-0 task reads and then overwrites), one
        // commit group per component: no staging registers, and the HBM
        // latency of components 1 and 2 hides behind component 0's DFT
        // (C4 f32: 0.584 -> 0.553 ms against a register pipeline that fetched
        // component c+1 while transforming c).
#pragma unroll
        for (int c = 0; c < 3; ++c) {
#pragma unroll
            for (int j = 0; j < R0 / 2; ++j) {
                const int pos = R1 * j + n2;
                C2<T>* d = scol + pos * NCOL + c * CO;
                if (live && (FZ || pos < nz)) cp_async_c2<T>(d, gcol + c * cstride + (long long)pos * g.S_k);
                else *d = mk<T>(0, 0);
            }
            cp_commit();
        }
        C2<T> twr[R0];
#pragma unroll
        for (int k = 1; k < R0; ++k) twr[k] = __ldg(tw_dense<T, L>(tw) + n2 * k);
#pragma unroll 1
        for (int c = 0; c < 3; ++c) {
            if (c == 0) cp_wait<2>();
            else if (c == 1) cp_wait<1>();
            else cp_wait<0>();
            // first phase's tensor bins in flight during the last component's DFT
            if constexpr (CF::KPRE && MFD_K3_KEARLY) if (c == 2 && live) kfetch(0);
            C2<T> x[R0];
#pragma unroll
            for (int j = 0; j < R0; ++j) x[j] = 2 * j < R0 ? scol[(R1 * j + n2) * NCOL + c * CO] : mk<T>(0, 0);
            dft<T, R0, false, true>(x);
#pragma unroll
            for (int k = 1; k < R0; ++k) x[k] = cmul<T>(x[k], twr[k]);
#pragma unroll
            for (int k = 0; k < R0; ++k) scol[(k * R1 + n2) * NCOL + c * CO] = x[k];
        }
    }
    // ---- stage 1 + tensor product + inverse stage 1, in registers.  The
    // tensor bins of iteration it are loaded one phase ahead (before the
    // barrier for it = 0, after the product of it - 1 otherwise), so their
    // HBM latency overlaps the shared-memory gather and the stage-1 DFTs.
    if constexpr (CF::KPRE && !MFD_K3_KEARLY) if (live) kfetch(0);
    __syncthreads();
#pragma unroll
    for (int it = 0; it < R0 / R1; ++it) {
        const int k0 = n2 + R1 * it;
        C2<T> y[3][R1];
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
            for (int q = 0; q < R1; ++q) y[c][q] = scol[(k0 * R1 + q) * NCOL + c * CO];
#pragma unroll
        for (int c = 0; c < 3; ++c) dft<T, R1, false>(y[c]);
        if (live) {
#pragma unroll
            for (int k1 = 0; k1 < R1; ++k1) {
                const int f = k0 + R0 * k1;
                const bool hi = 2 * f > L;
                if constexpr (CF::KPRE)
                    kmul<T>(y[0][k1], y[1][k1], y[2][k1], kv[k1], sy, hi ? T(-1) : T(1));
                else
                    kmul<T>(y[0][k1], y[1][k1], y[2][k1], kb + (long long)(hi ? L - f : f) * Wb * 6, sy,
                            hi ? T(-1) : T(1));
            }
            if constexpr (CF::KPRE) if (it + 1 < R0 / R1) kfetch(it + 1);
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) dft<T, R1, true>(y[c]);
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
            for (int q = 0; q < R1; ++q) scol[(k0 * R1 + q) * NCOL + c * CO] = y[c][q];
    }
    __syncthreads();
    // ---- inverse stage 0 (transposed): gather k0*R1 + n2, conj twiddle, IDFT, keep z < nz
    C2<T> twr[R0];
#pragma unroll
    for (int k = 1; k < R0; ++k) twr[k] = __ldg(tw_dense<T, L>(tw) + n2 * k);
#pragma unroll 1
    for (int c = 0; c < 3; ++c) {
        C2<T> x[R0];
#pragma unroll
        for (int k = 0; k < R0; ++k) x[k] = scol[(k * R1 + n2) * NCOL + c * CO];
#pragma unroll
        for (int k = 1; k < R0; ++k) x[k] = cmulc<T>(x[k], twr[k]);
        dft<T, R0, true, false, true>(x);
        if (live) {
#pragma unroll
            for (int j = 0; 2 * j < R0; ++j) {
                const int pos = R1 * j + n2;
                if (FZ || pos < nz) gcol[c * cstride + (long long)pos * g.S_k] = x[j];
            }
        }
    }
}

// Which K3 variant a z length uses: 1 = all-register (L <= 16), 2 = two-stage
// register product (fits shared memory), 0 = generic staged kernel.
template <class T, int L>
constexpr int z_variant() {
    if constexpr (L <= 16 && Plan<T, L>::S <= 1) return 1;
    else if constexpr (Plan<T, L>::S == 2 && Z2Cfg<T, L>::SMEM <= 200 * 1024 && Z2Cfg<T, L>::NT <= 1024) return 2;
    else return 0;
}

// K3, single-stage plans (Pz <= 16): one thread per (x-bin, y-row) keeps the
// three whole z-columns in registers; no shared memory, no barrier.
template <class T, int L>
__global__ void __launch_bounds__(64)
k_fft_z_conv1(Geo g, C2<T>* __restrict__ B, const T* __restrict__ Kt, const int* __restrict__ ybuf, Ctl ctl) {
    // no halt check: K2-K4 touch only spectrum scratch (see Ctl)
    const int w = threadIdx.x & 31, r = threadIdx.x >> 5;
    const int u = blockIdx.x * 32 + w;           // x-bin within this rank's block
    const int v = blockIdx.y;
    const int Py = g.Py, nz = g.nzg, Wb = g.Wb;
    const int vp = (Py - v) & (Py - 1);
    if (u >= g.Hv || (r == 1 && vp == v)) return;
    const long long row = r ? ybuf[vp] : ybuf[v];
    const long long cstride = g.S_c;
    C2<T>* base = B + row * Wb + u;
    C2<T> x[3][L];
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int k = 0; k < L; ++k) x[c][k] = (k < nz && 2 * k < L) ? base[c * cstride + (long long)k * g.S_k] : mk<T>(0, 0);
#pragma unroll
    for (int c = 0; c < 3; ++c) dft<T, L, false, true>(x[c]);
    const int Hz = L / 2 + 1;
    const T* kb = Kt + ((long long)v * Hz * Wb + u) * 6;
    const T sy = r ? T(-1) : T(1);
#pragma unroll
    for (int f = 0; f < L; ++f) {
        const bool hi = 2 * f > L;
        kmul<T>(x[0][f], x[1][f], x[2][f], kb + (long long)(hi ? L - f : f) * Wb * 6, sy, hi ? T(-1) : T(1));
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) dft<T, L, true, false, true>(x[c]);
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int k = 0; k < L; ++k)
            if (k < nz && 2 * k < L) base[c * cstride + (long long)k * g.S_k] = x[c][k];
}

// ------------------------------------------------------------ K2+K3+K4
// Thin / small problems (Pz <= 16 and the y-z spectrum of a few x bins fits
// in shared memory, e.g. SP4 128x32x1 and 512x128x4): one kernel per step does
// the forward y FFT (A -> shared), the z transform + tensor product + inverse z
// in registers (one thread per (y frequency, x bin), as k_fft_z_conv1) and
// the inverse y FFT (shared -> A), so the three passes cost one launch and no
// B round trip.  Arithmetic per column is the same as K2 / K3 / K4.
#ifndef MFD_YZ_W
// y-z small pass: x bins per CTA (upper bound).  One bin per 32-thread CTA (129 CTAs at
// SP4) instead of 4 per 128 threads: SP4 0.0114 -> 0.0106 ms/step
#define MFD_YZ_W 1
#endif
template <class T, int LY, int LZ> struct YZCfg {
    static constexpr int CS = sizeof(C2<T>);
    static constexpr int NZH = LZ / 2 > 0 ? LZ / 2 : 1;               // z planes held (nz <= LZ/2)
    static constexpr int W = cmax(1, cmin(MFD_YZ_W, 4096 / (3 * NZH * LY)));  // x bins per CTA
    static constexpr int NCOL = 3 * NZH * W;                            // columns (comp, z, bin)
    static constexpr int NT = MFD_YZ_W == 4 ? 128 : 32 * MFD_YZ_W;
    static constexpr int SMEM = NCOL * LY * CS;
    // Measured (f32): SP4 128x32x1 0.0164 -> 0.0107 ms/step; at 512x128x4 (W = 1)
    // the per-CTA work is too thin and the separate passes win (0.040 vs 0.057 ms)
    static constexpr bool OK = LZ <= 16 && Plan<T, LZ>::S <= 1 && SMEM <= 48 * 1024 && Plan<T, LY>::S >= 1 &&
                               3 * NZH * LY <= 1024;
};

template <class T, int LY, int LZ>
__device__ __forceinline__ void yz_body(const Geo& g, C2<T>* __restrict__ A, const T* __restrict__ Kt,
                                        const C2<T>* __restrict__ tw, const int* __restrict__ ybuf, int bx,
                                        unsigned char* smem_raw) {
    using CF = YZCfg<T, LY, LZ>;
    constexpr int W = CF::W, NZH = CF::NZH, NCOL = CF::NCOL, NT = CF::NT;
    C2<T>* sm = reinterpret_cast<C2<T>*>(smem_raw);    // [y position][NCOL]
    const int u0 = bx * W;
    const int ny = g.ny, nz = g.nz, Hp = g.Hp;
    // column col = (comp * NZH + z) * W + w
    auto arow = [&](int col, int y) -> long long {
        const int w = col % W, z = (col / W) % NZH, c = col / (W * NZH);
        return ((long long)(c * nz + z) * ny + y) * Hp + u0 + w;
    };
    auto zok = [&](int col) { return (col / W) % NZH < nz; };
    auto ld0 = [&](int col, int pos) -> C2<T> {
        return (pos < ny && zok(col)) ? A[arow(col, pos)] : mk<T>(0, 0);
    };
    auto lds = [&](int col, int pos) -> C2<T> { return sm[pos * NCOL + col]; };
    auto sts = [&](int col, int pos, C2<T> v) { sm[pos * NCOL + col] = v; };
    const int Hz = LZ / 2 + 1;
    fft_forward<T, LY, NCOL, NT, true, false, true>(ld0, lds, sts, sts, tw);
    __syncthreads();
    // z: one item per (y frequency v, bin w); frequencies in natural order
    for (int e = threadIdx.x; e < LY * W; e += NT) {
        const int w = e % W, v = e / W;
        const int pos = ybuf[v];
        const bool vhi = 2 * v > LY;
        C2<T> x[3][LZ];
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
            for (int k = 0; k < LZ; ++k)
                x[c][k] = (k < NZH && 2 * k < LZ && k < nz) ? sm[pos * NCOL + (c * NZH + k) * W + w] : mk<T>(0, 0);
#pragma unroll
        for (int c = 0; c < 3; ++c) dft<T, LZ, false, true>(x[c]);
        const T* kb = Kt + ((long long)(vhi ? LY - v : v) * Hz * g.Wb + u0 + w) * 6;
        const T sy = vhi ? T(-1) : T(1);
#pragma unroll
        for (int f = 0; f < LZ; ++f) {
            const bool hi = 2 * f > LZ;
            kmul<T>(x[0][f], x[1][f], x[2][f], kb + (long long)(hi ? LZ - f : f) * g.Wb * 6, sy, hi ? T(-1) : T(1));
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) dft<T, LZ, true, false, true>(x[c]);
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
            for (int k = 0; k < NZH; ++k) sm[pos * NCOL + (c * NZH + k) * W + w] = x[c][k];
    }
    __syncthreads();
    auto stn = [&](int col, int pos, C2<T> v) {
        if (pos < ny && zok(col)) A[arow(col, pos)] = v;
    };
    fft_inverse<T, LY, NCOL, NT, true, true, false>(lds, lds, sts, stn, tw);
}

template <class T, int LY, int LZ>
__global__ void __launch_bounds__(YZCfg<T, LY, LZ>::NT)
k_fft_yz_small(Geo g, C2<T>* __restrict__ A, const T* __restrict__ Kt, const C2<T>* __restrict__ tw,
               const int* __restrict__ ybuf, Ctl ctl) {
    // no halt check: K2-K4 touch only spectrum scratch (see Ctl)
    extern __shared__ __align__(16) unsigned char smem_raw[];
    yz_body<T, LY, LZ>(g, A, Kt, tw, ybuf, blockIdx.x, smem_raw);
}

// ------------------------------------------------------------------ K5
// Local fields + LLG + Euler on one cell, in the reference's operation order
// without FMA contraction (fields.hpp:33-48, 72-76, 246-250; dynamics.hpp:58-62, 101-108).
template <class T> struct LocalParams {
    T cx, cy, cz;          // exchange 2A/(mu0 Ms^2)/d^2 (fields.hpp:25-27)
    int exch, anis, zee;   // gates (fields.hpp:239-245)
    T ca;                  // 2Ku/(mu0 Ms^2)
    T ax, ay, az;          // easy axis
    T hx, hy, hz;          // uniform external field
    T precess, damp, mu0;  // LLG (dynamics.hpp:54-57)
    T dt, Ms;
    double dA, dMs, dKu, dV;   // energy scalars (double)
    double dax, day, daz, dhx, dhy, dhz;
    double wx, wy, wz;     // 1/d^2 (fields.hpp:147-148)
};

struct StepIO {
    int update;            // write M_new
    int renorm;            // renormalise this step
    int write_h;           // 0 none, 1 H_eff, 2 H_demag
    int sums;              // accumulate sample sums
    int iter;              // iteration index stored in err on failure
    unsigned long long* torque;   // max |rhs|^2 bits
    double* partials;      // [gridDim.x][8]
    double* sums_out;      // [8]
    unsigned int* ticket;
};

template <class T>
__device__ __forceinline__ void cell_update(const Geo& g, const LocalParams<T>& P, const StepIO& io,
                                            const T* __restrict__ M, T* __restrict__ Mn,
                                            T* __restrict__ Hout, const Halo<T>& hl, long long c, int i, int j,
                                            int k, T hdx, T hdy, T hdz, double& tmax, double* acc,
                                            int& bad) {
    const long long n = g.ncell;
    const T mx = M[c], my = M[c + n], mz = M[c + 2 * n];
    T Hx = hdx, Hy = hdy, Hz = hdz;
    double elink = 0;
    if (P.exch) {
        T h0 = 0, h1 = 0, h2 = 0;
        const long long sy = g.nx, sz = (long long)g.nx * g.ny;
        // neighbour values at q[0], q[cs], q[2cs] (cs = component stride)
        auto add = [&](const T* q, long long cs, T w) {
            h0 = add_rn(h0, mul_rn(w, sub_rn(q[0], mx)));
            h1 = add_rn(h1, mul_rn(w, sub_rn(q[cs], my)));
            h2 = add_rn(h2, mul_rn(w, sub_rn(q[2 * cs], mz)));
        };
        auto link = [&](const T* q, long long cs, double w) {
            const double e0 = (double)q[0] - mx, e1 = (double)q[cs] - my, e2 = (double)q[2 * cs] - mz;
            elink += w * (e0 * e0 + e1 * e1 + e2 * e2);
        };
        const int kg = g.k0 + k;
        const long long inplane = c - (long long)k * sz;
        const T* zlo = k > 0 ? M + c - sz : hl.lo + inplane;
        const T* zhi = k < g.nz - 1 ? M + c + sz : hl.hi + inplane;
        const long long zlo_cs = k > 0 ? n : sz, zhi_cs = k < g.nz - 1 ? n : sz;
        if (i > 0) add(M + c - 1, n, P.cx);
        if (i < g.nx - 1) { add(M + c + 1, n, P.cx); if (io.sums) link(M + c + 1, n, P.wx); }
        if (j > 0) add(M + c - sy, n, P.cy);
        if (j < g.ny - 1) { add(M + c + sy, n, P.cy); if (io.sums) link(M + c + sy, n, P.wy); }
        if (kg > 0) add(zlo, zlo_cs, P.cz);
        if (kg < g.nzg - 1) { add(zhi, zhi_cs, P.cz); if (io.sums) link(zhi, zhi_cs, P.wz); }
        Hx = add_rn(Hx, h0);
        Hy = add_rn(Hy, h1);
        Hz = add_rn(Hz, h2);
    }
    if (P.anis) {
        const T proj = mul_rn(P.ca, add_rn(add_rn(mul_rn(mx, P.ax), mul_rn(my, P.ay)), mul_rn(mz, P.az)));
        Hx = add_rn(Hx, mul_rn(proj, P.ax));
        Hy = add_rn(Hy, mul_rn(proj, P.ay));
        Hz = add_rn(Hz, mul_rn(proj, P.az));
    }
    if (P.zee) {
        Hx = add_rn(Hx, P.hx);
        Hy = add_rn(Hy, P.hy);
        Hz = add_rn(Hz, P.hz);
    }
    if (io.write_h == 1) {
        Hout[c] = Hx; Hout[c + n] = Hy; Hout[c + 2 * n] = Hz;
    } else if (io.write_h == 2) {
        Hout[c] = hdx; Hout[c + n] = hdy; Hout[c + 2 * n] = hdz;
    }
    if (io.sums) {
        acc[0] += (double)mx;
        acc[1] += (double)my;
        acc[2] += (double)mz;
        acc[3] += elink;
        const double m0 = (double)mx / P.dMs, m1 = (double)my / P.dMs, m2 = (double)mz / P.dMs;
        const double p = m0 * P.dax + m1 * P.day + m2 * P.daz;
        acc[4] += 1.0 - p * p;
        acc[5] += (double)hdx * mx + (double)hdy * my + (double)hdz * mz;
        acc[6] += P.dhx * mx + P.dhy * my + P.dhz * mz;
    }
    // llgRhs: h = mu0*H; mxh = m x h; rhs = precess*mxh + damp*(m x mxh)
    const T b0 = mul_rn(P.mu0, Hx), b1 = mul_rn(P.mu0, Hy), b2 = mul_rn(P.mu0, Hz);
    const T c0 = sub_rn(mul_rn(my, b2), mul_rn(mz, b1));
    const T c1 = sub_rn(mul_rn(mz, b0), mul_rn(mx, b2));
    const T c2 = sub_rn(mul_rn(mx, b1), mul_rn(my, b0));
    const T d0 = sub_rn(mul_rn(my, c2), mul_rn(mz, c1));
    const T d1 = sub_rn(mul_rn(mz, c0), mul_rn(mx, c2));
    const T d2 = sub_rn(mul_rn(mx, c1), mul_rn(my, c0));
    const T r0 = add_rn(mul_rn(P.precess, c0), mul_rn(P.damp, d0));
    const T r1 = add_rn(mul_rn(P.precess, c1), mul_rn(P.damp, d1));
    const T r2 = add_rn(mul_rn(P.precess, c2), mul_rn(P.damp, d2));
    {
        const double v0 = r0, v1 = r1, v2 = r2;
        const double t2 = __dadd_rn(__dadd_rn(__dmul_rn(v0, v0), __dmul_rn(v1, v1)), __dmul_rn(v2, v2));
        tmax = fmax(tmax, t2);
    }
    if (io.update) {
        T e0 = add_rn(mx, mul_rn(P.dt, r0));
        T e1 = add_rn(my, mul_rn(P.dt, r1));
        T e2 = add_rn(mz, mul_rn(P.dt, r2));
        if (io.renorm) {
            const T n2 = add_rn(add_rn(mul_rn(e0, e0), mul_rn(e1, e1)), mul_rn(e2, e2));
            if (!(n2 > T(0)) || !isfinite((double)n2)) { bad = 1; return; }
            const T f = P.Ms / sqrt(n2);
            e0 = mul_rn(f, e0); e1 = mul_rn(f, e1); e2 = mul_rn(f, e2);
        } else if (!isfinite((double)add_rn(add_rn(e0, e1), e2))) {
            bad = 1;
            return;
        }
        Mn[c] = e0; Mn[c + n] = e1; Mn[c + 2 * n] = e2;
    }
}

// Block-level epilogue shared by K5 and the demag-free kernel: torque max
// (exact; one atomicMax on the ordered bit pattern), error flag, and the
// deterministic two-level sample sums (fixed tree per block, last block
// combines the per-block partials in index order).
template <int NT>
__device__ __forceinline__ void block_finish(const StepIO& io, const Ctl& ctl, double tmax, double* acc,
                                             int bad) {
    __shared__ double red[NT / 32][8];
    __shared__ int anybad;
    __shared__ bool last;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (threadIdx.x == 0) anybad = 0;
    __syncthreads();
    if (bad) anybad = 1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tmax = fmax(tmax, __shfl_xor_sync(0xffffffffu, tmax, o));
    if (io.sums) {
#pragma unroll
        for (int q = 0; q < 7; ++q)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], o);
    }
    if (lane == 0) {
        red[wid][7] = tmax;
        if (io.sums)
            for (int q = 0; q < 7; ++q) red[wid][q] = acc[q];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = red[0][7];
        for (int w = 1; w < NT / 32; ++w) t = fmax(t, red[w][7]);
        atomicMax(io.torque, (unsigned long long)__double_as_longlong(t));
        if (anybad) atomicCAS(ctl.err, 0, io.iter + 1);
        if (io.sums) {
            double* p = io.partials + (long long)(blockIdx.x + (long long)gridDim.x * blockIdx.y) * 8;
            for (int q = 0; q < 7; ++q) {
                double s = red[0][q];
                for (int w = 1; w < NT / 32; ++w) s += red[w][q];
                p[q] = s;
            }
            __threadfence();
            const unsigned int total = gridDim.x * gridDim.y;
            last = atomicAdd(io.ticket, 1u) == total - 1;
        }
    }
    if (!io.sums) return;
    __syncthreads();
    if (!last) return;
    __threadfence();
    const unsigned int total = gridDim.x * gridDim.y;
    // fixed-order final combine by warp 0: lane l sums partials l, l+32, ... in
    // order, then a fixed xor-shuffle tree — independent of scheduling.
    if (wid != 0) return;
    for (int q = 0; q < 7; ++q) {
        double s = 0;
        for (unsigned int b = lane; b < total; b += 32) s += ((volatile double*)io.partials)[b * 8 + q];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) io.sums_out[q] = s;
    }
    if (lane == 0) *io.ticket = 0;
}

template <class T, int N, bool MULTI = false>
__global__ void __launch_bounds__(LCfg<T, N>::NT, LCfg<T, N>::MINB)
k_c2r_x_llg(Geo g, const C2<T>* __restrict__ A, const T* __restrict__ M, T* __restrict__ Mn,
            T* __restrict__ Hout, const C2<T>* __restrict__ tw, T scale, LocalParams<T> P, StepIO io,
            Ctl ctl, Halo<T> hl) {
    using CF = LCfg<T, N>;
    constexpr int ROWS = CF::ROWS, NT = CF::NT, LP = xpitch<T, N>(), NCOL = 3 * ROWS;
    if (halted(ctl)) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C2<T>* sm = reinterpret_cast<C2<T>*>(smem_raw);
    const long long nrows = (long long)g.ny * g.nz;
    const long long row0 = (long long)blockIdx.x * ROWS;
    // Complex-to-real pre-process (pairs k, N-k): Z[k] = (X[k] + conj X[N-k]) + i W^-k (X[k] - conj X[N-k]),
    // written at buffer positions so the transposed inverse stages emit natural order.
    constexpr int HALF = N / 2 + 1;
    for (int e = threadIdx.x; e < NCOL * HALF; e += NT) {
        const int col = e / HALF, k = e % HALF;
        const int comp = col / ROWS, r = col % ROWS;
        const long long row = row0 + r;
        C2<T> a = mk<T>(0, 0), b = mk<T>(0, 0);
        if (row < nrows) {
            const C2<T>* src = A + ((long long)comp * nrows + row) * g.Hp;
            a = *abin<MULTI>(g, src, k);
            b = *abin<MULTI>(g, src, N - k);
        }
        const C2<T> w = __ldg(tw_dense<T, 2 * N>(tw) + k);   // W_Px^k, used conjugated
        {
            const C2<T> s = cadd<T>(a, cconj<T>(b)), d = csub<T>(a, cconj<T>(b));
            const C2<T> wd = cmulc<T>(d, w);                     // W^-k d
            sm[col * LP + xpad<T>(bufpos<T, N>(k % N))] = mk<T>(s.x - wd.y, s.y + wd.x);
        }
        if (N - k != k && N - k < N) {
            const C2<T> s = cadd<T>(b, cconj<T>(a)), d = csub<T>(b, cconj<T>(a));
            const C2<T> wn = mk<T>(-w.x, w.y);                  // W_Px^{N-k} = -conj(W^k)
            const C2<T> wd = cmulc<T>(d, wn);
            sm[col * LP + xpad<T>(bufpos<T, N>(N - k))] = mk<T>(s.x - wd.y, s.y + wd.x);
        }
    }
    __syncthreads();
    if constexpr (Plan<T, N>::S > 0) {
        auto lds = [&](int col, int pos) -> C2<T> { return sm[col * LP + xpad<T>(pos)]; };
        auto sts = [&](int col, int pos, C2<T> v) { sm[col * LP + xpad<T>(pos)] = v; };
        fft_inverse<T, N, NCOL, NT, false, true, true>(lds, lds, sts, sts, tw);
        __syncthreads();
    }
    double tmax = 0;
    double acc[7] = {0, 0, 0, 0, 0, 0, 0};
    int bad = 0;
    const int nx = g.nx;
    for (int e = threadIdx.x; e < ROWS * nx; e += NT) {
        const int r = e / nx, i = e % nx;
        const long long row = row0 + r;
        if (row >= nrows) continue;
        const int j = (int)(row % g.ny), k = (int)(row / g.ny);
        const int pos = xpad<T>(i >> 1);
        const C2<T> zx = sm[(0 * ROWS + r) * LP + pos];
        const C2<T> zy = sm[(1 * ROWS + r) * LP + pos];
        const C2<T> zz = sm[(2 * ROWS + r) * LP + pos];
        const bool odd = i & 1;
        const T hdx = (odd ? zx.y : zx.x) * scale;
        const T hdy = (odd ? zy.y : zy.x) * scale;
        const T hdz = (odd ? zz.y : zz.x) * scale;
        cell_update<T>(g, P, io, M, Mn, Hout, hl, row * nx + i, i, j, k, hdx, hdy, hdz, tmax, acc, bad);
    }
    block_finish<NT>(io, ctl, tmax, acc, bad);
}

// 16-byte vector of V = 16/sizeof(T) consecutive cells.
template <class T> struct V16;
template <> struct V16<float> { using type = float4; static constexpr int V = 4; };
template <> struct V16<double> { using type = double2; static constexpr int V = 2; };

template <class T>
__device__ __forceinline__ void vload(const T* p, T* out) {
    using VT = typename V16<T>::type;
    const VT v = __ldg(reinterpret_cast<const VT*>(p));
    if constexpr (V16<T>::V == 4) { out[0] = v.x; out[1] = v.y; out[2] = v.z; out[3] = v.w; }
    else { out[0] = v.x; out[1] = v.y; }
}
template <class T>
__device__ __forceinline__ void vlds(const T* p, T* out) {   // shared-memory 16-byte vector
    using VT = typename V16<T>::type;
    const VT v = *reinterpret_cast<const VT*>(p);
    if constexpr (V16<T>::V == 4) { out[0] = v.x; out[1] = v.y; out[2] = v.z; out[3] = v.w; }
    else { out[0] = v.x; out[1] = v.y; }
}
template <class T>
__device__ __forceinline__ void vstore(T* p, const T* in) {
    using VT = typename V16<T>::type;
    VT v;
    if constexpr (V16<T>::V == 4) { v.x = in[0]; v.y = in[1]; v.z = in[2]; v.w = in[3]; }
    else { v.x = in[0]; v.y = in[1]; }
    *reinterpret_cast<VT*>(p) = v;
}

// Vectorised epilogue over V cells [i0, i0+V) of one row: M, its six
// neighbours and the results move as 16-byte vectors.  Requires nx % V == 0.
// The exchange field of component c needs only component c of the
// neighbours, so the stencil runs one component at a time (register use
// independent of the component count); per cell and component the sum is
// accumulated in the reference order x-, x+, y-, y+, z-, z+ (fields.hpp:33-48),
// with separate round-to-nearest multiplies and adds as the reference build
// (no FMA).  fsm (fused next-step x pass): the new M of the V cells also goes
// to shared memory as (x[2n], x[2n+1]) pairs at component stride fstride.
// The per-vector arithmetic, independent of where M and its neighbours live:
// Acc supplies the loads (m, ym, yp, zm, zp as V-vectors; xl, xr scalars) and
// the stores of H and the new M; nb = {hx0, hx1, hy0, hy1, hz0, hz1} says
// which neighbours exist (Neumann boundaries).
template <class T, bool SUMS, class Acc>
__device__ __forceinline__ void cells_core(const Acc& ac, const LocalParams<T>& P, const StepIO& io,
                                           const bool (&nb)[6], const T (&hd)[3][V16<T>::V], double& tmax,
                                           double* acc, int& bad, C2<T>* fsm, int fstride, int i0) {
    constexpr int V = V16<T>::V;
    constexpr bool sums = SUMS;
    // f64: fused multiply-adds and rsqrt in the epilogue (the f64 passes are
    // FP64-issue-bound; the f32 epilogue measured faster in the strict form).
    // The separate-rounding form stays in cell_update (the bitwise demag-free path).
    constexpr bool FMA = sizeof(T) == 8 && MFD_K5_F64_FMA;
    auto mad = [](T a, T b, T c) -> T {
        if constexpr (FMA) return fma(a, b, c);
        else return add_rn(mul_rn(a, b), c);
    };
    auto msub = [](T a, T b, T c) -> T {   // a*b - c
        if constexpr (FMA) return fma(a, b, -c);
        else return sub_rn(mul_rn(a, b), c);
    };
    const bool hx0 = nb[0], hx1 = nb[1], hy0 = nb[2], hy1 = nb[3], hz0 = nb[4], hz1 = nb[5];
    T m[3][V], H[3][V];
    double elink[V];
#pragma unroll
    for (int q = 0; q < V; ++q) elink[q] = 0;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        ac.m(c, m[c]);
        if (!P.exch) {
#pragma unroll
            for (int q = 0; q < V; ++q) H[c][q] = hd[c][q];
            continue;
        }
        T ym[V], yp[V], zm[V], zp[V];
        if (hz0) ac.zm(c, zm);
        if (hz1) ac.zp(c, zp);
        if (hy0) ac.ym(c, ym);
        if (hy1) ac.yp(c, yp);
        const T xl = hx0 ? ac.xl(c) : T(0);
        const T xr = hx1 ? ac.xr(c) : T(0);
#pragma unroll
        for (int q = 0; q < V; ++q) {
            const T mc = m[c][q];
            const T xm = q > 0 ? m[c][q - 1] : xl, xp = q < V - 1 ? m[c][q + 1] : xr;
            T h = 0;
            if (q > 0 || hx0) h = mad(P.cx, sub_rn(xm, mc), h);
            if (q < V - 1 || hx1) h = mad(P.cx, sub_rn(xp, mc), h);
            if (hy0) h = mad(P.cy, sub_rn(ym[q], mc), h);
            if (hy1) h = mad(P.cy, sub_rn(yp[q], mc), h);
            if (hz0) h = mad(P.cz, sub_rn(zm[q], mc), h);
            if (hz1) h = mad(P.cz, sub_rn(zp[q], mc), h);
            H[c][q] = add_rn(hd[c][q], h);
            if (sums) {   // exchange link energy, links to +x, +y, +z (fields.hpp:141-160)
                if (q < V - 1 || hx1) { const double e = (double)xp - mc; elink[q] += P.wx * e * e; }
                if (hy1) { const double e = (double)yp[q] - mc; elink[q] += P.wy * e * e; }
                if (hz1) { const double e = (double)zp[q] - mc; elink[q] += P.wz * e * e; }
            }
        }
    }
    T mo[3][V];
    bool all = true;
#pragma unroll
    for (int q = 0; q < V; ++q) {
        const T mx = m[0][q], my = m[1][q], mz = m[2][q];
        T Hx = H[0][q], Hy = H[1][q], Hz = H[2][q];
        if (P.anis) {
            const T proj = mul_rn(P.ca, add_rn(add_rn(mul_rn(mx, P.ax), mul_rn(my, P.ay)), mul_rn(mz, P.az)));
            Hx = add_rn(Hx, mul_rn(proj, P.ax));
            Hy = add_rn(Hy, mul_rn(proj, P.ay));
            Hz = add_rn(Hz, mul_rn(proj, P.az));
        }
        if (P.zee) {
            Hx = add_rn(Hx, P.hx);
            Hy = add_rn(Hy, P.hy);
            Hz = add_rn(Hz, P.hz);
        }
        if (io.write_h == 1) { H[0][q] = Hx; H[1][q] = Hy; H[2][q] = Hz; }
        if (sums) {
            acc[0] += (double)mx;
            acc[1] += (double)my;
            acc[2] += (double)mz;
            acc[3] += elink[q];
            const double m0 = (double)mx / P.dMs, m1 = (double)my / P.dMs, m2 = (double)mz / P.dMs;
            const double pp = m0 * P.dax + m1 * P.day + m2 * P.daz;
            acc[4] += 1.0 - pp * pp;
            acc[5] += (double)hd[0][q] * mx + (double)hd[1][q] * my + (double)hd[2][q] * mz;
            acc[6] += P.dhx * mx + P.dhy * my + P.dhz * mz;
        }
        // llgRhs (dynamics.hpp:49-64): b = mu0 H, c = m x b, d = m x c, r = P c + D d
        const T b0 = mul_rn(P.mu0, Hx), b1 = mul_rn(P.mu0, Hy), b2 = mul_rn(P.mu0, Hz);
        const T c0x = msub(my, b2, mul_rn(mz, b1));
        const T c1x = msub(mz, b0, mul_rn(mx, b2));
        const T c2x = msub(mx, b1, mul_rn(my, b0));
        const T d0 = msub(my, c2x, mul_rn(mz, c1x));
        const T d1 = msub(mz, c0x, mul_rn(mx, c2x));
        const T d2 = msub(mx, c1x, mul_rn(my, c0x));
        const T r0 = mad(P.precess, c0x, mul_rn(P.damp, d0));
        const T r1 = mad(P.precess, c1x, mul_rn(P.damp, d1));
        const T r2 = mad(P.precess, c2x, mul_rn(P.damp, d2));
        {   // maxTorqueRate: |rhs|^2 in double (dynamics.hpp:75-82)
            const double v0 = r0, v1 = r1, v2 = r2;
            tmax = fmax(tmax, __dadd_rn(__dadd_rn(__dmul_rn(v0, v0), __dmul_rn(v1, v1)), __dmul_rn(v2, v2)));
        }
        // eulerUpdate (dynamics.hpp:93-121)
        T e0 = mad(P.dt, r0, mx);
        T e1 = mad(P.dt, r1, my);
        T e2 = mad(P.dt, r2, mz);
        if (io.renorm) {
            const T n2 = add_rn(add_rn(mul_rn(e0, e0), mul_rn(e1, e1)), mul_rn(e2, e2));
            if (!(n2 > T(0)) || !isfinite((double)n2)) {
                all = false;
            } else {
                const T f = FMA ? mul_rn(P.Ms, rsqrt(n2)) : P.Ms / sqrt(n2);
                e0 = mul_rn(f, e0); e1 = mul_rn(f, e1); e2 = mul_rn(f, e2);
            }
        } else if (!isfinite((double)add_rn(add_rn(e0, e1), e2))) {
            all = false;
        }
        mo[0][q] = e0; mo[1][q] = e1; mo[2][q] = e2;
    }
    if (io.write_h) {
#pragma unroll
        for (int c = 0; c < 3; ++c) ac.store_h(c, io.write_h == 1 ? H[c] : hd[c]);
    }
    if (io.update) {
        if (!all) bad = 1;
#pragma unroll
        for (int c = 0; c < 3; ++c) ac.store_m(c, mo[c]);
        if (fsm) {
#pragma unroll
            for (int c = 0; c < 3; ++c)
#pragma unroll
                for (int q = 0; q < V; q += 2) fsm[c * fstride + xpad<T>((i0 + q) >> 1)] = mk<T>(mo[c][q], mo[c][q + 1]);
        }
    }
}

// Global-memory accessor of cells_core: M / Mn / Hout are SoA lattices, the
// z neighbours of a slab's edge planes come from the halo planes.
template <class T>
struct GAcc {
    static constexpr int V = V16<T>::V;
    const T* p;              // M + c0 (component 0)
    T* mn;                   // Mn + c0
    T* h;                    // Hout + c0
    long long n, sy, sz;
    const T* zlo;            // component-0 address of the z- neighbour vector
    const T* zhi;
    long long zlo_cs, zhi_cs;   // their component strides
    __device__ __forceinline__ void m(int c, T* o) const { vload<T>(p + c * n, o); }
    __device__ __forceinline__ void ym(int c, T* o) const { vload<T>(p + c * n - sy, o); }
    __device__ __forceinline__ void yp(int c, T* o) const { vload<T>(p + c * n + sy, o); }
    __device__ __forceinline__ void zm(int c, T* o) const { vload<T>(zlo + c * zlo_cs, o); }
    __device__ __forceinline__ void zp(int c, T* o) const { vload<T>(zhi + c * zhi_cs, o); }
    __device__ __forceinline__ T xl(int c) const { return __ldg(p + c * n - 1); }
    __device__ __forceinline__ T xr(int c) const { return __ldg(p + c * n + V); }
    __device__ __forceinline__ void store_h(int c, const T* v) const { vstore<T>(h + c * n, v); }
    __device__ __forceinline__ void store_m(int c, const T* v) const { vstore<T>(mn + c * n, v); }
};

template <class T, bool SUMS>
__device__ __forceinline__ void cells_vec(const Geo& g, const LocalParams<T>& P, const StepIO& io,
                                          const T* __restrict__ M, T* __restrict__ Mn, T* __restrict__ Hout,
                                          const Halo<T>& hl, long long c0, int i0, int j, int k,
                                          const T (&hd)[3][V16<T>::V], double& tmax, double* acc, int& bad,
                                          C2<T>* fsm = nullptr, int fstride = 0) {
    constexpr int V = V16<T>::V;
    const long long n = g.ncell, sy = g.nx, sz = (long long)g.nx * g.ny;
    const int kg = g.k0 + k;                         // global plane: Neumann boundaries are global
    const long long inplane = c0 - (long long)k * sz;  // j*nx + i0
    const bool nb[6] = {i0 > 0, i0 + V < g.nx, j > 0, j < g.ny - 1, kg > 0, kg < g.nzg - 1};
    GAcc<T> ac;
    ac.p = M + c0;
    ac.mn = Mn + c0;
    ac.h = Hout + c0;
    ac.n = n;
    ac.sy = sy;
    ac.sz = sz;
    ac.zlo = k > 0 ? M + c0 - sz : hl.lo + inplane;            // slab edge: halo plane
    ac.zhi = k < g.nz - 1 ? M + c0 + sz : hl.hi + inplane;
    ac.zlo_cs = k > 0 ? n : sz;
    ac.zhi_cs = k < g.nz - 1 ? n : sz;
    cells_core<T, SUMS>(ac, P, io, nb, hd, tmax, acc, bad, fsm, fstride, i0);
}

// FWD: also run the NEXT step's x pass (K1) on the new M of this CTA's rows
// while they are in shared memory, writing A in place of the spectrum this
// CTA consumed (only its own rows: no cross-CTA hazard).  Saves K1's M read
// and launch on every step but the first of a graph chunk.
template <class T, int N, bool SUMS, int RS = 0, bool FWD = false, bool MULTI = false>
__device__ __forceinline__ void k5_body(const Geo& g, C2<T>* __restrict__ A, const T* __restrict__ M,
                                        T* __restrict__ Mn, T* __restrict__ Hout, const C2<T>* __restrict__ tw,
                                        T scale, const LocalParams<T>& P, const StepIO& io, const Halo<T>& hl,
                                        long long bx, unsigned char* smem_raw, double& tmax, double* acc, int& bad,
                                        const Ctl* hctl = nullptr, HaltRaw hold = {}) {
    constexpr bool fwd = FWD;
    using CF = LCfg<T, N, RS>;
    constexpr int ROWS = CF::ROWS, NT = CF::NT, LP = xpitch<T, N>(), NCOL = 3 * ROWS;
    constexpr int V = V16<T>::V;
    C2<T>* sm = reinterpret_cast<C2<T>*>(smem_raw);
    const long long nrows = (long long)g.ny * g.nz;
    const long long row0 = bx * ROWS;
    if ((g.pfm & 6) && threadIdx.x < 3) {
        // this CTA's M rows with their y / z neighbour rows (read by the
        // epilogue, after the inverse FFT) ...
        const int c = threadIdx.x;
        if (g.pfm & 2) {
            const T* Mc = M + c * g.ncell;
            const long long nx = g.nx, ny = g.ny;
            const long long ra = row0 - 1 > 0 ? row0 - 1 : 0, rb = row0 + ROWS + 1 < nrows ? row0 + ROWS + 1 : nrows;
            l2_prefetch(Mc + ra * nx, (rb - ra) * nx * (long long)sizeof(T));
            const long long re = row0 + ROWS < nrows ? row0 + ROWS : nrows;
            if (row0 >= ny) l2_prefetch(Mc + (row0 - ny) * nx, (re - row0) * nx * (long long)sizeof(T));
            if (re + ny <= nrows) l2_prefetch(Mc + (row0 + ny) * nx, (re - row0) * nx * (long long)sizeof(T));
        }
        // ... and the spectrum rows of the CTA one resident wave later
        const long long r1 = row0 + (long long)g.pf5 * ROWS;
        if ((g.pfm & 4) && r1 < nrows) {
            const long long nr = nrows - r1 < ROWS ? nrows - r1 : ROWS;
            l2_prefetch(A + ((long long)c * nrows + r1) * g.Hp, nr * g.Hp * (long long)sizeof(C2<T>));
        }
    }
    // C2R pre-process over pairs (k, N-k): item e -> (k = e % (N/2), column
    // = e / (N/2)); the k = 0 item also carries the self-paired k = N/2.  All
    // HBM loads of the thread are issued before any use (compile-time trip
    // count) so the latency is paid once (measured faster than staging the
    // rows in shared memory by cp.async first: 0.384 vs 0.395 ms at C4 f32).
    // Z is written in natural order; the first inverse stage reads natural order.
    constexpr int HP = N / 2 > 0 ? N / 2 : 1;
    constexpr int ITEMS = NCOL * HP;
    constexpr int IT = (ITEMS + NT - 1) / NT;
    auto pre = [&](C2<T>* scol, int k, C2<T> a, C2<T> b) {
        const C2<T> w = __ldg(tw_dense<T, 2 * N>(tw) + k);
        {
            const C2<T> s = cadd<T>(a, cconj<T>(b)), d = csub<T>(a, cconj<T>(b));
            const C2<T> wd = cmulc<T>(d, w);
            scol[xpad<T>(k & (N - 1))] = mk<T>(s.x - wd.y, s.y + wd.x);
        }
        if (N - k != k && N - k < N) {
            const C2<T> s = cadd<T>(b, cconj<T>(a)), d = csub<T>(b, cconj<T>(a));
            const C2<T> wn = mk<T>(-w.x, w.y);
            const C2<T> wd = cmulc<T>(d, wn);
            scol[xpad<T>(N - k)] = mk<T>(s.x - wd.y, s.y + wd.x);
        }
    };
    {
        C2<T> pa[IT], pb[IT], pc[IT];
#pragma unroll
        for (int it = 0; it < IT; ++it) {
            const int e = threadIdx.x + it * NT;
            const int col = e / HP, k = N / 2 > 0 ? e % HP : 0;
            const long long row = row0 + col % ROWS;
            pa[it] = pb[it] = pc[it] = mk<T>(0, 0);
            if (e < ITEMS && row < nrows) {
                const C2<T>* src = A + ((long long)(col / ROWS) * nrows + row) * g.Hp;
                pa[it] = *abin<MULTI>(g, src, k);
                pb[it] = *abin<MULTI>(g, src, N - k);
                if (k == 0 && N > 1) pc[it] = *abin<MULTI>(g, src, N / 2);
            }
        }
#pragma unroll
        for (int it = 0; it < IT; ++it) {
            const int e = threadIdx.x + it * NT;
            if (ITEMS % NT != 0 && e >= ITEMS) continue;
            const int col = e / HP, k = N / 2 > 0 ? e % HP : 0;
            pre(sm + col * LP, k, pa[it], pb[it]);
            if (k == 0 && N > 1) pre(sm + col * LP, N / 2, pc[it], pc[it]);
        }
    }
    // hold: the caller's deferred halt-flag read (nothing global is written before this barrier)
    if (__syncthreads_or(hctl ? halted_test(*hctl, hold) : 0)) {
        bad = -1;
        return;
    }
    if constexpr (Plan<T, N>::S > 0) {
        auto lds = [&](int col, int pos) -> C2<T> { return sm[col * LP + xpad<T>(pos)]; };
        auto sts = [&](int col, int pos, C2<T> v) { sm[col * LP + xpad<T>(pos)] = v; };
        fft_inverse<T, N, NCOL, NT, false, true, true, true, true>(lds, lds, sts, sts, tw);
        __syncthreads();
    }
    const int nx = g.nx, nvec = nx / V;
    constexpr int EIT = (ROWS * (N / V) + NT - 1) / NT;   // nx <= N
#pragma unroll
    for (int it = 0; it < EIT; ++it) {
        const int e = threadIdx.x + it * NT;
        if (e >= ROWS * nvec) break;
        const int r = e / nvec, i0 = (e % nvec) * V;
        const long long row = row0 + r;
        if (row >= nrows) continue;
        const int j = (int)(row % g.ny), k = (int)(row / g.ny);
        T hd[3][V];
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
            for (int q = 0; q < V; q += 2) {
                const C2<T> z = sm[(c * ROWS + r) * LP + xpad<T>((i0 + q) >> 1)];
                hd[c][q] = z.x * scale;
                hd[c][q + 1] = z.y * scale;
            }
        cells_vec<T, SUMS>(g, P, io, M, Mn, Hout, hl, row * nx + i0, i0, j, k, hd, tmax, acc, bad,
                           fwd ? sm + r * LP : nullptr, ROWS * LP);
    }
    if constexpr (FWD && N >= 2) {
        // next step's K1 on the rows in shared memory (pairs beyond nx/2 are padding)
        __syncthreads();
        const int nxh = nx / 2;
        auto ldf = [&](int col, int pos) -> C2<T> { return pos < nxh ? sm[col * LP + xpad<T>(pos)] : mk<T>(0, 0); };
        auto lds = [&](int col, int pos) -> C2<T> { return sm[col * LP + xpad<T>(pos)]; };
        auto sts = [&](int col, int pos, C2<T> v) { sm[col * LP + xpad<T>(pos)] = v; };
        fft_forward<T, N, NCOL, NT, false, true, true, true, true>(ldf, lds, sts, sts, tw);
        __syncthreads();
        constexpr int HPF = N / 2;
        for (int e = threadIdx.x; e < NCOL * HPF; e += NT) {
            const int col = e / HPF, kk = e % HPF;
            const int comp = col / ROWS, r = col % ROWS;
            if (row0 + r >= nrows) continue;
            C2<T>* dst = A + ((long long)comp * nrows + row0 + r) * g.Hp;
            r2c_post<T, N>(sm + col * LP, dst, kk, __ldg(tw_dense<T, 2 * N>(tw) + kk));
            if (kk == 0) r2c_post<T, N>(sm + col * LP, dst, N / 2, __ldg(tw_dense<T, 2 * N>(tw) + N / 2));
        }
    }
}

template <class T, int N, bool SUMS, int RS = 0, bool FWD = false, bool MULTI = false>
__global__ void __launch_bounds__(LCfg<T, N, RS>::NT, LCfg<T, N, RS>::MINB)
k_c2r_x_llg_v(Geo g, C2<T>* __restrict__ A, const T* __restrict__ M, T* __restrict__ Mn,
              T* __restrict__ Hout, const C2<T>* __restrict__ tw, T scale, LocalParams<T> P, StepIO io, Ctl ctl,
              Halo<T> hl) {
    // small grids (latency-bound): the halt flag loads alongside the spectrum rows
    // and is acted on at k5_body's first barrier, before any global write
    constexpr bool DEFER = RS > 0 && MFD_K5_DEFER_HALT;
    if (!DEFER && halted(ctl)) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double tmax = 0;
    double acc[7] = {0, 0, 0, 0, 0, 0, 0};
    int bad = 0;
    const HaltRaw hr = DEFER ? halted_load(ctl) : HaltRaw{};
    k5_body<T, N, SUMS, RS, FWD, MULTI>(g, A, M, Mn, Hout, tw, scale, P, io, hl, blockIdx.x, smem_raw, tmax, acc, bad,
                                        DEFER ? &ctl : nullptr, hr);
    if (DEFER && bad < 0) return;
    block_finish<LCfg<T, N, RS>::NT>(io, ctl, tmax, acc, bad);
}

// Demag-free step (terms.demag = false): H_eff from local terms only.
template <class T>
__global__ void __launch_bounds__(256)
k_local_llg(Geo g, const T* __restrict__ M, T* __restrict__ Mn, T* __restrict__ Hout, LocalParams<T> P,
            StepIO io, Ctl ctl, Halo<T> hl) {
    if (halted(ctl)) return;
    double tmax = 0;
    double acc[7] = {0, 0, 0, 0, 0, 0, 0};
    int bad = 0;
    const long long c = (long long)blockIdx.x * 256 + threadIdx.x;
    if (c < g.ncell) {
        const int i = (int)(c % g.nx);
        const int j = (int)((c / g.nx) % g.ny);
        const int k = (int)(c / ((long long)g.nx * g.ny));
        cell_update<T>(g, P, io, M, Mn, Hout, hl, c, i, j, k, T(0), T(0), T(0), tmax, acc, bad);
    }
    block_finish<256>(io, ctl, tmax, acc, bad);
}

} // namespace mfd
