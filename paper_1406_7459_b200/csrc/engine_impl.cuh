// Engine<T> method definitions; included once per precision by engine_f32.cu /
// engine_f64.cu (explicit instantiation keeps the two builds parallel).
#pragma once
#include <algorithm>
#include <cstdio>

#include "engine.cuh"

namespace mfd {

template <class T>
__global__ void k_ybuf(int Py, int Hy, int* out) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= Hy) return;
    // dispatch on Py inside the kernel (setup only)
    int r = 0;
    switch (Py) {
#define YB(L) case L: r = bufpos<T, L>(v); break;
        YB(2) YB(4) YB(8) YB(16) YB(32) YB(64) YB(128) YB(256) YB(512) YB(1024) YB(2048)
#undef YB
        default: r = -1;
    }
    out[v] = r;
}

template <class T>
__global__ void k_fill3(T* m, long long n, T x, T y, T z) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    m[i] = x;
    m[i + n] = y;
    m[i + 2 * n] = z;
}

// makeVortexState (state.hpp:83-108) per cell, fp64 in the reference's
// operation order with explicit round-to-nearest ops (no contraction), so the
// cast to T is bitwise the host result.  Global plane index k0 + k.
template <class T>
__global__ void k_vortex(T* m, int nx, int ny, int nz, int nzg, int k0, double dx, double dy, double dz, double ax,
                         double ay, double az, double Ms) {
    const long long n = (long long)nx * ny * nz;
    const long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n) return;
    const int i = (int)(c % nx), j = (int)((c / nx) % ny), k = k0 + (int)(c / ((long long)nx * ny));
    const bool along_x = ax != 0, along_y = ay != 0;
    const double d1 = along_x ? dy : dx, d2 = (along_x || along_y) ? dz : dy;
    const double core = fmin(d1, d2);
    const double cx = __dmul_rn(0.5, (double)(nx - 1)), cy = __dmul_rn(0.5, (double)(ny - 1)),
                 cz = __dmul_rn(0.5, (double)(nzg - 1));
    const double rx = __dmul_rn(__dsub_rn((double)i, cx), dx), ry = __dmul_rn(__dsub_rn((double)j, cy), dy),
                 rz = __dmul_rn(__dsub_rn((double)k, cz), dz);
    const double ra = __dadd_rn(__dadd_rn(__dmul_rn(rx, ax), __dmul_rn(ry, ay)), __dmul_rn(rz, az));
    const double px = __dsub_rn(rx, __dmul_rn(ra, ax)), py = __dsub_rn(ry, __dmul_rn(ra, ay)),
                 pz = __dsub_rn(rz, __dmul_rn(ra, az));
    const double pn = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(px, px), __dmul_rn(py, py)), __dmul_rn(pz, pz)));
    double mx = ax, my = ay, mz = az;
    if (!(pn < core)) {
        const double qx = __dsub_rn(__dmul_rn(ay, pz), __dmul_rn(az, py));
        const double qy = __dsub_rn(__dmul_rn(az, px), __dmul_rn(ax, pz));
        const double qz = __dsub_rn(__dmul_rn(ax, py), __dmul_rn(ay, px));
        const double qn = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(qx, qx), __dmul_rn(qy, qy)), __dmul_rn(qz, qz)));
        mx = __ddiv_rn(qx, qn);
        my = __ddiv_rn(qy, qn);
        mz = __ddiv_rn(qz, qn);
    }
    m[c] = static_cast<T>(__dmul_rn(Ms, mx));
    m[c + n] = static_cast<T>(__dmul_rn(Ms, my));
    m[c + 2 * n] = static_cast<T>(__dmul_rn(Ms, mz));
}

// Largest x length with the 1-2-row K1/K5 variants for few-row grids (SP4
// 128x32x1: N = 128; SP4 refined 512x128x4: N = 512, 512 rows).
#ifndef MFD_SMALL_X_MAX
#define MFD_SMALL_X_MAX 512
#endif
constexpr int kSmallXMax = MFD_SMALL_X_MAX;

template <class T>
static void set_smem(const void* fn, int bytes, bool carve = true) {
    if (bytes > 48 * 1024)
        ck(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes), "smem attr");
    // Forcing the full shared-memory carveout was measured slower on B200
    // (512x512x64 f32: K2 0.31 -> 0.39 ms, K3 0.69 -> 0.73 ms): the passes'
    // strided column loads profit from L1.  Kept switchable.
    constexpr bool kCarveout = false;
    if (kCarveout && carve && bytes > 0)
        ck(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100), "carveout attr");
}

template <class T>
Engine<T>::Engine(const mfd_grid& g, const mfd_material& m, const mfd_terms& te, const mfd_stepper& st,
                  int device, Slab slab, Transport* tr)
    : grid_(g), mat_(m), terms_(te), st_(st), device_(device), slab_(slab), tr_(tr) {
    // The engine owns tr and every buffer from the first statement on: a
    // failure part-way releases them (the destructor does not run then).
    try {
        init();
    } catch (...) {
        release();
        throw;
    }
}

template <class T>
void Engine<T>::init() {
    const mfd_grid& g = grid_;
    const mfd_terms& te = terms_;
    const mfd_material& m = mat_;
    const mfd_stepper& st = st_;
    precision = sizeof(T) == 4 ? 32 : 64;
    if (slab_.world <= 1) slab_ = Slab::of(g.nz, 0, 1);
    if (slab_.world > 1 && (g.nz % slab_.world != 0))
        throw Error(MFD_EINVAL, "magfd-b200: nz must be divisible by the number of GPUs (z-slab decomposition)");
    ck(cudaSetDevice(device_), "cudaSetDevice");
    ck(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "stream");
    const int Px = padded_size(g.nx);
    Py_ = padded_size(g.ny);
    Pz_ = padded_size(g.nz);
    if (Px / 2 > kMaxL || Py_ > kMaxL || Pz_ > kMaxL)
        throw Error(MFD_EINVAL, "magfd-b200: padded FFT size exceeds the engine limit (nx <= 2048, ny,nz <= 1024)");
    const int G = slab_.world, nzl = slab_.nzl;
    geo_.nx = g.nx; geo_.ny = g.ny; geo_.nz = nzl;
    geo_.Px = Px; geo_.Py = Py_; geo_.Pz = Pz_;
    geo_.N = Px / 2;
    geo_.Hx = geo_.N + 1;
    // A row pitch: all bins on one GPU; the x-bin block width when sharded
    geo_.ncell = (long long)g.nx * g.ny * nzl;
    geo_.nzg = g.nz;
    geo_.k0 = slab_.k0;
    geo_.G = G;
    geo_.ublk = slab_.rank;
    // x-bin blocks: multiples of 16 so no y/z tile straddles two ranks
    geo_.Wb = G == 1 ? (geo_.Hx + 15) / 16 * 16 : ((geo_.Hx + G - 1) / G + 15) / 16 * 16;
    geo_.Hp = geo_.Wb;
    geo_.binv = (unsigned)(((1u << 24) + geo_.Wb - 1) / geo_.Wb);
    geo_.Hv = std::max(0, std::min(geo_.Wb, geo_.Hx - slab_.rank * geo_.Wb));
    geo_.SA = 3LL * nzl * g.ny * geo_.Hp;
    geo_.S_k = (long long)Py_ * geo_.Wb;
    geo_.S_c = (long long)g.nz * geo_.S_k;   // B holds all nzg planes of this rank's x-bin block
    ncell = geo_.ncell;
    Hy_ = Py_ / 2 + 1;
    Hz_ = Pz_ / 2 + 1;
    scale_ = static_cast<T>(1.0 / ((double)Px * Py_ * Pz_));   // plan.normalization() (fft.hpp:261)

    // Local-term coefficients, double then cast to T as the reference does.
    const double Ms = m.Ms;
    const double base = 2.0 * m.A / (kMu0 * Ms * Ms);
    lp_.cx = static_cast<T>(base / (g.dx * g.dx));   // fields.hpp:25-27
    lp_.cy = static_cast<T>(base / (g.dy * g.dy));
    lp_.cz = static_cast<T>(base / (g.dz * g.dz));
    lp_.exch = te.exchange && m.A > 0;                // fields.hpp:239
    lp_.anis = te.anisotropy && m.Ku != 0;            // fields.hpp:241
    lp_.ca = static_cast<T>(2.0 * m.Ku / (kMu0 * Ms * Ms));
    lp_.ax = static_cast<T>(m.easy_axis[0]);
    lp_.ay = static_cast<T>(m.easy_axis[1]);
    lp_.az = static_cast<T>(m.easy_axis[2]);
    lp_.hx = static_cast<T>(te.h_ext[0]);
    lp_.hy = static_cast<T>(te.h_ext[1]);
    lp_.hz = static_cast<T>(te.h_ext[2]);
    lp_.zee = te.zeeman && (lp_.hx != 0 || lp_.hy != 0 || lp_.hz != 0);   // fields.hpp:243-245
    const double a2 = 1.0 + m.alpha * m.alpha;
    lp_.precess = static_cast<T>(-m.gamma / a2);                            // dynamics.hpp:54-57
    lp_.damp = static_cast<T>(-m.alpha * m.gamma / (a2 * Ms));
    lp_.mu0 = static_cast<T>(kMu0);
    lp_.dt = static_cast<T>(st.dt);
    lp_.Ms = static_cast<T>(Ms);
    lp_.dA = m.A; lp_.dMs = Ms; lp_.dKu = m.Ku; lp_.dV = g.dx * g.dy * g.dz;
    lp_.dax = m.easy_axis[0]; lp_.day = m.easy_axis[1]; lp_.daz = m.easy_axis[2];
    lp_.dhx = te.h_ext[0]; lp_.dhy = te.h_ext[1]; lp_.dhz = te.h_ext[2];
    lp_.wx = 1.0 / (g.dx * g.dx); lp_.wy = 1.0 / (g.dy * g.dy); lp_.wz = 1.0 / (g.dz * g.dz);

    const long long n = geo_.ncell;
    guards_ = getenv("MFD_GUARD") && atoi(getenv("MFD_GUARD")) != 0;
    auto alloc = [&](auto** p, size_t bytes) { *p = reinterpret_cast<std::remove_reference_t<decltype(*p)>>(dalloc(bytes)); };
    alloc(&M_[0], 3 * n * sizeof(T));
    alloc(&M_[1], 3 * n * sizeof(T));
    alloc(&H_, 3 * n * sizeof(T));
    alloc(&err_, sizeof(int));
    alloc(&torque_, kMaxChunk * sizeof(unsigned long long));
    alloc(&sums_, kMaxChunk * 8 * sizeof(double));
    alloc(&ticket_, sizeof(unsigned int));
    ck(cudaMallocHost((void**)&h_perr_, kMaxPending * sizeof(int)), "host alloc");
    ck(cudaMemset(err_, 0, sizeof(int)), "memset");
    ck(cudaMemset(ticket_, 0, sizeof(unsigned int)), "memset");
    ck(cudaMemset(M_[0], 0, 3 * n * sizeof(T)), "memset");
    ck(cudaMallocHost((void**)&h_torque_, kMaxChunk * sizeof(unsigned long long)), "host alloc");
    ck(cudaMallocHost((void**)&h_sums_, kMaxChunk * 8 * sizeof(double)), "host alloc");
    ck(cudaMallocHost((void**)&h_err_, sizeof(int)), "host alloc");

    if (G > 1) alloc(&halo_, 2 * 3 * (long long)g.nx * g.ny * sizeof(T));
    if (G > 1 && tr_) {   // one process per GPU: transposes on a second stream (enqueue)
        ck(cudaStreamCreateWithFlags(&cstream_, cudaStreamNonBlocking), "stream");
        for (auto& e : xev_) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
        tr_->reserve(terms_.demag ? (size_t)geo_.nz * g.ny * geo_.Hp * sizeof(C2<T>) : 0,
                     (size_t)g.nx * g.ny * sizeof(T));
    }
    if (terms_.demag) {
        const long long nrows = (long long)g.ny * nzl;
        (void)nrows;
        alloc(&A_, (size_t)G * geo_.SA * sizeof(C2<T>));          // send blocks (G = 1: the A spectrum)
        if (G > 1) alloc(&Ar_, (size_t)G * geo_.SA * sizeof(C2<T>));   // receive blocks
        else Ar_ = A_;
        alloc(&B_, (size_t)3 * geo_.S_c * sizeof(C2<T>));
        alloc(&Kt_, 6 * (long long)Hy_ * Hz_ * geo_.Wb * sizeof(T));
        alloc(&ybuf_, Py_ * sizeof(int));   // buffer row of every y frequency
        // twiddles exp(-2 pi i k / TWN), long double on the host, cast to T (fft.hpp:70-74)
        std::vector<C2<T>> tw(TWN);
        for (int k = 0; k < TWN; ++k) {
            const long double a = -2.0L * (long double)kPi * k / TWN;
            tw[k].x = static_cast<T>(cosl(a));
            tw[k].y = static_cast<T>(sinl(a));
        }
        tw.resize(TW_ALLOC);
        for (int LT = 1; LT <= TWN; LT *= 2)   // dense per-length copies (fft_engine.cuh)
            for (int e = 0; e < LT; ++e) tw[TWN + LT + e] = tw[(long long)e * (TWN / LT)];
        alloc(&tw_, TW_ALLOC * sizeof(C2<T>));
        ck(cudaMemcpy(tw_, tw.data(), TW_ALLOC * sizeof(C2<T>), cudaMemcpyHostToDevice), "tw upload");
        k_ybuf<T><<<(Py_ + 127) / 128, 128, 0, stream_>>>(Py_, Py_, ybuf_);
        ck(cudaGetLastError(), "k_ybuf");
        // shared-memory opt-in for the instantiations this grid uses
        with_pow2(geo_.N, [&]<int L>() {
            set_smem<T>((const void*)k_r2c_x<T, L>, XCfg<T, L>::SMEM);
            if (G > 1) set_smem<T>((const void*)k_r2c_x<T, L, 0, true>, XCfg<T, L>::SMEM);
            set_smem<T>((const void*)k_c2r_x_llg<T, L>, LCfg<T, L>::SMEM, false);
            set_smem<T>((const void*)k_c2r_x_llg_v<T, L, true>, k5_smem<T, L, 0, false>(), false);
            set_smem<T>((const void*)k_c2r_x_llg_v<T, L, false>, k5_smem<T, L, 0, false>(), false);
            set_smem<T>((const void*)k_c2r_x_llg_v<T, L, true, 0, true>, k5_smem<T, L, 0, true>(), false);
            set_smem<T>((const void*)k_c2r_x_llg_v<T, L, false, 0, true>, k5_smem<T, L, 0, true>(), false);
            if (G > 1) {
                set_smem<T>((const void*)k_c2r_x_llg<T, L, true>, LCfg<T, L>::SMEM, false);
                set_smem<T>((const void*)k_c2r_x_llg_v<T, L, true, 0, false, true>, k5_smem<T, L, 0, false>(), false);
                set_smem<T>((const void*)k_c2r_x_llg_v<T, L, false, 0, false, true>, k5_smem<T, L, 0, false>(), false);
            }
            k5_blocks_ = (nrows + LCfg<T, L>::ROWS - 1) / LCfg<T, L>::ROWS;
            // small grids (e.g. SP4, 32 rows): 1-2 rows per CTA so the x passes use the SMs
            int nsm = 148;
            cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device_);
            small_x_ = L >= 2 && L <= kSmallXMax && k5_blocks_ < 2 * nsm && g.nx % V16<T>::V == 0;
            if (const char* e = getenv("MFD_SMALL_X"))   // A/B switch: 0 off, 1 on where the variants exist
                small_x_ = L >= 2 && L <= kSmallXMax && g.nx % V16<T>::V == 0 && atoi(e) != 0;
            if (small_x_) k5_blocks_ = nrows;
            // L2 prefetch distances: one resident wave of CTAs
            int per1 = 0, per5 = 0;
            ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per1, k_r2c_x<T, L>, XCfg<T, L>::NT,
                                                             XCfg<T, L>::SMEM), "occupancy");
            ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per5, k_c2r_x_llg_v<T, L, false>, LCfg<T, L>::NT,
                                                             k5_smem<T, L, 0, false>()), "occupancy");
            geo_.pf1 = per1 * nsm;
            geo_.pf5 = per5 * nsm;
            geo_.pfm = small_x_ ? 0 : kL2PrefetchMask;
            if (const char* e = getenv("MFD_PF_MASK")) geo_.pfm = atoi(e);   // tuning override
        });
        with_pow2(Py_, [&]<int L>() {
            set_smem<T>((const void*)k_fft_y_fwd<T, L, true>, YCfg<T, L>::SMEM);
            set_smem<T>((const void*)k_fft_y_inv<T, L, true>, YCfg<T, L>::SMEM);
            set_smem<T>((const void*)k_fft_y_fwd<T, L, false>, YCfg<T, L>::SMEM);
            set_smem<T>((const void*)k_fft_y_inv<T, L, false>, YCfg<T, L>::SMEM);
        });
        with_pow2(Pz_, [&]<int L>() {
            if constexpr (z_variant<T, L>() == 2) {
                set_smem<T>((const void*)k_fft_z_conv2<T, L, true>, Z2Cfg<T, L>::SMEM);
                set_smem<T>((const void*)k_fft_z_conv2<T, L, false>, Z2Cfg<T, L>::SMEM);
                set_smem<T>((const void*)k_fft_z_conv2<T, L, true, true>, Z2Cfg<T, L, true>::SMEM);
                set_smem<T>((const void*)k_fft_z_conv2<T, L, false, true>, Z2Cfg<T, L, true>::SMEM);
            }
            else if constexpr (z_variant<T, L>() == 0) set_smem<T>((const void*)k_fft_z_conv<T, L>, ZCfg<T, L>::SMEM);
        });
        // tensor octant (K0a) and spectra (K0b) of this rank's x-bin block
        build_tensor(nullptr);
    } else {
        k5_blocks_ = (n + 255) / 256;
    }
    if (kYZSmall && terms_.demag && slab_.world == 1)
        with_yz([&]<int LY, int LZ>() {
            yz_small_ = true;
            set_smem<T>((const void*)k_fft_yz_small<T, LY, LZ>, YZCfg<T, LY, LZ>::SMEM);
        });
    if (const char* e = getenv("MFD_YZ_SMALL")) yz_small_ = yz_small_ && atoi(e) != 0;   // A/B switch
    if (kK2Tma && terms_.demag && !yz_small_ && (g.ny <= 256 || g.ny % 256 == 0)) {
        with_pow2(Py_, [&]<int L>() {
            if constexpr (YTCfg<T, L>::OK) {
                const int cs = (int)sizeof(C2<T>);
                k2_box_ = std::min(256, g.ny);
                if (make_tmap_2d(&tmA_, Ar_, (unsigned long long)geo_.Hp * cs / 8,
                                 (unsigned long long)geo_.G * 3 * geo_.nz * geo_.ny, (unsigned long long)geo_.Hp * cs,
                                 (unsigned)(YTCfg<T, L>::W * cs / 8), (unsigned)k2_box_)) {
                    set_smem<T>((const void*)k_fft_y_fwd_tma<T, L, true>, YTCfg<T, L>::SMEM);
                    set_smem<T>((const void*)k_fft_y_fwd_tma<T, L, false>, YTCfg<T, L>::SMEM);
                    int per = 0, nsm = 148;
                    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device_);
                    ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_fft_y_fwd_tma<T, L, true>,
                                                                     YTCfg<T, L>::NT, YTCfg<T, L>::SMEM),
                       "occupancy");
                    const long long tiles = 3LL * geo_.nzg * ((geo_.Hv + YTCfg<T, L>::W - 1) / YTCfg<T, L>::W);
                    k2_grid_ = (int)std::min<long long>(tiles, (long long)std::max(1, per) * nsm);
                    k2_tma_ = per > 0;
                }
            }
        });
    }
    if (const char* e = getenv("MFD_K2_TMA")) k2_tma_ = k2_tma_ && atoi(e) != 0;   // A/B switch
    if (kK4Tma && terms_.demag && !yz_small_) {
        with_pow2(Py_, [&]<int L>() {
            if constexpr (YICfg<T, L>::OK) {
                using CF = YICfg<T, L>;
                const int cs = (int)sizeof(C2<T>);
                if (make_tmap_2d(&tmB_, B_, (unsigned long long)geo_.Wb * cs / 8,
                                 3ULL * geo_.nzg * Py_,
                                 (unsigned long long)geo_.Wb * cs, (unsigned)(CF::W * cs / 8), (unsigned)CF::BOX)) {
                    set_smem<T>((const void*)k_fft_y_inv_tma<T, L, true>, CF::SMEM);
                    set_smem<T>((const void*)k_fft_y_inv_tma<T, L, false>, CF::SMEM);
                    int per = 0, nsm = 148;
                    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device_);
                    ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_fft_y_inv_tma<T, L, true>, CF::NT,
                                                                     CF::SMEM),
                       "occupancy");
                    const long long tiles = 3LL * geo_.nzg * ((geo_.Hv + CF::W - 1) / CF::W);
                    k4_grid_ = (int)std::min<long long>(tiles, (long long)std::max(1, per) * nsm);
                    k4_tma_ = per > 0;
                }
            }
        });
    }
    if (const char* e = getenv("MFD_K4_TMA")) k4_tma_ = k4_tma_ && atoi(e) != 0;   // A/B switch
    // Measured on B200 (f32): fusing pays on small and mid grids, where K1 is a
    // short latency-bound launch (SP4 0.023 -> 0.015 ms, 512x128x4 -8 %, 128^3 -6 %),
    // and costs +1-3 % on the large films (K5's register budget then spills)
    fuse_k1_ = kFuseK1 && G == 1 && terms_.demag && geo_.N >= 2 && g.nx % V16<T>::V == 0 && geo_.ncell <= kFuseK1MaxCells;
    if (const char* e = getenv("MFD_FUSE_K1"))   // A/B switch: 0 off, 2 on regardless of the grid size
        fuse_k1_ = atoi(e) == 2 ? (kFuseK1 && G == 1 && terms_.demag && geo_.N >= 2 && g.nx % V16<T>::V == 0)
                                : fuse_k1_ && atoi(e) != 0;
    // block_finish partials: one slot per CTA of a K5 launch
    alloc(&partials_, (size_t)k5_blocks_ * 8 * sizeof(double));
    // Measured (single-row vs pair): f32 C4 0.609 -> 0.583 ms, C3 -12 %, C5 -14 %; f64 C4 1.18 -> 1.30 ms
    k3_srow_ = kK3SingleRow && sizeof(T) == 4;
    if (const char* e = getenv("MFD_K3_SROW")) k3_srow_ = atoi(e) != 0;   // A/B switch
    if (getenv("MFD_VERBOSE"))
        fprintf(stderr, "mfd: K2 tma %d grid %d | K4 tma %d grid %d | yz_small %d fuse_k1 %d\n", (int)k2_tma_,
                k2_grid_, (int)k4_tma_, k4_grid_, (int)yz_small_, (int)fuse_k1_);
    ck(cudaStreamSynchronize(stream_), "setup");
}

// Device allocation of a persistent buffer.  With MFD_GUARD=1 every buffer
// gets kGuard bytes of 0xA5 before and after it (a write-overrun detector for
// the tests: compute-sanitizer is not available on the B200 pool);
// guard_check() counts the guard bytes that changed.
template <class T>
void* Engine<T>::dalloc(size_t bytes) {
    if (bytes == 0) bytes = 16;
    const size_t pad = guards_ ? kGuard : 0;
    void* base = nullptr;
    ck(cudaMalloc(&base, bytes + 2 * pad), "cudaMalloc");
    if (pad) {
        ck(cudaMemset(base, 0xA5, pad), "guard");
        ck(cudaMemset(static_cast<char*>(base) + pad + bytes, 0xA5, pad), "guard");
    }
    allocs_.push_back(Alloc{base, bytes});
    return static_cast<char*>(base) + pad;
}

template <class T>
long long Engine<T>::guard_check() {
    if (!guards_) return -1;
    ck(cudaStreamSynchronize(stream_), "sync");
    long long bad = 0;
    std::vector<unsigned char> h(kGuard);
    for (const auto& a : allocs_) {
        for (int side = 0; side < 2; ++side) {
            const char* g = static_cast<const char*>(a.base) + (side ? kGuard + a.bytes : 0);
            ck(cudaMemcpy(h.data(), g, kGuard, cudaMemcpyDeviceToHost), "guard read");
            for (unsigned char c : h) bad += c != 0xA5;
        }
    }
    return bad;
}

template <class T>
Engine<T>::~Engine() {
    release();
}

template <class T>
void Engine<T>::release() {
    cudaSetDevice(device_);
    if (stream_) cudaStreamSynchronize(stream_);
    if (cstream_) cudaStreamSynchronize(cstream_);
    if (copy_stream_) cudaStreamSynchronize(copy_stream_);
    for (auto& kv : graphs_) cudaGraphExecDestroy(kv.second);
    for (auto& a : allocs_) cudaFree(a.base);
    allocs_.clear();
    delete tr_;
    if (h_torque_) cudaFreeHost(h_torque_);
    if (h_sums_) cudaFreeHost(h_sums_);
    if (h_err_) cudaFreeHost(h_err_);
    if (h_perr_) cudaFreeHost(h_perr_);
    if (h_stage_) cudaFreeHost(h_stage_);
    for (auto& e : xev_)
        if (e) cudaEventDestroy(e);
    for (int q = 0; q < 2; ++q) {
        if (st_ready_[q]) cudaEventDestroy(st_ready_[q]);
        if (st_free_[q]) cudaEventDestroy(st_free_[q]);
    }
    if (copy_stream_) cudaStreamDestroy(copy_stream_);
    if (cstream_) cudaStreamDestroy(cstream_);
    if (stream_) cudaStreamDestroy(stream_);
}

// K0a + K0b, rank-local and memory-bounded.  The fp64 octant (computed on the
// device, or uploaded by the set_octant test hook) is produced a chunk of z
// planes at a time, and each chunk goes straight through the x transform
// restricted to this rank's x-bin block (Hv columns), so neither the full
// octant (6 N doubles: 6.4 GB at 1024x1024x128) nor a full-width intermediate
// is ever resident: per rank 6 x [nz][ny][Hv] + [nz][Hy][Hv] doubles plus one
// <= 256 MB octant chunk, all freed before the first step.  Per output
// element the GEMMs sum in the same order as a full-width transform, so every
// rank's block is bitwise the single-GPU spectrum.  The spectra are separable
// cos / sin transforms (the mirrored lattice has per-axis parity), so K~ comes
// out real: only its octant Kt is stored (layout in step_kernels.cuh).
template <class T>
void Engine<T>::build_tensor(const double* host_oct) {
    Nvtx r("setup: demag tensor + spectra (K0a/K0b)");
    const int nx = grid_.nx, ny = grid_.ny, nz = grid_.nz;   // global grid
    const int Hx = geo_.Hx, Wb = geo_.Wb, Hv = geo_.Hv, u0 = geo_.ublk * geo_.Wb;
    ck(cudaMemsetAsync(Kt_, 0, 6 * (long long)Hy_ * Hz_ * Wb * sizeof(T), stream_), "memset");
    if (Hv <= 0) {
        ck(cudaStreamSynchronize(stream_), "tensor setup");
        return;
    }
    const long long plane = (long long)nx * ny, n = plane * nz;
    const int KC = (int)std::max<long long>(1, std::min<long long>(nz, (256LL << 20) / (6 * plane * 8)));
    std::vector<void*> tmp;
    auto dalloc = [&](size_t bytes) {
        void* p = nullptr;
        ck(cudaMalloc(&p, bytes), "cudaMalloc (tensor setup)");
        tmp.push_back(p);
        return (double*)p;
    };
    try {
        double *Cx[2], *Cy[2], *Cz[2];
        auto mat = [&](double** C, int H, int nn, int P) {
            for (int odd = 0; odd < 2; ++odd) {
                C[odd] = dalloc((size_t)H * nn * sizeof(double));
                launch_axis_matrix(H, nn, P, odd, C[odd], stream_);
            }
        };
        mat(Cx, Hx, nx, geo_.Px);
        mat(Cy, Hy_, ny, Py_);
        mat(Cz, Hz_, nz, Pz_);
        double* Ech = dalloc((size_t)6 * KC * plane * sizeof(double));
        const long long t1c = (long long)nz * ny * Hv;               // T1 component stride
        double* T1 = dalloc((size_t)6 * t1c * sizeof(double));
        double* T2 = dalloc((size_t)nz * Hy_ * Hv * sizeof(double));
        // parity per component (xx,yy,zz,xy,xz,yz): odd along x / y / z
        const int ox[6] = {0, 0, 0, 1, 1, 0}, oy[6] = {0, 0, 0, 1, 0, 1}, oz[6] = {0, 0, 0, 0, 1, 1};
        for (int kb = 0; kb < nz; kb += KC) {
            const int kc = std::min(KC, nz - kb);
            const long long cs = (long long)kc * plane;               // chunk component stride
            if (host_oct) {
                for (int c = 0; c < 6; ++c)
                    ck(cudaMemcpyAsync(Ech + c * cs, host_oct + c * n + kb * plane, cs * sizeof(double),
                                       cudaMemcpyHostToDevice, stream_), "octant upload");
            } else {
                launch_tensor_octant(nx, ny, kb, kc, grid_.dx, grid_.dy, grid_.dz, Ech, stream_);
                ck(cudaGetLastError(), "k_tensor_octant");
            }
            for (int c = 0; c < 6; ++c) {
                // x: T1[k][j][u] = sum_i E[k][j][i] Cx[u0+u][i], u < Hv
                GemmDesc d{};
                d.Mdim = kc * ny; d.Ndim = Hv; d.Kdim = nx;
                d.a_m = nx; d.a_k = 1; d.b_k = 1; d.b_n = nx; d.o_m = Hv; d.o_n = 1; d.nb2 = 1; d.scale = 1.0;
                launch_gemm64(d, 1, Ech + c * cs, Cx[ox[c]] + (long long)u0 * nx, T1 + c * t1c + (long long)kb * ny * Hv,
                              stream_);
            }
            ck(cudaGetLastError(), "tensor gemm");
            if (host_oct) ck(cudaStreamSynchronize(stream_), "octant upload");   // pageable source
        }
        for (int c = 0; c < 6; ++c) {
            // y: T2[k][v][u] = sum_j Cy[v][j] T1[k][j][u]
            GemmDesc d{};
            d.Mdim = Hy_; d.Ndim = Hv; d.Kdim = ny;
            d.a_m = ny; d.a_k = 1; d.b_k = Hv; d.b_n = 1; d.o_m = Hv; d.o_n = 1;
            d.b_b1 = (long long)ny * Hv; d.o_b1 = (long long)Hy_ * Hv; d.nb2 = 1; d.scale = 1.0;
            launch_gemm64(d, nz, Cy[oy[c]], T1 + c * t1c, T2, stream_);
            // z: Kt[v][w][u][c] = s * sum_k Cz[w][k] T2[k][v][u]; two odd axes give
            // (-2i)^2 = -4 -> s = -1.  The six components of a bin are interleaved
            // so K3 reads them as three vectors.
            d = GemmDesc{};
            d.Mdim = Hz_; d.Ndim = Hv; d.Kdim = nz;
            d.a_m = nz; d.a_k = 1; d.b_k = (long long)Hy_ * Hv; d.b_n = 1; d.o_m = 6LL * Wb; d.o_n = 6;
            d.b_b1 = Hv; d.o_b1 = 6LL * Hz_ * Wb; d.nb2 = 1; d.scale = c >= 3 ? -1.0 : 1.0;
            launch_gemm64(d, Hy_, Cz[oz[c]], T2, Kt_ + c, stream_);
            ck(cudaGetLastError(), "tensor gemm");
        }
        ck(cudaStreamSynchronize(stream_), "tensor setup");
    } catch (...) {
        cudaStreamSynchronize(stream_);
        for (void* p : tmp) cudaFree(p);
        throw;
    }
    for (void* p : tmp) cudaFree(p);
}

template <class T>
void Engine<T>::set_octant(const double* oct) {
    if (!terms_.demag) throw Error(MFD_ELOGIC, "lastDemagField: demag term is disabled");
    build_tensor(oct);
}

// Test hook: the device octant is transient (freed after setup), so it is
// recomputed here for the caller.
template <class T>
void Engine<T>::get_octant(double* oct) {
    if (!terms_.demag) throw Error(MFD_ELOGIC, "lastDemagField: demag term is disabled");
    const long long n = 6LL * grid_.nx * grid_.ny * grid_.nz;
    double* d = nullptr;
    ck(cudaMalloc((void**)&d, n * sizeof(double)), "cudaMalloc");
    launch_tensor_octant(grid_.nx, grid_.ny, 0, grid_.nz, grid_.dx, grid_.dy, grid_.dz, d, stream_);
    const cudaError_t e1 = cudaGetLastError();
    const cudaError_t e2 = cudaMemcpyAsync(oct, d, n * sizeof(double), cudaMemcpyDeviceToHost, stream_);
    const cudaError_t e3 = cudaStreamSynchronize(stream_);
    cudaFree(d);
    ck(e1, "k_tensor_octant");
    ck(e2, "octant download");
    ck(e3, "octant download");
}

template <class T>
void Engine<T>::get_spectrum(double* out) {
    if (!terms_.demag) throw Error(MFD_ELOGIC, "lastDemagField: demag term is disabled");
    if (geo_.G != 1) throw Error(MFD_EINVAL, "get_spectrum: single-GPU contexts only");
    const long long cnt = 6LL * Hy_ * Hz_ * geo_.Wb;
    std::vector<T> h(cnt);
    ck(cudaMemcpy(h.data(), Kt_, cnt * sizeof(T), cudaMemcpyDeviceToHost), "spectrum download");
    const int Hx = geo_.Hx;
    for (int c = 0; c < 6; ++c)
        for (int v = 0; v < Hy_; ++v)
            for (int w = 0; w < Hz_; ++w)
                for (int u = 0; u < Hx; ++u)
                    out[(((long long)c * Hy_ + v) * Hz_ + w) * Hx + u] =
                        (double)h[(((long long)v * Hz_ + w) * geo_.Wb + u) * 6 + c];
}

// --------------------------------------------------------------- enqueue
template <class T>
Ctl Engine<T>::make_ctl(const Iter& it) const {
    return Ctl{err_, it.check_prev && it.slot > 0 ? torque_ + it.slot - 1 : nullptr, mat_.Ms,
               st_.torque_tol_deg_per_ns, kRadToDegPerNs};
}

template <class T>
StepIO Engine<T>::make_io(const Iter& it) const {
    StepIO io{};
    io.update = it.update;
    io.renorm = it.renorm;
    io.write_h = it.write_h;
    io.sums = it.sums;
    io.iter = it.slot;
    io.torque = torque_ + it.slot;
    io.partials = partials_;
    io.sums_out = sums_ + 8 * it.slot;
    io.ticket = ticket_;
    return io;
}

template <class T>
Halo<T> Engine<T>::halo_ptrs() const {
    const long long plane = 3LL * grid_.nx * grid_.ny;
    Halo<T> h{nullptr, nullptr};
    if (slab_.world > 1 && slab_.rank > 0) h.lo = halo_;
    if (slab_.world > 1 && slab_.rank < slab_.world - 1) h.hi = halo_ + plane;
    return h;
}

template <class T>
void Engine<T>::enq_local(const Iter& it, int cur) {
    Nvtx r("localFields + integrate");
    note("K5 k_local_llg<%s>", tn());
    k_local_llg<T><<<(unsigned)((geo_.ncell + 255) / 256), 256, 0, stream_>>>(
        geo_, M_[cur], M_[cur ^ 1], H_, lp_, make_io(it), make_ctl(it), halo_ptrs());
}

// A: K1 (x, R2C) -> A_ (on several GPUs: the send blocks, one per rank's x-bins)
template <class T>
void Engine<T>::enq_A(const Iter& it, int cur, cudaEvent_t* ev, bool skip_k1) {
    Nvtx r("pad+forwardFft x (K1)");
    const Ctl ctl = make_ctl(it);
    const long long nrows = (long long)geo_.ny * geo_.nz;
    if (!skip_k1) with_pow2(geo_.N, [&]<int L>() {
        using CF = XCfg<T, L>;
        if (small_x_) {
            if constexpr (L >= 2 && L <= kSmallXMax) {
                using CS = XCfg<T, L, 2>;
                dim3 grid((unsigned)((nrows + 1) / 2), 3);
                auto* k = geo_.G > 1 ? k_r2c_x<T, L, 2, true> : k_r2c_x<T, L, 2, false>;
                note("K1 k_r2c_x<%s,%d,RS=2,MULTI=%d>", tn(), L, (int)(geo_.G > 1));
                k<<<grid, CS::NT, CS::SMEM, stream_>>>(geo_, M_[cur], A_, tw_, ctl);
            }
        } else {
            dim3 grid((unsigned)((nrows + CF::ROWS - 1) / CF::ROWS), 3);
            auto* k = geo_.G > 1 ? k_r2c_x<T, L, 0, true> : k_r2c_x<T, L, 0, false>;
            note("K1 k_r2c_x<%s,%d,RS=0,MULTI=%d>", tn(), L, (int)(geo_.G > 1));
            k<<<grid, CF::NT, CF::SMEM, stream_>>>(geo_, M_[cur], A_, tw_, ctl);
        }
    });
    if (ev) ck(cudaEventRecordWithFlags(ev[1], stream_, cudaEventRecordExternal), "event");
}

// B: K2 (y forward) -> K3 (z, tensor product, inverse z) -> K4 (y inverse) on
// this rank's x-bin block of every plane: Ar_ -> B_ -> Ar_ (Ar_ = A_ on one GPU)
template <class T>
void Engine<T>::enq_B(const Iter& it, cudaEvent_t* ev) {
    const Ctl ctl = make_ctl(it);
    if (yz()) {   // K2 + K3 + K4 in one kernel (thin / small grids, one GPU)
        if (stop_after_ >= 2 && stop_after_ <= 3) return;
        with_yz([&]<int LY, int LZ>() {
            using CF = YZCfg<T, LY, LZ>;
            note("K234 k_fft_yz_small<%s,%d,%d>", tn(), LY, LZ);
            k_fft_yz_small<T, LY, LZ><<<(geo_.Hx + CF::W - 1) / CF::W, CF::NT, CF::SMEM, stream_>>>(
                geo_, A_, Kt_, tw_, ybuf_, ctl);
        });
        if (ev) for (int q = 2; q <= 4; ++q) ck(cudaEventRecordWithFlags(ev[q], stream_, cudaEventRecordExternal), "event");
        return;
    }
    enq_K2(ctl, 0, 3);
    if (ev) ck(cudaEventRecordWithFlags(ev[2], stream_, cudaEventRecordExternal), "event");
    if (stop_after_ == 2) return;
    enq_K3(ctl);
    if (ev) ck(cudaEventRecordWithFlags(ev[3], stream_, cudaEventRecordExternal), "event");
    if (stop_after_ == 3) return;
    enq_K4(ctl, 0, 3);
    if (ev) ck(cudaEventRecordWithFlags(ev[4], stream_, cudaEventRecordExternal), "event");
}

// K2 (y forward) of components [comp0, comp0 + ncomp): Ar_ -> B_
template <class T>
void Engine<T>::enq_K2(const Ctl& ctl, int comp0, int ncomp) {
    Nvtx r("forwardFft y (K2)");
    if (geo_.Hv <= 0) return;
    if (k2_tma_) {
        with_pow2(Py_, [&]<int L>() {
            if constexpr (YTCfg<T, L>::OK) {
                using CF = YTCfg<T, L>;
                const int ntx = (geo_.Hv + CF::W - 1) / CF::W;
                auto* k = 2 * geo_.ny == L ? k_fft_y_fwd_tma<T, L, true> : k_fft_y_fwd_tma<T, L, false>;
                note("K2 k_fft_y_fwd_tma<%s,%d,FY=%d>", tn(), L, (int)(2 * geo_.ny == L));
                const int grid = (int)std::min<long long>(k2_grid_, (long long)ntx * geo_.nzg * ncomp);
                k<<<grid, CF::NT, CF::SMEM, stream_>>>(geo_, tmA_, B_, tw_, ctl, ntx, k2_box_, comp0, ncomp);
            }
        });
    } else {
        with_pow2(Py_, [&]<int L>() {
            using CF = YCfg<T, L>;
            dim3 grid((geo_.Hv + CF::W - 1) / CF::W, geo_.nzg, ncomp);
            note("K2 k_fft_y_fwd<%s,%d,FY=%d>", tn(), L, (int)(2 * geo_.ny == L));
            if (2 * geo_.ny == L)
                k_fft_y_fwd<T, L, true><<<grid, CF::NT, CF::SMEM, stream_>>>(geo_, Ar_, B_, tw_, ctl, comp0);
            else
                k_fft_y_fwd<T, L, false><<<grid, CF::NT, CF::SMEM, stream_>>>(geo_, Ar_, B_, tw_, ctl, comp0);
        });
    }
}

// K3 (z transform, tensor product, inverse z) on B_, all components
template <class T>
void Engine<T>::enq_K3(const Ctl& ctl) {
    Nvtx r("forwardFft z + spectralMultiply + inverseFft z (K3)");
    if (geo_.Hv <= 0) return;
    with_pow2(Pz_, [&]<int L>() {
        if constexpr (z_variant<T, L>() == 1) {
            dim3 grid((geo_.Hv + 31) / 32, Hy_, 1);
            note("K3 k_fft_z_conv1<%s,%d>", tn(), L);
            k_fft_z_conv1<T, L><<<grid, 64, 0, stream_>>>(geo_, B_, Kt_, ybuf_, ctl);
        } else if constexpr (z_variant<T, L>() == 2) {
            if (k3_srow_) {
                using CF = Z2Cfg<T, L, true>;
                dim3 grid((geo_.Hv + CF::W - 1) / CF::W, Py_, 1);
                auto* k = 2 * geo_.nzg == L ? k_fft_z_conv2<T, L, true, true> : k_fft_z_conv2<T, L, false, true>;
                note("K3 k_fft_z_conv2<%s,%d,FZ=%d,SROW=1>", tn(), L, (int)(2 * geo_.nzg == L));
                k<<<grid, CF::NT, CF::SMEM, stream_>>>(geo_, B_, Kt_, tw_, ybuf_, ctl);
            } else {
                using CF = Z2Cfg<T, L>;
                dim3 grid((geo_.Hv + CF::W - 1) / CF::W, Hy_, 1);
                auto* k = 2 * geo_.nzg == L ? k_fft_z_conv2<T, L, true> : k_fft_z_conv2<T, L, false>;
                note("K3 k_fft_z_conv2<%s,%d,FZ=%d,SROW=0>", tn(), L, (int)(2 * geo_.nzg == L));
                k<<<grid, CF::NT, CF::SMEM, stream_>>>(geo_, B_, Kt_, tw_, ybuf_, ctl);
            }
        } else {
            using CF = ZCfg<T, L>;
            dim3 grid((geo_.Hv + CF::W - 1) / CF::W, Hy_, 1);
            note("K3 k_fft_z_conv<%s,%d>", tn(), L);
            k_fft_z_conv<T, L><<<grid, CF::NT, CF::SMEM, stream_>>>(geo_, B_, Kt_, tw_, ybuf_, ctl);
        }
    });
}

// K4 (y inverse) of components [comp0, comp0 + ncomp): B_ -> Ar_
template <class T>
void Engine<T>::enq_K4(const Ctl& ctl, int comp0, int ncomp) {
    Nvtx r("inverseFft y (K4)");
    if (geo_.Hv <= 0) return;
    if (k4_tma_) with_pow2(Py_, [&]<int L>() {
        if constexpr (YICfg<T, L>::OK) {
            using CF = YICfg<T, L>;
            const int ntx = (geo_.Hv + CF::W - 1) / CF::W;
            auto* k = 2 * geo_.ny == L ? k_fft_y_inv_tma<T, L, true> : k_fft_y_inv_tma<T, L, false>;
            note("K4 k_fft_y_inv_tma<%s,%d,FY=%d>", tn(), L, (int)(2 * geo_.ny == L));
            const int grid = (int)std::min<long long>(k4_grid_, (long long)ntx * geo_.nzg * ncomp);
            k<<<grid, CF::NT, CF::SMEM, stream_>>>(geo_, tmB_, Ar_, tw_, ctl, ntx, comp0, ncomp);
        }
    });
    else with_pow2(Py_, [&]<int L>() {
        using CF = YCfg<T, L>;
        dim3 grid((geo_.Hv + CF::W - 1) / CF::W, geo_.nzg, ncomp);
        note("K4 k_fft_y_inv<%s,%d,FY=%d>", tn(), L, (int)(2 * geo_.ny == L));
        if (2 * geo_.ny == L)
            k_fft_y_inv<T, L, true><<<grid, CF::NT, CF::SMEM, stream_>>>(geo_, B_, Ar_, tw_, ctl, comp0);
        else
            k_fft_y_inv<T, L, false><<<grid, CF::NT, CF::SMEM, stream_>>>(geo_, B_, Ar_, tw_, ctl, comp0);
    });
}

// C: K5 (x inverse + H_eff + LLG + Euler) on A_ (the receive side of the second transpose)
template <class T>
void Engine<T>::enq_C(const Iter& it, int cur, cudaEvent_t* ev, bool fwd) {
    Nvtx r("inverseFft x + localFields + integrate (K5)");
    const Ctl ctl = make_ctl(it);
    const StepIO io = make_io(it);
    const Halo<T> hl = halo_ptrs();
    const long long nrows = (long long)geo_.ny * geo_.nz;
    const T* Mc = M_[cur];
    T* Mn = M_[cur ^ 1];
    with_pow2(geo_.N, [&]<int L>() {
        using CF = LCfg<T, L>;
        dim3 grid((unsigned)((nrows + CF::ROWS - 1) / CF::ROWS), 1);
        if constexpr (L >= 2 && L <= kSmallXMax) {
            if (small_x_) {   // one row per CTA (few-row grids such as SP4)
                using CS = LCfg<T, L, 1>;
                auto* k = geo_.G > 1
                              ? (io.sums ? k_c2r_x_llg_v<T, L, true, 1, false, true>
                                         : k_c2r_x_llg_v<T, L, false, 1, false, true>)
                          : io.sums ? (fwd ? k_c2r_x_llg_v<T, L, true, 1, true> : k_c2r_x_llg_v<T, L, true, 1, false>)
                                    : (fwd ? k_c2r_x_llg_v<T, L, false, 1, true> : k_c2r_x_llg_v<T, L, false, 1, false>);
                note("K5 k_c2r_x_llg_v<%s,%d,SUMS=%d,RS=1,FWD=%d,MULTI=%d>", tn(), L, (int)(io.sums != 0),
                     (int)(fwd && geo_.G == 1), (int)(geo_.G > 1));
                k<<<(unsigned)nrows, CS::NT, CS::SMEM, stream_>>>(geo_, A_, Mc, Mn, H_, tw_, scale_, lp_, io, ctl, hl);
                return;
            }
        }
        const bool multi = geo_.G > 1;
        if (geo_.nx % V16<T>::V == 0) {
            auto* k = multi ? (io.sums ? k_c2r_x_llg_v<T, L, true, 0, false, true>
                                       : k_c2r_x_llg_v<T, L, false, 0, false, true>)
                    : io.sums ? (fwd ? k_c2r_x_llg_v<T, L, true, 0, true> : k_c2r_x_llg_v<T, L, true, 0, false>)
                              : (fwd ? k_c2r_x_llg_v<T, L, false, 0, true> : k_c2r_x_llg_v<T, L, false, 0, false>);
            const int smem = fwd && !multi ? k5_smem<T, L, 0, true>() : k5_smem<T, L, 0, false>();
            note("K5 k_c2r_x_llg_v<%s,%d,SUMS=%d,RS=0,FWD=%d,MULTI=%d>", tn(), L, (int)(io.sums != 0),
                 (int)(fwd && !multi), (int)multi);
            k<<<grid, CF::NT, smem, stream_>>>(geo_, A_, Mc, Mn, H_, tw_, scale_, lp_, io, ctl, hl);
        } else {
            auto* k = multi ? k_c2r_x_llg<T, L, true> : k_c2r_x_llg<T, L, false>;
            note("K5 k_c2r_x_llg<%s,%d,MULTI=%d>", tn(), L, (int)multi);
            k<<<grid, CF::NT, CF::SMEM, stream_>>>(geo_, A_, Mc, Mn, H_, tw_, scale_, lp_, io, ctl, hl);
        }
    });
}

// One iteration.  Multi-GPU (tr_ set): the M halo, the two all-to-all
// transposes and the scalar allreduces are enqueued like the kernels, so they
// are captured into the step graph.  The transposes run per component on a
// second stream (cstream_) and overlap the y passes:
// all-to-all #1 of component c+1 flies while K2 transforms component c, and
// all-to-all #2 of component c while K4 transforms c+1; the halo (needed only
// by K5) flies during K1-K4.  The passes themselves are the single-GPU ones.
template <class T>
void Engine<T>::enqueue(const Iter& it, int cur, bool events, cudaEvent_t* ev, bool skip_k1, bool fwd) {
    const size_t tsz = sizeof(T);
    const bool multi = tr_ && slab_.world > 1;
    if (events) ck(cudaEventRecordWithFlags(ev[0], stream_, cudaEventRecordExternal), "event");
    if (multi) {   // fork: the comm stream joins everything enqueued so far
        ck(cudaEventRecord(xev_[0], stream_), "event");
        ck(cudaStreamWaitEvent(cstream_, xev_[0], 0), "wait");
        tr_->halo(M_[cur], geo_.ncell * tsz, (size_t)grid_.nx * grid_.ny * tsz, geo_.nz, halo_,
                  halo_ + 3LL * grid_.nx * grid_.ny, cstream_);
    }
    if (!terms_.demag) {
        if (multi) {   // join before the stencil
            ck(cudaEventRecord(xev_[1], cstream_), "event");
            ck(cudaStreamWaitEvent(stream_, xev_[1], 0), "wait");
        }
        enq_local(it, cur);
        if (events)
            for (int q = 1; q < 6; ++q) ck(cudaEventRecordWithFlags(ev[q], stream_, cudaEventRecordExternal), "event");
    } else if (!multi) {
        enq_A(it, cur, events ? ev : nullptr, skip_k1);
        if (stop_after_ == 1) return;
        enq_B(it, events ? ev : nullptr);
        if (stop_after_ >= 2 && stop_after_ <= 4) return;
        enq_C(it, cur, events ? ev : nullptr, fwd);
        if (events) ck(cudaEventRecordWithFlags(ev[5], stream_, cudaEventRecordExternal), "event");
    } else {
        const Ctl ctl = make_ctl(it);
        // component c of x-bin block p sits at p * SA + c * cblk (contiguous)
        const size_t cblk = (size_t)geo_.nz * geo_.ny * geo_.Hp, stride = (size_t)geo_.SA * sizeof(C2<T>);
        const size_t cbytes = cblk * sizeof(C2<T>);
        enq_A(it, cur, events ? ev : nullptr, false);
        ck(cudaEventRecord(xev_[1], stream_), "event");
        ck(cudaStreamWaitEvent(cstream_, xev_[1], 0), "wait");
        for (int c = 0; c < 3; ++c) {   // transpose #1: x-bin block p of every local plane -> rank p
            Nvtx r("transpose #1 (all-to-all, x-spectrum)");
            tr_->alltoall(A_ + c * cblk, Ar_ + c * cblk, cbytes, stride, cstream_);
            ck(cudaEventRecord(xev_[2 + c], cstream_), "event");
        }
        for (int c = 0; c < 3; ++c) {
            ck(cudaStreamWaitEvent(stream_, xev_[2 + c], 0), "wait");
            enq_K2(ctl, c, 1);
        }
        if (events) ck(cudaEventRecordWithFlags(ev[2], stream_, cudaEventRecordExternal), "event");
        enq_K3(ctl);
        if (events) ck(cudaEventRecordWithFlags(ev[3], stream_, cudaEventRecordExternal), "event");
        for (int c = 0; c < 3; ++c) {   // transpose #2 (inverse): back to this rank's planes, all x-bins
            enq_K4(ctl, c, 1);
            ck(cudaEventRecord(xev_[5 + c], stream_), "event");
            ck(cudaStreamWaitEvent(cstream_, xev_[5 + c], 0), "wait");
            Nvtx r("transpose #2 (all-to-all, x-spectrum)");
            tr_->alltoall(Ar_ + c * cblk, A_ + c * cblk, cbytes, stride, cstream_);
        }
        if (events) ck(cudaEventRecordWithFlags(ev[4], stream_, cudaEventRecordExternal), "event");
        ck(cudaEventRecord(xev_[8], cstream_), "event");   // join (also covers the halo)
        ck(cudaStreamWaitEvent(stream_, xev_[8], 0), "wait");
        enq_C(it, cur, events ? ev : nullptr, false);
        if (events) ck(cudaEventRecordWithFlags(ev[5], stream_, cudaEventRecordExternal), "event");
    }
    if (multi) {
        tr_->allreduce_max_u64(torque_ + it.slot, 1, stream_);
        tr_->allreduce_max_i32(err_, 1, stream_);
        if (it.sums) tr_->allreduce_sum_f64(sums_ + 8 * it.slot, 7, stream_);
    }
}

// The CUDA graph of a chunk of iterations (captured once, cached by its shape).
template <class T>
cudaGraphExec_t Engine<T>::chunk_graph(const std::vector<Iter>& its, int cur) {
    auto key = std::make_pair(its, cur);
    auto f = graphs_.find(key);
    if (f == graphs_.end()) {
        if (graphs_.size() > 64) {
            for (auto& kv : graphs_) cudaGraphExecDestroy(kv.second);
            graphs_.clear();
            graph_kernels_.clear();
        }
        cudaGraph_t g;
        ck(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal), "capture");
        cudaMemsetAsync(torque_, 0, its.size() * sizeof(unsigned long long), stream_);
        // a launch that halted part-way (error flag raised by an earlier CTA)
        // leaves the last-block ticket short; every graph starts from zero
        cudaMemsetAsync(ticket_, 0, sizeof(unsigned int), stream_);
        int c = cur;
        bool fused_prev = false;
        for (size_t j = 0; j < its.size(); ++j) {
            const Iter& it = its[j];
            // K5 of an updating iteration followed by another one in this graph
            // also produces the next iteration's K1 output
            const bool fuse = fuse_k1_ && it.update && j + 1 < its.size();
            enqueue(it, c, false, nullptr, fused_prev, fuse);
            fused_prev = fuse;
            if (it.update) c ^= 1;
        }
        ck(cudaStreamEndCapture(stream_, &g), "end capture");
        size_t nn = 0;
        ck(cudaGraphGetNodes(g, nullptr, &nn), "graph nodes");
        std::vector<cudaGraphNode_t> nodes(nn);
        if (nn) ck(cudaGraphGetNodes(g, nodes.data(), &nn), "graph nodes");
        int nk = 0;
        for (auto nd : nodes) {
            cudaGraphNodeType ty;
            ck(cudaGraphNodeGetType(nd, &ty), "node type");
            nk += ty == cudaGraphNodeTypeKernel;
        }
        graph_kernels_[key] = nk;
        cudaGraphExec_t ex;
        ck(cudaGraphInstantiate(&ex, g, 0), "graph instantiate");
        cudaGraphDestroy(g);
        f = graphs_.emplace(key, ex).first;
    }
    return f->second;
}

// Launch a chunk of iterations.
template <class T>
void Engine<T>::run_chunk(const std::vector<Iter>& its, int cur) {
    Nvtx r("step chunk (graph launch)");
    ck(cudaGraphLaunch(chunk_graph(its, cur), stream_), "graph launch");
}

template <class T>
void Engine<T>::fetch_chunk(int n, std::vector<double>& torque, int& err) {
    ck(cudaMemcpyAsync(h_torque_, torque_, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost, stream_), "d2h");
    ck(cudaMemcpyAsync(h_sums_, sums_, (size_t)n * 8 * sizeof(double), cudaMemcpyDeviceToHost, stream_), "d2h");
    ck(cudaMemcpyAsync(h_err_, err_, sizeof(int), cudaMemcpyDeviceToHost, stream_), "d2h");
    ck(cudaStreamSynchronize(stream_), "sync");
    torque.resize(n);
    for (int i = 0; i < n; ++i) torque[i] = torque_of(h_torque_[i]);
    err = *h_err_;
    if (err) ck(cudaMemsetAsync(err_, 0, sizeof(int), stream_), "memset");
}

template <class T>
double Engine<T>::torque_of(unsigned long long bits) const {
    double r;
    std::memcpy(&r, &bits, sizeof r);
    return std::sqrt(r) / mat_.Ms * kRadToDegPerNs;   // dynamics.hpp:81
}

// --------------------------------------------------------------- state io
// Same-precision transfers go straight from the caller's buffers (DMA at full
// PCIe speed when they are pinned); cross-precision ones convert through the
// pinned staging buffer.
template <class T>
static void copy3_h2d(T* dst, const T* x, const T* y, const T* z, long long n, cudaStream_t s) {
    ck(cudaMemcpyAsync(dst, x, n * sizeof(T), cudaMemcpyHostToDevice, s), "h2d");
    ck(cudaMemcpyAsync(dst + n, y, n * sizeof(T), cudaMemcpyHostToDevice, s), "h2d");
    ck(cudaMemcpyAsync(dst + 2 * n, z, n * sizeof(T), cudaMemcpyHostToDevice, s), "h2d");
    ck(cudaStreamSynchronize(s), "sync");
}
template <class T>
static void copy3_d2h(const T* src, T* x, T* y, T* z, long long n, cudaStream_t s) {
    ck(cudaMemcpyAsync(x, src, n * sizeof(T), cudaMemcpyDeviceToHost, s), "d2h");
    ck(cudaMemcpyAsync(y, src + n, n * sizeof(T), cudaMemcpyDeviceToHost, s), "d2h");
    ck(cudaMemcpyAsync(z, src + 2 * n, n * sizeof(T), cudaMemcpyDeviceToHost, s), "d2h");
    ck(cudaStreamSynchronize(s), "sync");
}

template <class T>
void Engine<T>::set_m(const double* x, const double* y, const double* z) {
    consume_staged();   // a later direct write wins over earlier staged states
    const long long n = geo_.ncell;
    if constexpr (std::is_same_v<T, double>) {
        copy3_h2d<T>(M_[cur_], x, y, z, n, stream_);
        return;
    }
    ensure_stage();
    for (long long i = 0; i < n; ++i) {
        h_stage_[i] = static_cast<T>(x[i]);
        h_stage_[i + n] = static_cast<T>(y[i]);
        h_stage_[i + 2 * n] = static_cast<T>(z[i]);
    }
    ck(cudaMemcpyAsync(M_[cur_], h_stage_, 3 * n * sizeof(T), cudaMemcpyHostToDevice, stream_), "h2d");
    ck(cudaStreamSynchronize(stream_), "sync");
}
template <class T>
void Engine<T>::set_m32(const float* x, const float* y, const float* z) {
    consume_staged();   // a later direct write wins over earlier staged states
    const long long n = geo_.ncell;
    if constexpr (std::is_same_v<T, float>) {
        copy3_h2d<T>(M_[cur_], x, y, z, n, stream_);
        return;
    }
    ensure_stage();
    for (long long i = 0; i < n; ++i) {
        h_stage_[i] = static_cast<T>(x[i]);
        h_stage_[i + n] = static_cast<T>(y[i]);
        h_stage_[i + 2 * n] = static_cast<T>(z[i]);
    }
    ck(cudaMemcpyAsync(M_[cur_], h_stage_, 3 * n * sizeof(T), cudaMemcpyHostToDevice, stream_), "h2d");
    ck(cudaStreamSynchronize(stream_), "sync");
}
template <class T>
void Engine<T>::get_m(double* x, double* y, double* z) {
    consume_staged();
    const long long n = geo_.ncell;
    if constexpr (std::is_same_v<T, double>) {
        copy3_d2h<T>(M_[cur_], x, y, z, n, stream_);
        return;
    }
    ensure_stage();
    ck(cudaMemcpyAsync(h_stage_, M_[cur_], 3 * n * sizeof(T), cudaMemcpyDeviceToHost, stream_), "d2h");
    ck(cudaStreamSynchronize(stream_), "sync");
    for (long long i = 0; i < n; ++i) {
        x[i] = h_stage_[i];
        y[i] = h_stage_[i + n];
        z[i] = h_stage_[i + 2 * n];
    }
}
template <class T>
void Engine<T>::get_m32(float* x, float* y, float* z) {
    consume_staged();
    const long long n = geo_.ncell;
    if constexpr (std::is_same_v<T, float>) {
        copy3_d2h<T>(M_[cur_], x, y, z, n, stream_);
        return;
    }
    ensure_stage();
    ck(cudaMemcpyAsync(h_stage_, M_[cur_], 3 * n * sizeof(T), cudaMemcpyDeviceToHost, stream_), "d2h");
    ck(cudaStreamSynchronize(stream_), "sync");
    for (long long i = 0; i < n; ++i) {
        x[i] = (float)h_stage_[i];
        y[i] = (float)h_stage_[i + n];
        z[i] = (float)h_stage_[i + 2 * n];
    }
}
// Overlapped state upload: the host arrays (pinned for a true async copy; they
// must stay untouched until the next call that reads the state returns) go to
// a device staging buffer on a copy stream, so the transfer of the next
// step's state overlaps the current step; two slots in flight at most.
template <class T>
void Engine<T>::stage_m(const void* x, const void* y, const void* z, int bits) {
    if (bits != (int)(8 * sizeof(T))) {   // other precision: converting copy, synchronous
        consume_staged();
        if (bits == 32) set_m32((const float*)x, (const float*)y, (const float*)z);
        else set_m((const double*)x, (const double*)y, (const double*)z);
        return;
    }
    const long long n = geo_.ncell;
    if (!copy_stream_) {
        ck(cudaStreamCreateWithFlags(&copy_stream_, cudaStreamNonBlocking), "stream");
        for (int s = 0; s < 2; ++s) {
            Mst_[s] = static_cast<T*>(dalloc(3 * n * sizeof(T)));
            ck(cudaEventCreateWithFlags(&st_ready_[s], cudaEventDisableTiming), "event");
            ck(cudaEventCreateWithFlags(&st_free_[s], cudaEventDisableTiming), "event");
            ck(cudaEventRecord(st_free_[s], stream_), "event");
        }
    }
    if ((int)st_pending_.size() == 2) consume_staged();   // at most two states in flight
    const int s = st_next_;
    st_next_ ^= 1;
    ck(cudaStreamWaitEvent(copy_stream_, st_free_[s], 0), "wait");   // its previous install is done
    ck(cudaMemcpyAsync(Mst_[s], x, n * sizeof(T), cudaMemcpyHostToDevice, copy_stream_), "h2d");
    ck(cudaMemcpyAsync(Mst_[s] + n, y, n * sizeof(T), cudaMemcpyHostToDevice, copy_stream_), "h2d");
    ck(cudaMemcpyAsync(Mst_[s] + 2 * n, z, n * sizeof(T), cudaMemcpyHostToDevice, copy_stream_), "h2d");
    ck(cudaEventRecord(st_ready_[s], copy_stream_), "event");
    st_pending_.push_back(s);
}

// Install the oldest staged state (if any) into M_[cur_], in stream order.
template <class T>
void Engine<T>::consume_staged() {
    while (!st_pending_.empty()) {
        const int s = st_pending_.front();
        st_pending_.erase(st_pending_.begin());
        ck(cudaStreamWaitEvent(stream_, st_ready_[s], 0), "wait");
        ck(cudaMemcpyAsync(M_[cur_], Mst_[s], 3 * geo_.ncell * sizeof(T), cudaMemcpyDeviceToDevice, stream_), "d2d");
        ck(cudaEventRecord(st_free_[s], stream_), "event");   // a later staged state overwrites this one
    }
}

template <class T>
void Engine<T>::set_uniform(const double dir[3]) {
    consume_staged();   // a later direct write wins over earlier staged states
    // makeUniformState: (Ms * direction).cast<T>() (state.hpp:71-78)
    const double Ms = mat_.Ms;
    k_fill3<T><<<(unsigned)((geo_.ncell + 255) / 256), 256, 0, stream_>>>(
        M_[cur_], geo_.ncell, static_cast<T>(Ms * dir[0]), static_cast<T>(Ms * dir[1]), static_cast<T>(Ms * dir[2]));
    ck(cudaGetLastError(), "fill");
    ck(cudaStreamSynchronize(stream_), "sync");
}

template <class T>
void Engine<T>::set_vortex(int axis) {
    consume_staged();   // a later direct write wins over earlier staged states
    static const double av[6][3] = {{1, 0, 0}, {-1, 0, 0}, {0, 1, 0}, {0, -1, 0}, {0, 0, 1}, {0, 0, -1}};
    if (axis < 0 || axis > 5) throw Error(MFD_EINVAL, "axisVector: bad axis");
    const double* a = av[axis];
    const bool along_x = a[0] != 0, along_y = a[1] != 0;
    const int p1 = along_x ? grid_.ny : grid_.nx, p2 = (along_x || along_y) ? grid_.nz : grid_.ny;
    if (p1 < 2 || p2 < 2)
        throw Error(MFD_EINVAL, "makeVortexState: need >= 2 cells along each axis perpendicular to the core");
    if (geo_.ncell > 0)
        k_vortex<T><<<(unsigned)((geo_.ncell + 255) / 256), 256, 0, stream_>>>(
            M_[cur_], grid_.nx, grid_.ny, geo_.nz, grid_.nz, geo_.k0, grid_.dx, grid_.dy, grid_.dz, a[0], a[1], a[2],
            mat_.Ms);
    ck(cudaGetLastError(), "vortex");
    ck(cudaStreamSynchronize(stream_), "sync");
}

// One evaluation without update (H, torque and optionally the sample sums).
template <class T>
void Engine<T>::eval(int write_h, bool sums, double& torque, double sum_out[8]) {
    consume_staged();
    Iter it;
    it.update = 0;
    it.renorm = 0;
    it.write_h = write_h;
    it.sums = sums;
    it.slot = 0;
    run_chunk({it}, cur_);
    std::vector<double> tq;
    int err = 0;
    fetch_chunk(1, tq, err);
    torque = tq[0];
    if (sum_out) std::memcpy(sum_out, h_sums_, 8 * sizeof(double));
}

template <class T>
void Engine<T>::field(int which, double* x, double* y, double* z) {
    if (which == 2 && !terms_.demag) throw Error(MFD_ELOGIC, "lastDemagField: demag term is disabled");
    double tq;
    eval(which, false, tq, nullptr);
    const long long n = geo_.ncell;
    ensure_stage();
    ck(cudaMemcpyAsync(h_stage_, H_, 3 * n * sizeof(T), cudaMemcpyDeviceToHost, stream_), "d2h");
    ck(cudaStreamSynchronize(stream_), "sync");
    for (long long i = 0; i < n; ++i) {
        x[i] = h_stage_[i];
        y[i] = h_stage_[i + n];
        z[i] = h_stage_[i + 2 * n];
    }
}

template <class T>
void Engine<T>::field32(int which, float* x, float* y, float* z) {
    if (which == 2 && !terms_.demag) throw Error(MFD_ELOGIC, "lastDemagField: demag term is disabled");
    double tq;
    eval(which, false, tq, nullptr);
    const long long n = geo_.ncell;
    if constexpr (std::is_same_v<T, float>) {
        copy3_d2h<T>(H_, x, y, z, n, stream_);
        return;
    }
    ensure_stage();
    ck(cudaMemcpyAsync(h_stage_, H_, 3 * n * sizeof(T), cudaMemcpyDeviceToHost, stream_), "d2h");
    ck(cudaStreamSynchronize(stream_), "sync");
    for (long long i = 0; i < n; ++i) {
        x[i] = (float)h_stage_[i];
        y[i] = (float)h_stage_[i + n];
        z[i] = (float)h_stage_[i + 2 * n];
    }
}

// Replace the stepper configuration (dt, renormalisation cadence, relax
// limits).  dt is baked into the captured graphs' parameters: drop them.
template <class T>
void Engine<T>::set_stepper(const mfd_stepper& s) {
    ck(cudaStreamSynchronize(stream_), "sync");
    st_ = s;
    lp_.dt = static_cast<T>(s.dt);
    for (auto& kv : graphs_) cudaGraphExecDestroy(kv.second);
    graphs_.clear();
    graph_kernels_.clear();
}

// --------------------------------------------------------------- stepping
// Simulation<T>::step x n: renormalise iff (step+1) % renormalizeEvery == 0 (sim.hpp:38).
template <class T>
void Engine<T>::step(long n, double* last, double* all) {
    consume_staged();
    long done = 0;
    std::vector<double> tq;
    while (done < n) {
        const int K = (int)std::min<long>(n - done, 64);
        std::vector<Iter> its(K);
        for (int i = 0; i < K; ++i) {
            its[i].slot = i;
            its[i].renorm = ((stepno + i + 1) % st_.renorm_every) == 0;
        }
        run_chunk(its, cur_);
        int err = 0;
        fetch_chunk(K, tq, err);
        const int ok = err ? err - 1 : K;      // iterations that completed their update
        for (int i = 0; i < ok; ++i) {
            t += st_.dt;                        // dynamics.hpp:118-119
            stepno += 1;
            cur_ ^= 1;
            if (all) all[done + i] = tq[i];
        }
        if (err) {
            if (last) *last = tq[ok];
            throw Error(MFD_ENONFINITE, "eulerUpdate: non-finite magnetization after step (time step too large?)");
        }
        done += K;
        if (last) *last = tq[K - 1];
    }
}

// Iterations of a K-step step_async chunk starting at step count step0:
// renormalise iff (step+1) % renormalizeEvery == 0 (sim.hpp:38).
template <class T>
std::vector<Iter> Engine<T>::async_chunk(int K, long step0) const {
    std::vector<Iter> its(K);
    for (int i = 0; i < K; ++i) {
        its[i].slot = i;
        its[i].renorm = ((step0 + i + 1) % st_.renorm_every) == 0;
    }
    return its;
}

template <class T>
long Engine<T>::prepare_async(long n) {
    long done = 0, s0 = stepno, launches = 0;
    int c = cur_;
    while (done < n) {
        const int K = (int)std::min<long>(n - done, 64);
        const std::vector<Iter> its = async_chunk(K, s0);
        chunk_graph(its, c);
        launches += graph_kernels_[std::make_pair(its, c)];
        s0 += K;
        c ^= K & 1;
        done += K;
    }
    return launches;
}

template <class T>
void Engine<T>::step_async(long n) {
    consume_staged();
    // Benchmark path: whole graphs of 64 steps, no host round trip; the
    // renormalisation pattern is fixed per graph.  The host clock advances
    // optimistically; each chunk's error word is copied out behind it, so
    // sync() can roll t / stepno / cur_ back to the last completed step.
    long done = 0;
    while (done < n) {
        const int K = (int)std::min<long>(n - done, 64);
        const std::vector<Iter> its = async_chunk(K, stepno);
        if ((int)pending_.size() == kMaxPending) sync();
        run_chunk(its, cur_);
        last_async_K_ = K;
        ck(cudaMemcpyAsync(h_perr_ + pending_.size(), err_, sizeof(int), cudaMemcpyDeviceToHost, stream_), "d2h");
        pending_.push_back(Pending{K, stepno, t, cur_});
        for (int i = 0; i < K; ++i) {
            t += st_.dt;
            stepno += 1;
            cur_ ^= 1;
        }
        done += K;
    }
}

template <class T>
void Engine<T>::sync() {
    ck(cudaMemcpyAsync(h_err_, err_, sizeof(int), cudaMemcpyDeviceToHost, stream_), "d2h");
    ck(cudaStreamSynchronize(stream_), "sync");
    std::vector<Pending> pend;
    pend.swap(pending_);
    if (*h_err_) {
        cudaMemsetAsync(err_, 0, sizeof(int), stream_);
        // the first chunk whose error word is set failed at iteration err - 1;
        // later chunks halted on the device (the word is never cleared in between)
        for (size_t c = 0; c < pend.size(); ++c) {
            if (!h_perr_[c]) continue;
            const Pending& p = pend[c];
            const int ok = std::min(h_perr_[c] - 1, p.K);
            t = p.t;
            for (int i = 0; i < ok; ++i) t += st_.dt;   // same accumulation as step()
            stepno = p.stepno + ok;
            cur_ = p.cur ^ (ok & 1);
            break;
        }
        throw Error(MFD_ENONFINITE, "eulerUpdate: non-finite magnetization after step (time step too large?)");
    }
}

template <class T>
double Engine<T>::sync_torque() {
    sync();
    if (last_async_K_ <= 0) throw Error(MFD_EINVAL, "sync_torque: no asynchronous step has run");
    unsigned long long bits = 0;
    ck(cudaMemcpy(&bits, torque_ + last_async_K_ - 1, sizeof bits, cudaMemcpyDeviceToHost), "d2h");
    return torque_of(bits);
}

template <class T>
mfd_sample Engine<T>::make_sample(const double s[8], double torque) const {
    // reducedMean (state.hpp:113-124) + energies (fields.hpp:127-190) from the device sums
    mfd_sample o{};
    o.step = stepno;
    o.t = t;
    const double sc = 1.0 / (mat_.Ms * ((double)grid_.nx * grid_.ny * grid_.nz));   // global N
    o.m[0] = s[0] * sc;
    o.m[1] = s[1] * sc;
    o.m[2] = s[2] * sc;
    const double V = lp_.dV;
    o.e_exchange = (terms_.exchange && mat_.A > 0) ? s[3] * (mat_.A * V / (mat_.Ms * mat_.Ms)) : 0.0;
    o.e_anisotropy = (terms_.anisotropy && mat_.Ku != 0) ? s[4] * (mat_.Ku * V) : 0.0;
    o.e_demag = terms_.demag ? s[5] * (-0.5 * kMu0 * V) : 0.0;
    const bool zee = terms_.zeeman && (terms_.h_ext[0] != 0 || terms_.h_ext[1] != 0 || terms_.h_ext[2] != 0);
    o.e_zeeman = zee ? s[6] * (-kMu0 * V) : 0.0;
    o.e_total = o.e_exchange + o.e_anisotropy + o.e_demag + o.e_zeeman;
    o.torque_deg_per_ns = torque;
    return o;
}

template <class T>
mfd_sample Engine<T>::sample_now() {
    double s[8], tq;
    eval(0, true, tq, s);
    return make_sample(s, tq);
}

// dynamics::relax (dynamics.hpp:157-198) in graph chunks.  Iteration i of a
// chunk skips itself on the device once iteration i-1 met the torque
// criterion, so the stop step is exactly the reference's; sample iterations
// (iter % sampleEvery == 0) reduce <m> and the energies inside K5.
template <class T>
bool Engine<T>::relax(mfd_sample_cb cb, void* user) {
    consume_staged();
    if (!(st_.dt > 0)) throw Error(MFD_EINVAL, "StepperConfig: dt must be > 0");
    const long startStep = stepno;
    long iter = 0;
    const long sampleEvery = st_.sample_every > 0 ? st_.sample_every : 1;
    std::vector<double> tq;
    while (true) {
        if (iter >= st_.max_steps) {
            // exhausted: evaluate, sample, stop (converged if the torque is within tolerance)
            double s[8], torque;
            eval(0, true, torque, s);
            mfd_sample smp = make_sample(s, torque);
            if (cb) cb(&smp, user);
            return torque <= st_.torque_tol_deg_per_ns;
        }
        const int K = (int)std::min<long>(st_.max_steps - iter, std::min<long>(kMaxChunk, 128));
        std::vector<Iter> its(K);
        for (int i = 0; i < K; ++i) {
            its[i].slot = i;
            its[i].check_prev = 1;
            its[i].sums = ((iter + i) % sampleEvery) == 0;
            its[i].renorm = ((stepno + i + 1 - startStep) % st_.renorm_every) == 0;   // dynamics.hpp:192
        }
        run_chunk(its, cur_);
        int err = 0;
        fetch_chunk(K, tq, err);
        for (int i = 0; i < K; ++i) {
            const bool converged = tq[i] <= st_.torque_tol_deg_per_ns;
            if (converged) {
                double s[8], torque;
                eval(0, true, torque, s);        // same state, same H: the iteration's sample
                mfd_sample smp = make_sample(s, torque);
                if (cb) cb(&smp, user);
                return true;
            }
            if (its[i].sums && cb) {
                mfd_sample smp = make_sample(h_sums_ + 8 * i, tq[i]);
                cb(&smp, user);
            }
            if (err && i == err - 1)
                throw Error(MFD_ENONFINITE, "eulerUpdate: non-finite magnetization after step (time step too large?)");
            t += st_.dt;
            stepno += 1;
            cur_ ^= 1;
        }
        iter += K;
    }
}

// Test hook: run the pipeline up to K<stage> on the current M and copy the
// intermediate spectrum (A after K1/K4, B after K2/K3) out as interleaved
// fp64 (re, im), pitch Hp included.
template <class T>
void Engine<T>::debug_stage(int stage, double* out) {
    if (!terms_.demag) throw Error(MFD_ELOGIC, "lastDemagField: demag term is disabled");
    if (stage < 1 || stage > 4) throw Error(MFD_EINVAL, "debug_stage: stage must be 1..4");
    Iter it;
    it.update = 0;
    stop_after_ = stage;
    try {
        enqueue(it, cur_);
    } catch (...) {
        stop_after_ = 0;
        throw;
    }
    stop_after_ = 0;
    ck(cudaStreamSynchronize(stream_), "debug sync");
    const bool isA = stage == 1 || stage == 4;
    const long long cnt = isA ? 3LL * geo_.ny * geo_.nz * geo_.Hp : 3LL * geo_.nz * Py_ * geo_.Hp;
    std::vector<C2<T>> h(cnt);
    ck(cudaMemcpy(h.data(), isA ? A_ : B_, cnt * sizeof(C2<T>), cudaMemcpyDeviceToHost), "debug d2h");
    for (long long i = 0; i < cnt; ++i) {
        out[2 * i] = h[i].x;
        out[2 * i + 1] = h[i].y;
    }
}

template <class T>
void Engine<T>::timing(double ms[7]) {
    consume_staged();
    // One real Simulation::step with an event after every pass (advances the state).
    // The pass boundaries are event-record nodes of a captured one-iteration
    // graph, so the passes run exactly as inside the step graphs.
    cudaEvent_t ev[6];
    for (auto& e : ev) ck(cudaEventCreate(&e), "event");
    Iter it;
    it.update = 1;
    it.renorm = ((stepno + 1) % st_.renorm_every) == 0;
    cudaGraph_t g;
    ck(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal), "capture");
    cudaMemsetAsync(torque_, 0, sizeof(unsigned long long), stream_);
    cudaMemsetAsync(ticket_, 0, sizeof(unsigned int), stream_);
    enqueue(it, cur_, true, ev);
    ck(cudaStreamEndCapture(stream_, &g), "end capture");
    cudaGraphExec_t ex;
    ck(cudaGraphInstantiate(&ex, g, 0), "graph instantiate");
    cudaGraphDestroy(g);
    const cudaError_t le = cudaGraphLaunch(ex, stream_);
    cudaGraphExecDestroy(ex);
    ck(le, "graph launch");
    std::vector<double> tq;
    int err = 0;
    fetch_chunk(1, tq, err);
    if (err) throw Error(MFD_ENONFINITE, "eulerUpdate: non-finite magnetization after step (time step too large?)");
    t += st_.dt;
    stepno += 1;
    cur_ ^= 1;
    for (int q = 0; q < 5; ++q) {
        float f = 0;
        ck(cudaEventElapsedTime(&f, ev[q], ev[q + 1]), "event time");
        ms[q] = f;
    }
    float tot = 0;
    ck(cudaEventElapsedTime(&tot, ev[0], ev[5]), "event time");
    ms[5] = tot;
    ms[6] = tq[0];   // the step's pre-step max torque (deg/ns), as Simulation::step returns it
    for (auto& e : ev) cudaEventDestroy(e);
}

// Algorithmic HBM bytes per step, 5-pass model.
template <class T>
double Engine<T>::model_bytes() const {
    const double s = sizeof(T), c = 2 * s, N = (double)geo_.ncell;
    if (!terms_.demag) return 3 * N * s * 2 + 6 * N * s;   // read M (7-pt, cached) + write M
    const double Hx = geo_.Hx, ny = geo_.ny, nz = geo_.nz;
    const double k1 = 3 * N * s + 3 * Hx * ny * nz * c;
    const double k2 = 3 * Hx * ny * nz * c + 3 * Hx * Py_ * nz * c;
    const double k3 = 2 * (3 * Hx * Py_ * nz * c) + 6 * Hx * Hy_ * Hz_ * s;
    const double k4 = k2;
    const double k5 = 3 * Hx * ny * nz * c + 3 * N * s + 3 * N * s;
    return k1 + k2 + k3 + k4 + k5;
}

} // namespace mfd
