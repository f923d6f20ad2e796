// Host side of the B200 engine: one Engine<T> per mfd_ctx.  Owns every device
// buffer, the CUDA stream, the cached CUDA graphs of K-step chunks, and the
// reference-semantics loop control of Simulation<T>::step / dynamics::relax
// (sim.hpp:33-62, dynamics.hpp:157-198).
#pragma once
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <cstdarg>
#include <map>
#include <memory>
#include <set>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/mfd.h"
#include "step_kernels.cuh"
#include "tensor_api.h"

namespace mfd {

struct Error : std::runtime_error {
    mfd_status code;
    Error(mfd_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

// NVTX range (header-only NVTX v3: free unless a profiler injects a tool).
// The per-pass ranges carry the reference's StepTiming phase names
// (backend.hpp:147-148); inside a CUDA graph they mark the capture, and the
// eager / instrumented paths (mfd_last_step_timing) and the chunk launches
// show them at run time.
struct Nvtx {
    explicit Nvtx(const char* name) { nvtxRangePushA(name); }
    ~Nvtx() { nvtxRangePop(); }
    Nvtx(const Nvtx&) = delete;
    Nvtx& operator=(const Nvtx&) = delete;
};

inline void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw Error(MFD_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

constexpr double kPi = 3.14159265358979323846;
constexpr double kMu0 = 4.0e-7 * kPi;                       // constants.hpp:9
constexpr double kRadToDegPerNs = 180.0 / kPi * 1e-9;       // dynamics.hpp:34
constexpr int kMaxL = 2048;
// Fuse the next step's x pass (K1) into K5 inside a graph chunk.
constexpr bool kFuseK1 = true;
// One-kernel K2-K4 for thin / small grids (YZCfg::OK).
constexpr bool kYZSmall = true;
// K2 input through TMA staging (persistent CTAs, next tile in flight).
constexpr bool kK2Tma = true;
// K4 input through a ring of TMA-staged half tiles (persistent CTAs).
constexpr bool kK4Tma = true;
// K3 with one y row per CTA (twice the CTAs per SM) instead of the pair {v, Py-v}.
constexpr bool kK3SingleRow = true;
constexpr long long kFuseK1MaxCells = 4LL << 20;
// L2 prefetch (cp.async.bulk.prefetch) of the x passes' inputs one resident
// wave of CTAs ahead, and of K5's epilogue rows while its FFT runs.
// Bit mask (Geo::pfm): 1 K1 ahead, 2 K5 own M rows, 4 K5 spectrum ahead.
constexpr int kL2PrefetchMask = 1;   // measured: K1 ahead -0.013 ms; the K5 prefetches do not pay

inline int next_pow2(int n) { int p = 1; while (p < n) p <<= 1; return p; }
inline int padded_size(int n) { return next_pow2(2 * n); }  // demag.hpp:24

// Calls f.template operator()<L>() for the power of two L (1..kMaxL).
template <class F>
void with_pow2(int L, F&& f) {
    switch (L) {
        case 1: f.template operator()<1>(); break;
        case 2: f.template operator()<2>(); break;
        case 4: f.template operator()<4>(); break;
        case 8: f.template operator()<8>(); break;
        case 16: f.template operator()<16>(); break;
        case 32: f.template operator()<32>(); break;
        case 64: f.template operator()<64>(); break;
        case 128: f.template operator()<128>(); break;
        case 256: f.template operator()<256>(); break;
        case 512: f.template operator()<512>(); break;
        case 1024: f.template operator()<1024>(); break;
        case 2048: f.template operator()<2048>(); break;
        default: throw Error(MFD_EINVAL, "magfd-b200: unsupported FFT length " + std::to_string(L));
    }
}

template <class T> __global__ void k_ybuf(int Py, int Hy, int* out);

// Collective transport of the z-slab decomposition.
// One implementation per backend; the engine only calls these between its
// passes, on its own stream (so they are captured into the step graphs).
struct Transport {
    virtual ~Transport() = default;
    // Called once by the engine with the largest all-to-all block and halo
    // plane it will move (before any transfer is enqueued).
    virtual void reserve(size_t /*blk_bytes*/, size_t /*plane_bytes*/) {}
    // all-to-all of `world` equal contiguous blocks of blk_bytes, block p at
    // send + p * stride -> rank p, block q of recv (recv + q * stride) <- rank q.
    virtual void alltoall(const void* send, void* recv, size_t blk_bytes, size_t stride, cudaStream_t s) = 0;
    // one-plane halo of the slab: planes 0 / nzl-1 of each component (stride
    // comp_stride bytes, plane_bytes each) go to rank-1 / rank+1; the
    // neighbours' planes land in lo / hi ([3][plane]).
    virtual void halo(const void* m, size_t comp_stride, size_t plane_bytes, int nzl, void* lo, void* hi,
                      cudaStream_t s) = 0;
    virtual void allreduce_max_u64(unsigned long long* p, int n, cudaStream_t s) = 0;
    virtual void allreduce_max_i32(int* p, int n, cudaStream_t s) = 0;
    virtual void allreduce_sum_f64(double* p, int n, cudaStream_t s) = 0;
    virtual void barrier(cudaStream_t s) = 0;
};
// NCCL transport over NVLink/NVSwitch (nccl_transport.cu).
Transport* make_nccl_transport(const unsigned char id[128], int rank, int world, int device);
// Host-staged transport through a shared-memory file (shm_transport.cu): the
// ranks are processes of one host, on one GPU or several.  Test harness of the
// one-process-per-GPU engine path on a single B200 (NCCL refuses two ranks on
// one device); no kernel ever waits on another process.
Transport* make_shm_transport(const unsigned char id[128], int rank, int world);
void nccl_unique_id(unsigned char id[128]);

class EngineBase;
// Factories (defined per precision in engine_f32.cu / engine_f64.cu).
template <class T>
EngineBase* make_engine(const mfd_grid& g, const mfd_material& m, const mfd_terms& te, const mfd_stepper& st,
                        int device, int rank, int world, Transport* tr);
template <class T>
EngineBase* make_virtual_group(const mfd_grid& g, const mfd_material& m, const mfd_terms& te,
                               const mfd_stepper& st, int device, int world);

// Slab of a rank: planes [k0, k0+nzl) of the global nz, x-bin block rank.
struct Slab {
    int rank = 0, world = 1, k0 = 0, nzl = 0;
    static Slab of(int nz, int rank, int world) {
        Slab s;
        s.rank = rank;
        s.world = world;
        s.nzl = nz / world;
        s.k0 = rank * s.nzl;
        return s;
    }
};

// One iteration of the per-step pipeline as enqueued in a graph.
struct Iter {
    int update = 1;
    int renorm = 1;
    int write_h = 0;
    int sums = 0;        // accumulate sample sums into sums slot `slot`
    int check_prev = 0;  // relax: skip if the previous slot converged
    int slot = 0;        // torque / sums slot within the chunk
    bool operator<(const Iter& o) const {
        return std::tie(update, renorm, write_h, sums, check_prev, slot) <
               std::tie(o.update, o.renorm, o.write_h, o.sums, o.check_prev, o.slot);
    }
};

class EngineBase {
public:
    virtual ~EngineBase() = default;
    virtual void set_m(const double*, const double*, const double*) = 0;
    virtual void set_m32(const float*, const float*, const float*) = 0;
    // Queue a new state from host memory on a copy stream (returns at once);
    // the next state-reading call installs it.  f32 / f64 by the pointer type.
    virtual void stage_m(const void* x, const void* y, const void* z, int bits) = 0;
    virtual void get_m(double*, double*, double*) = 0;
    virtual void get_m32(float*, float*, float*) = 0;
    virtual void set_uniform(const double dir[3]) = 0;
    virtual void set_vortex(int axis) = 0;
    virtual void field(int which, double*, double*, double*) = 0;
    virtual void field32(int which, float*, float*, float*) = 0;
    virtual void set_stepper(const mfd_stepper& s) = 0;
    virtual void step(long n, double* last, double* all) = 0;
    virtual void step_async(long n) = 0;
    // Capture (without launching) the graphs the next step_async(n) will use;
    // returns the number of kernel launches those graphs contain.
    virtual long prepare_async(long n) = 0;
    virtual void sync() = 0;
    // sync() + the pre-step max torque (deg/ns) of the last asynchronous step
    virtual double sync_torque() = 0;
    virtual bool relax(mfd_sample_cb cb, void* user) = 0;
    virtual mfd_sample sample_now() = 0;
    virtual void timing(double ms[7]) = 0;
    virtual void set_octant(const double*) = 0;
    virtual void get_octant(double*) = 0;
    virtual void get_spectrum(double*) = 0;
    virtual void debug_stage(int stage, double* out) = 0;
    virtual void* state_ptr() = 0;
    virtual cudaStream_t stream() const = 0;
    virtual int launches_per_step() const = 0;
    virtual double model_bytes() const = 0;
    // Kernel template instantiations enqueued since creation, one per line
    // (test hook: lets the parity tests assert which production variant ran).
    virtual std::string variants() const = 0;
    // Test hook: guard-band bytes overwritten since creation (-1: guards off).
    virtual long long guard_check() = 0;
    double t = 0;
    long stepno = 0;
    long long ncell = 0;
    int precision = 64;
};

template <class T> class VirtualGroup;

template <class T>
class Engine final : public EngineBase {
    friend class VirtualGroup<T>;

public:
    // slab / tr: z-slab of a multi-GPU run (tr = null with world > 1: the
    // passes are orchestrated externally, e.g. by VirtualGroup).
    Engine(const mfd_grid& g, const mfd_material& m, const mfd_terms& te, const mfd_stepper& st, int device,
           Slab slab = Slab{}, Transport* tr = nullptr);
    ~Engine() override;

    void set_m(const double* x, const double* y, const double* z) override;
    void set_m32(const float* x, const float* y, const float* z) override;
    void stage_m(const void* x, const void* y, const void* z, int bits) override;
    void get_m(double* x, double* y, double* z) override;
    void get_m32(float* x, float* y, float* z) override;
    void set_uniform(const double dir[3]) override;
    void set_vortex(int axis) override;
    void field(int which, double* x, double* y, double* z) override;
    void field32(int which, float* x, float* y, float* z) override;
    void set_stepper(const mfd_stepper& s) override;
    void step(long n, double* last, double* all) override;
    void step_async(long n) override;
    long prepare_async(long n) override;
    void sync() override;
    double sync_torque() override;
    int last_async_K_ = 0;                     // steps in the last step_async chunk
    bool relax(mfd_sample_cb cb, void* user) override;
    mfd_sample sample_now() override;
    void timing(double ms[7]) override;
    void set_octant(const double* oct) override;
    void get_octant(double* oct) override;
    void get_spectrum(double* out) override;
    void debug_stage(int stage, double* out) override;
    void* state_ptr() override { return M_[cur_]; }
    cudaStream_t stream() const override { return stream_; }
    int launches_per_step() const override { return terms_.demag ? 5 : 1; }
    double model_bytes() const override;
    std::string variants() const override {
        std::string o;
        for (const auto& v : launched_) o += v + "\n";
        return o;
    }
    long long guard_check() override;

private:
    void note(const char* fmt, ...) {
        char b[256];
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(b, sizeof b, fmt, ap);
        va_end(ap);
        launched_.insert(b);
    }
    static constexpr const char* tn() { return sizeof(T) == 4 ? "f32" : "f64"; }
    std::set<std::string> launched_;
    void init();
    void release();
    void* dalloc(size_t bytes);
    struct Alloc { void* base; size_t bytes; };
    std::vector<Alloc> allocs_;              // every persistent device buffer
    bool guards_ = false;                    // MFD_GUARD: guard bands around each buffer
    static constexpr size_t kGuard = 4096;
    void build_tensor(const double* host_octant);
    void enqueue(const Iter& it, int cur, bool events = false, cudaEvent_t* ev = nullptr, bool skip_k1 = false,
                 bool fwd = false);
    // pass groups of one iteration: A = K1,K2 (slab -> send blocks), B = K3
    // (receive blocks, full z), C = K4,K5 (send blocks -> slab + LLG)
    void enq_A(const Iter& it, int cur, cudaEvent_t* ev = nullptr, bool skip_k1 = false);
    void enq_B(const Iter& it, cudaEvent_t* ev = nullptr);
    void enq_C(const Iter& it, int cur, cudaEvent_t* ev = nullptr, bool fwd = false);
    void enq_local(const Iter& it, int cur);
    void enq_K2(const Ctl& ctl, int comp0, int ncomp);
    void enq_K3(const Ctl& ctl);
    void enq_K4(const Ctl& ctl, int comp0, int ncomp);
    Ctl make_ctl(const Iter& it) const;
    StepIO make_io(const Iter& it) const;
    Halo<T> halo_ptrs() const;
    void run_chunk(const std::vector<Iter>& its, int cur);
    cudaGraphExec_t chunk_graph(const std::vector<Iter>& its, int cur);
    std::vector<Iter> async_chunk(int K, long step0) const;
    void fetch_chunk(int n, std::vector<double>& torque, int& err);
    double torque_of(unsigned long long bits) const;
    mfd_sample make_sample(const double sums[8], double torque) const;
    void eval(int write_h, bool sums, double& torque, double sum_out[8]);
    // staged states (stage_m): device buffers filled on copy_stream_, installed
    // into M_[cur_] by consume_staged() at the next state-reading call
    void consume_staged();
    cudaStream_t copy_stream_ = nullptr;
    T* Mst_[2] = {nullptr, nullptr};
    cudaEvent_t st_ready_[2] = {}, st_free_[2] = {};
    int st_next_ = 0;
    std::vector<int> st_pending_;              // FIFO of filled slots
    void ensure_stage() {
        if (!h_stage_) ck(cudaMallocHost((void**)&h_stage_, 3 * geo_.ncell * sizeof(T)), "host alloc");
    }

    mfd_grid grid_;
    mfd_material mat_;
    mfd_terms terms_;
    mfd_stepper st_;
    int device_;
    Geo geo_{};
    LocalParams<T> lp_{};
    T scale_{};
    int Py_ = 2, Pz_ = 2, Hy_ = 2, Hz_ = 2;

    Slab slab_;
    Transport* tr_ = nullptr;           // owned
    cudaStream_t stream_ = nullptr;
    cudaStream_t cstream_ = nullptr;     // transposes / halo of a multi-process run
    cudaEvent_t xev_[9] = {};            // fork / join events of the transpose pipeline
    T* M_[2] = {nullptr, nullptr};
    int cur_ = 0;
    T* H_ = nullptr;                     // H_eff / H_demag output
    T* halo_ = nullptr;                  // [2][3][ny][nx]: lo, hi planes (world > 1)
    C2<T>* A_ = nullptr;
    C2<T>* B_ = nullptr;                 // send-side blocks (== receive side on one GPU)
    C2<T>* Ar_ = nullptr;                // receive-side A blocks (world > 1; = A_ on one GPU)
    T* Kt_ = nullptr;
    C2<T>* tw_ = nullptr;
    int* ybuf_ = nullptr;
    int* err_ = nullptr;
    unsigned long long* torque_ = nullptr;
    double* sums_ = nullptr;             // [kMaxChunk][8]
    double* partials_ = nullptr;
    unsigned int* ticket_ = nullptr;
    unsigned long long* h_torque_ = nullptr;   // pinned
    double* h_sums_ = nullptr;                 // pinned
    int* h_err_ = nullptr;                     // pinned
    // step_async chunks not yet checked by sync(): the error word of chunk c
    // lands in h_perr_[c] behind the chunk's graph
    struct Pending { int K; long stepno; double t; int cur; };
    static constexpr int kMaxPending = 1024;
    std::vector<Pending> pending_;
    int* h_perr_ = nullptr;                    // pinned [kMaxPending]
    T* h_stage_ = nullptr;                     // pinned 3N staging
    long long k5_blocks_ = 1;
    bool small_x_ = false;                     // few rows: small-CTA variants of K1 / K5
    int stop_after_ = 0;                       // debug_stage: stop the pipeline after K<n>
    bool fuse_k1_ = false;                     // K5 also runs the next step's K1 (within a graph chunk)
    bool yz_small_ = false;                    // K2-K4 as one kernel (k_fft_yz_small)
    bool k2_tma_ = false;                      // K2 with TMA-staged input (k_fft_y_fwd_tma)
    int k2_grid_ = 0, k2_box_ = 0;
    CUtensorMap tmA_{};                        // A as [3 nz ny] x [Hp] 8-byte elements
    bool k4_tma_ = false;                      // K4 with TMA-staged input (k_fft_y_inv_tma)
    bool k3_srow_ = false;                     // K3 one y row per CTA (Z2Cfg SROW)
    int k4_grid_ = 0;
    CUtensorMap tmB_{};                        // B as [G 3 nz Py] x [Wb] 8-byte elements
    bool yz() const { return yz_small_ && stop_after_ == 0; }   // debug_stage needs the separate passes
    // f.template operator()<Py, Pz>() when the single-kernel y-z pass exists for this grid
    template <class F>
    void with_yz(F&& f) const {
        with_pow2(Py_, [&]<int LY>() {
            with_pow2(Pz_, [&]<int LZ>() {
                if constexpr (LZ <= 16 && YZCfg<T, LY, LZ>::OK) f.template operator()<LY, LZ>();
            });
        });
    }
    static constexpr int kMaxChunk = 256;

    std::map<std::pair<std::vector<Iter>, int>, cudaGraphExec_t> graphs_;
    std::map<std::pair<std::vector<Iter>, int>, int> graph_kernels_;   // kernel nodes per cached graph
};

} // namespace mfd
