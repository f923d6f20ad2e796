// VirtualGroup<T>: the z-slab decomposition of G ranks run on ONE device.
// Each virtual rank is a full Engine<T> with its own slab, halo, send/receive
// blocks and tensor block; the group performs the halo exchange and the two
// all-to-all transposes with device-to-device copies between the ranks'
// buffers, in exactly the block layout the NCCL transport moves.  All ranks
// share one stream, so the passes run in order without host syncs inside an
// iteration.  This is the correctness harness of the multi-GPU path on a
// single B200 (results must match the one-rank engine); it is not a
// performance mode.
#pragma once
#include "engine.cuh"

namespace mfd {

template <class T>
class VirtualGroup final : public EngineBase {
public:
    VirtualGroup(const mfd_grid& g, const mfd_material& m, const mfd_terms& te, const mfd_stepper& st, int device,
                 int world)
        : grid_(g), mat_(m), terms_(te), st_(st), world_(world) {
        precision = sizeof(T) == 4 ? 32 : 64;
        if (world < 2 || g.nz % world != 0)
            throw Error(MFD_EINVAL, "magfd-b200: nz must be divisible by the number of (virtual) ranks");
        for (int r = 0; r < world; ++r)
            ranks_.push_back(std::make_unique<Engine<T>>(g, m, te, st, device, Slab::of(g.nz, r, world), nullptr));
        stream_ = ranks_[0]->stream_;
        for (int r = 1; r < world; ++r) {
            cudaStreamDestroy(ranks_[r]->stream_);
            ranks_[r]->stream_ = stream_;    // one in-order stream for the whole group
        }
        // the group owns the stream: the destructor detaches it from every rank first
        plane_ = (long long)g.nx * g.ny;
        ncell = plane_ * g.nz;
    }
    ~VirtualGroup() override {
        for (auto& e : ranks_) e->stream_ = nullptr;
        ranks_.clear();
        if (stream_) cudaStreamDestroy(stream_);
    }

    void set_m(const double* x, const double* y, const double* z) override {
        for (auto& e : ranks_) {
            const long long o = e->slab_.k0 * plane_;
            e->set_m(x + o, y + o, z + o);
        }
    }
    void set_m32(const float* x, const float* y, const float* z) override {
        for (auto& e : ranks_) {
            const long long o = e->slab_.k0 * plane_;
            e->set_m32(x + o, y + o, z + o);
        }
    }
    void get_m(double* x, double* y, double* z) override {
        for (auto& e : ranks_) {
            const long long o = e->slab_.k0 * plane_;
            e->get_m(x + o, y + o, z + o);
        }
    }
    void get_m32(float* x, float* y, float* z) override {
        for (auto& e : ranks_) {
            const long long o = e->slab_.k0 * plane_;
            e->get_m32(x + o, y + o, z + o);
        }
    }
    void stage_m(const void* x, const void* y, const void* z, int bits) override {
        if (bits == 32) set_m32((const float*)x, (const float*)y, (const float*)z);
        else set_m((const double*)x, (const double*)y, (const double*)z);
    }
    void set_uniform(const double dir[3]) override {
        for (auto& e : ranks_) e->set_uniform(dir);
    }
    void set_vortex(int axis) override {
        for (auto& e : ranks_) e->set_vortex(axis);
    }

    void field(int which, double* x, double* y, double* z) override {
        if (which == 2 && !terms_.demag) throw Error(MFD_ELOGIC, "lastDemagField: demag term is disabled");
        Iter it;
        it.update = 0;
        it.renorm = 0;
        it.write_h = which;
        iterate(it);
        for (auto& e : ranks_) {
            const long long o = e->slab_.k0 * plane_, n = e->geo_.ncell;
            std::vector<T> h(3 * n);
            ck(cudaMemcpy(h.data(), e->H_, 3 * n * sizeof(T), cudaMemcpyDeviceToHost), "d2h");
            for (long long i = 0; i < n; ++i) {
                x[o + i] = h[i];
                y[o + i] = h[i + n];
                z[o + i] = h[i + 2 * n];
            }
        }
    }

    void field32(int which, float* x, float* y, float* z) override {
        const long long n = (long long)grid_.nx * grid_.ny * grid_.nz;
        std::vector<double> a(n), b(n), c(n);
        field(which, a.data(), b.data(), c.data());
        for (long long i = 0; i < n; ++i) {
            x[i] = (float)a[i];
            y[i] = (float)b[i];
            z[i] = (float)c[i];
        }
    }
    void set_stepper(const mfd_stepper& s) override {
        st_ = s;
        for (auto& e : ranks_) e->set_stepper(s);
    }

    void step(long n, double* last, double* all) override {
        for (long s = 0; s < n; ++s) {
            Iter it;
            it.renorm = ((stepno + 1) % st_.renorm_every) == 0;   // sim.hpp:38
            double torque;
            bool bad;
            iterate(it, &torque, &bad);
            if (last) *last = torque;
            if (bad)
                throw Error(MFD_ENONFINITE, "eulerUpdate: non-finite magnetization after step (time step too large?)");
            if (all) all[s] = torque;
            advance();
        }
    }
    void step_async(long n) override { step(n, nullptr, nullptr); }
    long prepare_async(long n) override {
        return n * world_ * (long)ranks_[0]->launches_per_step();   // eager: no graphs
    }
    void sync() override { ck(cudaStreamSynchronize(stream_), "sync"); }
    double sync_torque() override { throw Error(MFD_EINVAL, "sync_torque: single-GPU / one-process-per-GPU contexts only"); }

    bool relax(mfd_sample_cb cb, void* user) override {
        const long startStep = stepno;
        const long every = st_.sample_every > 0 ? st_.sample_every : 1;
        for (long iter = 0;; ++iter) {
            // one pass: torque and sums of the current M, update into the other buffer
            // (only committed by advance() when the iteration does update)
            Iter it;
            it.sums = 1;
            it.renorm = ((stepno + 1 - startStep) % st_.renorm_every) == 0;   // dynamics.hpp:192
            double torque, sums[8];
            bool bad;
            iterate(it, &torque, &bad, sums);
            const bool converged = torque <= st_.torque_tol_deg_per_ns;
            const bool exhausted = iter >= st_.max_steps;
            if (converged || exhausted || iter % every == 0) {
                mfd_sample smp = ranks_[0]->make_sample(sums, torque);
                smp.step = stepno;
                smp.t = t;
                if (cb) cb(&smp, user);
            }
            if (converged) return true;
            if (exhausted) return false;
            if (bad)
                throw Error(MFD_ENONFINITE, "eulerUpdate: non-finite magnetization after step (time step too large?)");
            advance();
        }
    }

    mfd_sample sample_now() override {
        Iter it;
        it.update = 0;
        it.sums = 1;
        double torque, sums[8];
        bool bad;
        iterate(it, &torque, &bad, sums);
        mfd_sample s = ranks_[0]->make_sample(sums, torque);
        s.step = stepno;
        s.t = t;
        return s;
    }
    void timing(double[7]) override { throw Error(MFD_EINVAL, "step timing: single-GPU contexts only"); }
    void set_octant(const double* oct) override {
        for (auto& e : ranks_) e->set_octant(oct);
    }
    void get_octant(double* oct) override { ranks_[0]->get_octant(oct); }
    void get_spectrum(double*) override { throw Error(MFD_EINVAL, "get_spectrum: single-GPU contexts only"); }
    void debug_stage(int, double*) override { throw Error(MFD_EINVAL, "debug_stage: single-GPU contexts only"); }
    void* state_ptr() override { return nullptr; }
    cudaStream_t stream() const override { return stream_; }
    int launches_per_step() const override { return world_ * ranks_[0]->launches_per_step(); }
    double model_bytes() const override { return world_ * ranks_[0]->model_bytes(); }
    long long guard_check() override {
        long long s = 0;
        for (auto& e : ranks_) {
            const long long b = e->guard_check();
            if (b < 0) return -1;
            s += b;
        }
        return s;
    }
    std::string variants() const override {
        std::set<std::string> all;
        for (const auto& e : ranks_) {
            const std::string v = e->variants();
            size_t a = 0, b;
            while ((b = v.find('\n', a)) != std::string::npos) {
                all.insert(v.substr(a, b - a));
                a = b + 1;
            }
        }
        std::string o;
        for (const auto& v : all) o += v + "\n";
        return o;
    }

private:
    void advance() {
        t += st_.dt;
        stepno += 1;
        for (auto& e : ranks_) {
            e->cur_ ^= 1;
            e->t = t;
            e->stepno = stepno;
        }
    }

    // One iteration of all ranks: halo -> A (K1) -> all-to-all -> B (K2-K4) ->
    // all-to-all -> C (K5), then the torque max / error / sums combined on the host.
    void iterate(Iter it, double* torque = nullptr, bool* bad = nullptr, double* sums = nullptr) {
        it.slot = 0;
        it.check_prev = 0;
        const size_t ts = sizeof(T);
        for (auto& e : ranks_) {
            ck(cudaMemsetAsync(e->torque_, 0, sizeof(unsigned long long), stream_), "memset");
            ck(cudaMemsetAsync(e->err_, 0, sizeof(int), stream_), "memset");
            ck(cudaMemsetAsync(e->ticket_, 0, sizeof(unsigned int), stream_), "memset");
        }
        // halo: lo of r <- top plane of r-1, hi of r <- bottom plane of r+1 (per component)
        for (int r = 0; r < world_; ++r) {
            Engine<T>& e = *ranks_[r];
            for (int c = 0; c < 3; ++c) {
                if (r > 0) {
                    Engine<T>& d = *ranks_[r - 1];
                    const T* src = d.M_[d.cur_] + c * d.geo_.ncell + (long long)(d.geo_.nz - 1) * plane_;
                    ck(cudaMemcpyAsync(e.halo_ + c * plane_, src, plane_ * ts, cudaMemcpyDeviceToDevice, stream_), "halo");
                }
                if (r < world_ - 1) {
                    Engine<T>& d = *ranks_[r + 1];
                    const T* src = d.M_[d.cur_] + c * d.geo_.ncell;
                    ck(cudaMemcpyAsync(e.halo_ + 3 * plane_ + c * plane_, src, plane_ * ts, cudaMemcpyDeviceToDevice,
                                       stream_),
                       "halo");
                }
            }
        }
        if (terms_.demag) {
            for (auto& e : ranks_) e->enq_A(it, e->cur_);
            exchange(true);
            for (auto& e : ranks_) e->enq_B(it);
            exchange(false);
            for (auto& e : ranks_) e->enq_C(it, e->cur_);
        } else {
            for (auto& e : ranks_) e->enq_local(it, e->cur_);
        }
        ck(cudaStreamSynchronize(stream_), "iteration");
        double tq = 0, s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        bool any = false;
        for (auto& e : ranks_) {
            unsigned long long bits;
            int err;
            double sm[8];
            ck(cudaMemcpy(&bits, e->torque_, sizeof bits, cudaMemcpyDeviceToHost), "d2h");
            ck(cudaMemcpy(&err, e->err_, sizeof err, cudaMemcpyDeviceToHost), "d2h");
            ck(cudaMemcpy(sm, e->sums_, sizeof sm, cudaMemcpyDeviceToHost), "d2h");
            tq = std::max(tq, e->torque_of(bits));
            any = any || err != 0;
            for (int q = 0; q < 7; ++q) s[q] += sm[q];
        }
        if (torque) *torque = tq;
        if (bad) *bad = any;
        if (sums) std::memcpy(sums, s, sizeof s);
    }

    // forward: send block p of rank r -> receive block r of rank p; backward: the reverse.
    void exchange(bool forward) {
        const size_t blk = ranks_[0]->geo_.SA * sizeof(C2<T>);
        for (int r = 0; r < world_; ++r)
            for (int p = 0; p < world_; ++p) {
                Engine<T>& a = *ranks_[r];
                Engine<T>& b = *ranks_[p];
                const char* src = reinterpret_cast<const char*>(forward ? a.A_ : a.Ar_) + p * blk;
                char* dst = reinterpret_cast<char*>(forward ? b.Ar_ : b.A_) + r * blk;
                ck(cudaMemcpyAsync(dst, src, blk, cudaMemcpyDeviceToDevice, stream_), "all-to-all");
            }
    }

    mfd_grid grid_;
    mfd_material mat_;
    mfd_terms terms_;
    mfd_stepper st_;
    int world_;
    long long plane_ = 0;
    cudaStream_t stream_ = nullptr;
    std::vector<std::unique_ptr<Engine<T>>> ranks_;
};

} // namespace mfd
