// Host-staged transport of the z-slab decomposition through a shared-memory
// file: the test harness of the one-process-per-GPU engine path on a single
// B200 (NCCL refuses two ranks on one device, and kernels of different
// processes that wait on each other may never be co-resident).
//
// Every exchange is enqueued on the engine's stream like the NCCL calls, so it
// is captured into the step graphs: device -> host copies into this rank's
// slots of the mapped file (registered with cudaHostRegister), a host-function
// node that meets the other ranks at a process-shared barrier, host -> device
// copies out of the peers' slots, and a second barrier before the slots are
// reused.  Reductions combine the ranks' slots in rank order inside the
// barrier's host function.  No kernel waits on another process: only the
// host callbacks block.  A barrier that waits longer than MFD_SHM_TIMEOUT
// seconds (default 120) aborts the process with a message (a test-only
// transport: a lost peer must not hang the GPU box).
#include <fcntl.h>
#include <sched.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <deque>
#include <string>

#include "engine.cuh"

namespace mfd {

namespace {

struct ShmHeader {
    std::atomic<int> count;
    std::atomic<int> gen;
    std::atomic<int> fail;
};
static_assert(std::atomic<int>::is_always_lock_free, "process-shared atomics must be lock free");

class ShmTransport;

// One enqueued host step (stable address: the captured graphs keep pointing at it).
struct HostOp {
    ShmTransport* tr;
    int kind;        // 0 barrier, 1 barrier + max u64, 2 barrier + max i32, 3 barrier + sum f64
    int n;           // reduction length
};

class ShmTransport final : public Transport {
public:
    ShmTransport(const unsigned char id[128], int rank, int world) : rank_(rank), world_(world) {
        char hex[33];
        for (int i = 0; i < 16; ++i) snprintf(hex + 2 * i, 3, "%02x", id[i]);
        const char* dir = getenv("MFD_SHM_DIR");
        path_ = std::string(dir ? dir : (access("/dev/shm", W_OK) == 0 ? "/dev/shm" : "/tmp")) + "/mfd_shm_" + hex;
        if (const char* t = getenv("MFD_SHM_TIMEOUT")) timeout_s_ = atof(t);
        fd_ = open(path_.c_str(), O_RDWR | O_CREAT, 0600);
        if (fd_ < 0) throw Error(MFD_ENCCL, "shm transport: cannot open " + path_);
        // every rank extends the file to the same fixed size (never shrinks it)
        cap_ = (size_t)(getenv("MFD_SHM_MB") ? atol(getenv("MFD_SHM_MB")) : 64) << 20;
        struct stat st{};
        if (fstat(fd_, &st) != 0 || ((size_t)st.st_size < cap_ && ftruncate(fd_, (off_t)cap_) != 0))
            throw Error(MFD_ENCCL, "shm transport: cannot size " + path_);
        base_ = (unsigned char*)mmap(nullptr, cap_, PROT_READ | PROT_WRITE, MAP_SHARED, fd_, 0);
        if (base_ == MAP_FAILED) throw Error(MFD_ENCCL, "shm transport: mmap failed");
        hdr_ = reinterpret_cast<ShmHeader*>(base_);
    }
    ~ShmTransport() override {
        if (registered_) cudaHostUnregister(data_);
        if (base_ && base_ != MAP_FAILED) munmap(base_, cap_);
        if (fd_ >= 0) close(fd_);
        unlink(path_.c_str());   // the last rank out removes the name; the others' mappings stay valid
    }

    void reserve(size_t blk, size_t plane) override {
        blk_ = blk;
        plane_ = plane;
        // layout after the 4 KB header: a2a slots [world][world][blk], halo slots
        // [world][2][3][plane], scalar slots [world][kScal] doubles, results [world][kScal]
        a2a_off_ = 0;
        halo_off_ = a2a_off_ + (size_t)world_ * world_ * blk;
        scal_off_ = halo_off_ + (size_t)world_ * 6 * plane;
        res_off_ = scal_off_ + (size_t)world_ * kScal * 8;
        const size_t need = res_off_ + (size_t)world_ * kScal * 8;
        if (4096 + need > cap_)
            throw Error(MFD_ENCCL, "shm transport: " + std::to_string((4096 + need) >> 20) +
                                       " MB needed, raise MFD_SHM_MB (now " + std::to_string(cap_ >> 20) + ")");
        data_ = base_ + 4096;
        ck(cudaHostRegister(data_, need, cudaHostRegisterDefault), "cudaHostRegister (shm transport)");
        registered_ = true;
    }

    void alltoall(const void* send, void* recv, size_t blk, size_t stride, cudaStream_t s) override {
        const char* sp = static_cast<const char*>(send);
        char* rp = static_cast<char*>(recv);
        for (int p = 0; p < world_; ++p) {
            if (p == rank_) {
                ck(cudaMemcpyAsync(rp + p * stride, sp + p * stride, blk, cudaMemcpyDeviceToDevice, s), "self block");
                continue;
            }
            ck(cudaMemcpyAsync(slot(rank_, p), sp + p * stride, blk, cudaMemcpyDeviceToHost, s), "d2h");
        }
        host(s, 0, 0);
        for (int q = 0; q < world_; ++q)
            if (q != rank_) ck(cudaMemcpyAsync(rp + q * stride, slot(q, rank_), blk, cudaMemcpyHostToDevice, s), "h2d");
        host(s, 0, 0);
    }
    void halo(const void* m, size_t comp_stride, size_t plane, int nzl, void* lo, void* hi, cudaStream_t s) override {
        const char* b = static_cast<const char*>(m);
        for (int c = 0; c < 3; ++c) {
            ck(cudaMemcpyAsync(hslot(rank_, 0, c), b + c * comp_stride, plane, cudaMemcpyDeviceToHost, s), "d2h");
            ck(cudaMemcpyAsync(hslot(rank_, 1, c), b + c * comp_stride + (size_t)(nzl - 1) * plane, plane,
                               cudaMemcpyDeviceToHost, s), "d2h");
        }
        host(s, 0, 0);
        for (int c = 0; c < 3; ++c) {
            if (rank_ > 0)   // the lower neighbour's top plane
                ck(cudaMemcpyAsync(static_cast<char*>(lo) + c * plane, hslot(rank_ - 1, 1, c), plane,
                                   cudaMemcpyHostToDevice, s), "h2d");
            if (rank_ < world_ - 1)   // the upper neighbour's bottom plane
                ck(cudaMemcpyAsync(static_cast<char*>(hi) + c * plane, hslot(rank_ + 1, 0, c), plane,
                                   cudaMemcpyHostToDevice, s), "h2d");
        }
        host(s, 0, 0);
    }
    void allreduce_max_u64(unsigned long long* p, int n, cudaStream_t s) override { reduce(p, n, 8, 1, s); }
    void allreduce_max_i32(int* p, int n, cudaStream_t s) override { reduce(p, n, 4, 2, s); }
    void allreduce_sum_f64(double* p, int n, cudaStream_t s) override { reduce(p, n, 8, 3, s); }
    void barrier(cudaStream_t s) override {
        host(s, 0, 0);
        ck(cudaStreamSynchronize(s), "barrier");
    }

    // host side (called from the CUDA host-function nodes)
    void run(const HostOp& op) {
        wait_all();
        if (op.kind == 0) return;
        unsigned char* out = data_ + res_off_ + (size_t)rank_ * kScal * 8;
        for (int i = 0; i < op.n; ++i) {
            if (op.kind == 1) {
                unsigned long long v = 0;
                for (int r = 0; r < world_; ++r) {
                    unsigned long long x;
                    std::memcpy(&x, data_ + scal_off_ + ((size_t)r * kScal + i) * 8, 8);
                    v = x > v ? x : v;
                }
                std::memcpy(out + 8 * i, &v, 8);
            } else if (op.kind == 2) {
                int v = 0;
                for (int r = 0; r < world_; ++r) {
                    int x;
                    std::memcpy(&x, data_ + scal_off_ + ((size_t)r * kScal + i) * 8, 4);
                    v = r == 0 || x > v ? x : v;
                }
                std::memcpy(out + 8 * i, &v, 4);
            } else {
                double v = 0;   // rank order: deterministic
                for (int r = 0; r < world_; ++r) {
                    double x;
                    std::memcpy(&x, data_ + scal_off_ + ((size_t)r * kScal + i) * 8, 8);
                    v += x;
                }
                std::memcpy(out + 8 * i, &v, 8);
            }
        }
    }

private:
    static constexpr int kScal = 16;
    static void CUDART_CB host_fn(void* u) {
        const HostOp* op = static_cast<const HostOp*>(u);
        op->tr->run(*op);
    }
    void host(cudaStream_t s, int kind, int n) {
        ops_.push_back(HostOp{this, kind, n});
        ck(cudaLaunchHostFunc(s, host_fn, &ops_.back()), "cudaLaunchHostFunc");
    }
    // reduce n elements of `es` bytes (slots are 8-byte strided)
    void reduce(void* p, int n, int es, int kind, cudaStream_t s) {
        if (n > kScal) throw Error(MFD_EINVAL, "shm transport: reduction too long");
        unsigned char* mine = data_ + scal_off_ + (size_t)rank_ * kScal * 8;
        unsigned char* res = data_ + res_off_ + (size_t)rank_ * kScal * 8;
        for (int i = 0; i < n; ++i)
            ck(cudaMemcpyAsync(mine + 8 * i, static_cast<char*>(p) + (size_t)es * i, es, cudaMemcpyDeviceToHost, s),
               "d2h");
        host(s, kind, n);   // barrier, then combine every rank's slots into res
        for (int i = 0; i < n; ++i)
            ck(cudaMemcpyAsync(static_cast<char*>(p) + (size_t)es * i, res + 8 * i, es, cudaMemcpyHostToDevice, s),
               "h2d");
        host(s, 0, 0);      // nobody rewrites a slot before every rank has combined
    }
    void wait_all() {
        const int g = hdr_->gen.load(std::memory_order_acquire);
        if (hdr_->count.fetch_add(1, std::memory_order_acq_rel) == world_ - 1) {
            hdr_->count.store(0, std::memory_order_relaxed);
            hdr_->gen.fetch_add(1, std::memory_order_release);
            return;
        }
        const auto t0 = std::chrono::steady_clock::now();
        while (hdr_->gen.load(std::memory_order_acquire) == g) {
            if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > timeout_s_) {
                fprintf(stderr, "mfd shm transport: rank %d waited %.0f s at a barrier (peer lost); aborting\n",
                        rank_, timeout_s_);
                fflush(stderr);
                _exit(3);
            }
            sched_yield();
        }
    }
    unsigned char* slot(int from, int to) { return data_ + a2a_off_ + ((size_t)from * world_ + to) * blk_; }
    unsigned char* hslot(int r, int top, int c) { return data_ + halo_off_ + (((size_t)r * 2 + top) * 3 + c) * plane_; }

    int rank_, world_;
    std::string path_;
    int fd_ = -1;
    size_t cap_ = 0;
    unsigned char* base_ = nullptr;
    unsigned char* data_ = nullptr;
    ShmHeader* hdr_ = nullptr;
    bool registered_ = false;
    size_t blk_ = 0, plane_ = 0, a2a_off_ = 0, halo_off_ = 0, scal_off_ = 0, res_off_ = 0;
    double timeout_s_ = 120.0;
    std::deque<HostOp> ops_;
};

} // namespace

Transport* make_shm_transport(const unsigned char id[128], int rank, int world) {
    return new ShmTransport(id, rank, world);
}

} // namespace mfd
