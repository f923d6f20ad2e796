// NCCL transport of the z-slab decomposition: one process per GPU, NVLink 5 /
// NVSwitch.  All calls are enqueued on the engine's stream (and captured into
// its step graphs).  The all-to-all is a grouped ncclSend/ncclRecv of
// contiguous blocks (the spectral layout is blocked by destination rank, so no
// pack kernel exists); the halo is six plane-sized send/recv pairs; the
// scalar reductions are ncclAllReduce on the step's torque slot (uint64 max of
// the ordered bit pattern, exact), error word (int max) and sample sums.
#include <nccl.h>

#include <cstring>
#include <string>

#include "engine.cuh"

namespace mfd {

namespace {
inline void nk(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw Error(MFD_ENCCL, std::string(what) + ": " + ncclGetErrorString(r));
}

class NcclTransport final : public Transport {
public:
    NcclTransport(const unsigned char id[128], int rank, int world, int device) : rank_(rank), world_(world) {
        ck(cudaSetDevice(device), "cudaSetDevice");
        ncclUniqueId uid;
        static_assert(sizeof(uid.internal) == 128, "ncclUniqueId size");
        std::memcpy(uid.internal, id, 128);
        nk(ncclCommInitRank(&comm_, world, uid, rank), "ncclCommInitRank");
    }
    ~NcclTransport() override {
        if (comm_) ncclCommDestroy(comm_);
    }
    void alltoall(const void* send, void* recv, size_t blk, size_t stride, cudaStream_t s) override {
        nk(ncclGroupStart(), "ncclGroupStart");
        for (int p = 0; p < world_; ++p) {
            const char* sp = static_cast<const char*>(send) + p * stride;
            char* rp = static_cast<char*>(recv) + p * stride;
            if (p == rank_) {
                ck(cudaMemcpyAsync(rp, sp, blk, cudaMemcpyDeviceToDevice, s), "self block");
                continue;
            }
            nk(ncclSend(sp, blk, ncclInt8, p, comm_, s), "ncclSend");
            nk(ncclRecv(rp, blk, ncclInt8, p, comm_, s), "ncclRecv");
        }
        nk(ncclGroupEnd(), "ncclGroupEnd");
    }
    void halo(const void* m, size_t comp_stride, size_t plane, int nzl, void* lo, void* hi, cudaStream_t s) override {
        const char* base = static_cast<const char*>(m);
        nk(ncclGroupStart(), "ncclGroupStart");
        for (int c = 0; c < 3; ++c) {
            if (rank_ > 0) {   // bottom plane down, neighbour's top plane into lo
                nk(ncclSend(base + c * comp_stride, plane, ncclInt8, rank_ - 1, comm_, s), "ncclSend");
                nk(ncclRecv(static_cast<char*>(lo) + c * plane, plane, ncclInt8, rank_ - 1, comm_, s), "ncclRecv");
            }
            if (rank_ < world_ - 1) {   // top plane up, neighbour's bottom plane into hi
                nk(ncclSend(base + c * comp_stride + (size_t)(nzl - 1) * plane, plane, ncclInt8, rank_ + 1, comm_, s),
                   "ncclSend");
                nk(ncclRecv(static_cast<char*>(hi) + c * plane, plane, ncclInt8, rank_ + 1, comm_, s), "ncclRecv");
            }
        }
        nk(ncclGroupEnd(), "ncclGroupEnd");
    }
    void allreduce_max_u64(unsigned long long* p, int n, cudaStream_t s) override {
        nk(ncclAllReduce(p, p, n, ncclUint64, ncclMax, comm_, s), "ncclAllReduce");
    }
    void allreduce_max_i32(int* p, int n, cudaStream_t s) override {
        nk(ncclAllReduce(p, p, n, ncclInt32, ncclMax, comm_, s), "ncclAllReduce");
    }
    void allreduce_sum_f64(double* p, int n, cudaStream_t s) override {
        nk(ncclAllReduce(p, p, n, ncclFloat64, ncclSum, comm_, s), "ncclAllReduce");
    }
    void barrier(cudaStream_t s) override {
        int* d = nullptr;
        ck(cudaMallocAsync((void**)&d, sizeof(int), s), "alloc");
        ck(cudaMemsetAsync(d, 0, sizeof(int), s), "memset");
        allreduce_max_i32(d, 1, s);
        ck(cudaFreeAsync(d, s), "free");
        ck(cudaStreamSynchronize(s), "barrier");
    }

private:
    ncclComm_t comm_ = nullptr;
    int rank_, world_;
};
} // namespace

Transport* make_nccl_transport(const unsigned char id[128], int rank, int world, int device) {
    return new NcclTransport(id, rank, world, device);
}

void nccl_unique_id(unsigned char id[128]) {
    ncclUniqueId uid;
    nk(ncclGetUniqueId(&uid), "ncclGetUniqueId");
    std::memcpy(id, uid.internal, 128);
}

} // namespace mfd
