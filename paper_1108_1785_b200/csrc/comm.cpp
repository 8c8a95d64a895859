// comm.cpp — NCCL (dlopen'ed) and loopback collectives for the in-library
// multi-GPU combine. See comm.hpp.
#include "comm.hpp"

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstring>
#include <limits>
#include <mutex>

namespace gnm {

namespace {

// ---- NCCL, resolved at first use ----------------------------------------------

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    std::string error;
};

const NcclApi& nccl() {
    static NcclApi api = [] {
        NcclApi a;
        // A process that already mapped an NCCL (e.g. torch's bundled
        // libnccl.so.2) gets that one: same soname, same ABI.
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            a.error = std::string("libnccl.so.2 not loadable: ") + dlerror();
            return a;
        }
        auto sym = [&](auto& fp, const char* name) {
            fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, name));
            if (!fp && a.error.empty()) a.error = std::string("NCCL symbol missing: ") + name;
        };
        sym(a.GetUniqueId, "ncclGetUniqueId");
        sym(a.CommInitRank, "ncclCommInitRank");
        sym(a.CommInitAll, "ncclCommInitAll");
        sym(a.CommDestroy, "ncclCommDestroy");
        sym(a.CommAbort, "ncclCommAbort");
        sym(a.AllReduce, "ncclAllReduce");
        sym(a.AllGather, "ncclAllGather");
        sym(a.GroupStart, "ncclGroupStart");
        sym(a.GroupEnd, "ncclGroupEnd");
        sym(a.GetErrorString, "ncclGetErrorString");
        return a;
    }();
    if (!api.error.empty()) throw CommError(api.error);
    return api;
}

void nck(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw CommError(std::string(what) + ": " + nccl().GetErrorString(r));
}

ncclDataType_t nccl_type(DType t) {
    switch (t) {
    case DType::U32: return ncclUint32;
    case DType::U64: return ncclUint64;
    default: return ncclFloat64;
    }
}

ncclRedOp_t nccl_op(RedOp op) {
    switch (op) {
    case RedOp::Sum: return ncclSum;
    case RedOp::Min: return ncclMin;
    default: return ncclMax;
    }
}

class NcclComm final : public Comm {
public:
    NcclComm(ncclComm_t c, int n, int r) : comm_(c), n_(n), r_(r) {}
    ~NcclComm() override {
        if (ncclComm_t c = comm_.load()) nccl().CommDestroy(c);
    }
    void abort() override { // may run on another rank's thread
        if (ncclComm_t c = comm_.exchange(nullptr)) nccl().CommAbort(c);
    }
    int nranks() const override { return n_; }
    int rank() const override { return r_; }
    const char* kind() const override { return "nccl"; }
    void group_start() override { nck(nccl().GroupStart(), "ncclGroupStart"); }
    void group_end() override { nck(nccl().GroupEnd(), "ncclGroupEnd"); }
    void all_reduce(void* buf, size_t count, DType t, RedOp op, cudaStream_t s) override {
        live();
        nck(nccl().AllReduce(buf, buf, count, nccl_type(t), nccl_op(op), comm_.load(), s), "ncclAllReduce");
    }
    void all_gather(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
        live();
        nck(nccl().AllGather(send, recv, bytes, ncclUint8, comm_.load(), s), "ncclAllGather");
    }
    void live() const {
        if (!comm_) throw CommError("NCCL communicator was aborted");
    }
    bool capturable() const override { return true; }

private:
    std::atomic<ncclComm_t> comm_;
    int n_, r_;
};

// ---- loopback: host-staged exchange under a barrier ----------------------------

struct LoopShared {
    explicit LoopShared(int n) : n(n), buf(n) {}
    int n;
    std::mutex m;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t gen = 0;
    std::vector<std::vector<unsigned char>> buf;

    bool poisoned = false; // a rank aborted: every wait fails from now on

    void barrier() {
        std::unique_lock<std::mutex> l(m);
        if (poisoned) throw CommError("loopback group aborted by another rank");
        const uint64_t g = gen;
        if (++arrived == n) {
            arrived = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(l, [&] { return gen != g || poisoned; });
            if (gen == g) throw CommError("loopback group aborted by another rank");
        }
    }
    void poison() {
        std::lock_guard<std::mutex> l(m);
        poisoned = true;
        cv.notify_all();
    }
};

void cck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CommError(std::string(what) + ": " + cudaGetErrorString(e));
}

template <typename T>
void reduce_into(std::vector<unsigned char>& out, const std::vector<std::vector<unsigned char>>& in, size_t count,
                 RedOp op) {
    T* o = reinterpret_cast<T*>(out.data());
    std::memcpy(o, in[0].data(), count * sizeof(T));
    for (size_t r = 1; r < in.size(); ++r) {
        const T* x = reinterpret_cast<const T*>(in[r].data());
        for (size_t i = 0; i < count; ++i) {
            if (op == RedOp::Sum) o[i] += x[i];
            else if (op == RedOp::Min) o[i] = std::min(o[i], x[i]);
            else o[i] = std::max(o[i], x[i]);
        }
    }
}

class LoopComm final : public Comm {
public:
    LoopComm(std::shared_ptr<LoopShared> s, int r) : S_(std::move(s)), r_(r) {}
    int nranks() const override { return S_->n; }
    int rank() const override { return r_; }
    const char* kind() const override { return "loopback"; }
    void all_reduce(void* buf, size_t count, DType t, RedOp op, cudaStream_t s) override {
        const size_t esz = t == DType::U32 ? 4 : 8;
        stage_in(buf, count * esz, s);
        std::vector<unsigned char> out(count * esz);
        if (t == DType::U32) reduce_into<uint32_t>(out, S_->buf, count, op);
        else if (t == DType::U64) reduce_into<uint64_t>(out, S_->buf, count, op);
        else reduce_into<double>(out, S_->buf, count, op);
        stage_out(buf, out, s);
    }
    void all_gather(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
        stage_in(send, bytes, s);
        std::vector<unsigned char> out(bytes * S_->n);
        for (int r = 0; r < S_->n; ++r)
            if (bytes) std::memcpy(out.data() + bytes * r, S_->buf[r].data(), bytes);
        stage_out(recv, out, s);
    }
    bool capturable() const override { return false; }
    void abort() override { S_->poison(); }

private:
    void stage_in(const void* dev, size_t bytes, cudaStream_t s) {
        std::vector<unsigned char>& mine = S_->buf[r_];
        mine.resize(bytes);
        if (bytes) cck(cudaMemcpyAsync(mine.data(), dev, bytes, cudaMemcpyDeviceToHost, s), "loopback D2H");
        cck(cudaStreamSynchronize(s), "loopback sync");
        S_->barrier(); // every rank's contribution is staged
    }
    void stage_out(void* dev, const std::vector<unsigned char>& out, cudaStream_t s) {
        S_->barrier(); // every rank has read the staged contributions
        if (!out.empty())
            cck(cudaMemcpyAsync(dev, out.data(), out.size(), cudaMemcpyHostToDevice, s), "loopback H2D");
        cck(cudaStreamSynchronize(s), "loopback sync");
    }
    std::shared_ptr<LoopShared> S_;
    int r_;
};

} // namespace

void nccl_unique_id(unsigned char out[kUniqueIdBytes]) {
    static_assert(sizeof(ncclUniqueId) == kUniqueIdBytes, "ncclUniqueId size");
    ncclUniqueId id;
    nck(nccl().GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out, &id, kUniqueIdBytes);
}

std::unique_ptr<Comm> nccl_comm(int nranks, int rank, const unsigned char id[kUniqueIdBytes]) {
    ncclUniqueId uid;
    std::memcpy(&uid, id, kUniqueIdBytes);
    ncclComm_t c = nullptr;
    nck(nccl().CommInitRank(&c, nranks, uid, rank), "ncclCommInitRank");
    return std::make_unique<NcclComm>(c, nranks, rank);
}

std::vector<std::unique_ptr<Comm>> nccl_clique(const int* devices, int n) {
    std::vector<ncclComm_t> cs(n);
    nck(nccl().CommInitAll(cs.data(), n, devices), "ncclCommInitAll");
    std::vector<std::unique_ptr<Comm>> out;
    for (int i = 0; i < n; ++i) out.push_back(std::make_unique<NcclComm>(cs[i], n, i));
    return out;
}

std::vector<std::unique_ptr<Comm>> loopback_clique(int n) {
    auto s = std::make_shared<LoopShared>(n);
    std::vector<std::unique_ptr<Comm>> out;
    for (int i = 0; i < n; ++i) out.push_back(std::make_unique<LoopComm>(s, i));
    return out;
}

} // namespace gnm
