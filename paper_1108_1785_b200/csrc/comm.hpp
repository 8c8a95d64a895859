// comm.hpp — the collectives of the multi-GPU combine, inside
// the library: the two rounds of the exact median (round 1: sums / coarse
// SUM, min MIN, max MAX; round 2: fine SUM) and, in per-host mode, the
// all-gather of the ranks' (site, host) keys.
//
// Two implementations behind one interface:
//  * NCCL (libnccl.so.2, dlopen'ed on first use, so libgnetmon.so carries no
//    hard NCCL dependency): per process (ncclCommInitRank from a unique id
//    the caller distributes) or a clique of devices driven by one process
//    (ncclCommInitAll). Collectives are enqueued on the context's stream, so
//    the combine is stream-ordered after K2 and before K3a/K2b/K3b.
//  * Loopback: N contexts of one process (possibly on one device) exchange
//    through host memory under a barrier. A test hook: it runs the exact
//    orchestration of the NCCL path with two or more ranks on a single-GPU
//    box (NCCL refuses two ranks on one device).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace gnm {

enum class DType { U32, U64, F64 };
enum class RedOp { Sum, Min, Max };

struct CommError : std::runtime_error {
    explicit CommError(const std::string& m) : std::runtime_error(m) {}
};

class Comm {
public:
    virtual ~Comm() = default;
    virtual int nranks() const = 0;
    virtual int rank() const = 0;
    virtual const char* kind() const = 0;
    // Collectives between group_start/group_end are issued as one fused NCCL
    // group (one launch, one synchronisation) where the backend supports it.
    virtual void group_start() {}
    virtual void group_end() {}
    // In place: buf[count] <- op over every rank's buf (device memory).
    virtual void all_reduce(void* buf, size_t count, DType t, RedOp op, cudaStream_t s) = 0;
    // recv[nranks * bytes] <- every rank's send[bytes], rank-major.
    virtual void all_gather(const void* send, void* recv, size_t bytes, cudaStream_t s) = 0;
    // True when the collectives may be captured into a CUDA graph.
    virtual bool capturable() const = 0;
    // Abort every pending and future collective of this communicator (and,
    // for a clique, let the other ranks' waits fail instead of hanging): one
    // rank of a group failing must not leave the others blocked forever.
    // The communicator is unusable afterwards.
    virtual void abort() = 0;
};

constexpr size_t kUniqueIdBytes = 128; // sizeof(ncclUniqueId)

// ncclGetUniqueId (rank 0 of a per-process group; the caller broadcasts it).
void nccl_unique_id(unsigned char out[kUniqueIdBytes]);
// One rank of a per-process group (the current device is the rank's device).
std::unique_ptr<Comm> nccl_comm(int nranks, int rank, const unsigned char id[kUniqueIdBytes]);
// A clique over `devices`, all driven by this process (ncclCommInitAll).
std::vector<std::unique_ptr<Comm>> nccl_clique(const int* devices, int n);
// N loopback ranks of this process (see the file comment).
std::vector<std::unique_ptr<Comm>> loopback_clique(int n);

} // namespace gnm
