// netflow.cu — batched NetFlow v5 ingest on sm_100a.
//
// Collector::ingest_datagram (collector.cpp:101-129) for a whole batch of
// datagrams at once, minus the store and the per-exporter sequence tracker:
//   decode_packet  (netflow.cpp:78-113): header checks in the reference's
//                  order -- shorter than 24 bytes: Truncated; version != 5:
//                  BadVersion; count outside 1..30: BadCount; length !=
//                  24 + 48*count: Truncated -- then big-endian fields;
//   reject rule    (collector.cpp:120-123): d_pkts == 0 || d_octets < d_pkts;
//   resolve_times  (netflow.cpp:150-161): export wall clock minus the
//                  wrap-safe uptime difference, end clamped to start.
// Output: flowmon::FlowRecord rows (64 bytes, netflow.hpp:59-67) in datagram
// order, then record order -- exactly the order the collector appends to the
// FlowStore. Paths are relative to /root/reference/proj/core/src.
//
// Three kernels: N1 validates every datagram and counts its accepted
// records (thread per datagram), N2 turns the counts into output offsets (one
// CTA, exclusive scan), N3 decodes (warp per datagram, lane = record) and
// compacts the accepted records with a ballot.
#include <cuda_runtime.h>

#include <cstdint>

#include "netflow.cuh"

namespace gnm {
namespace {

constexpr uint32_t kHdr = 24, kRec = 48, kMaxRec = 30;

__device__ __forceinline__ uint32_t be16(const uint8_t* p) {
    return static_cast<uint32_t>(p[0]) << 8 | p[1];
}
__device__ __forceinline__ uint32_t be32(const uint8_t* p) {
    return static_cast<uint32_t>(p[0]) << 24 | static_cast<uint32_t>(p[1]) << 16 |
           static_cast<uint32_t>(p[2]) << 8 | p[3];
}

// wrap_diff (netflow.cpp:145-148): a - b modulo 2^32, 0 when "negative".
__device__ __forceinline__ uint32_t wrap_diff(uint32_t a, uint32_t b) {
    const uint32_t d = a - b;
    return d > 0x80000000u ? 0u : d;
}

// Status per datagram: 0 ok, else 1 + CodecError::Kind (BadVersion,
// Truncated, BadCount), as decode_packet checks them.
__device__ __forceinline__ uint32_t check_header(const uint8_t* p, uint64_t len, uint32_t& count) {
    count = 0;
    if (len < kHdr) return 2;
    const uint32_t version = be16(p);
    count = be16(p + 2);
    if (version != 5) return 1;
    if (count == 0 || count > kMaxRec) return 3;
    if (len != kHdr + static_cast<uint64_t>(kRec) * count) return 2;
    return 0;
}

__global__ void __launch_bounds__(256) n1_validate(const uint8_t* __restrict__ d,
                                                   const uint64_t* __restrict__ off, uint64_t n,
                                                   uint32_t* __restrict__ accepted,
                                                   uint8_t* __restrict__ status,
                                                   unsigned long long* __restrict__ stats) {
    uint32_t err = 0, rej = 0, acc = 0;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint8_t* p = d + off[i];
        uint32_t count;
        const uint32_t st = check_header(p, off[i + 1] - off[i], count);
        uint32_t a = 0;
        if (st == 0) {
            for (uint32_t r = 0; r < count; ++r) {
                const uint8_t* q = p + kHdr + kRec * r;
                const uint32_t pkts = be32(q + 16), oct = be32(q + 20);
                a += (pkts != 0 && oct >= pkts);
            }
            rej += count - a;
        } else {
            ++err;
        }
        acc += a;
        accepted[i] = a;
        if (status) status[i] = static_cast<uint8_t>(st);
    }
    err = __reduce_add_sync(0xFFFFFFFFu, err);
    rej = __reduce_add_sync(0xFFFFFFFFu, rej);
    acc = __reduce_add_sync(0xFFFFFFFFu, acc);
    if ((threadIdx.x & 31u) == 0) {
        if (err) atomicAdd(stats + 1, static_cast<unsigned long long>(err));
        if (rej) atomicAdd(stats + 2, static_cast<unsigned long long>(rej));
        if (acc) atomicAdd(stats + 3, static_cast<unsigned long long>(acc));
    }
}

// Exclusive scan of n u32 counts into u64 offsets, one 1024-thread CTA:
// thread t owns the contiguous slice [t*chunk, (t+1)*chunk).
__global__ void __launch_bounds__(1024) n2_scan(const uint32_t* __restrict__ in, uint64_t n,
                                                uint64_t* __restrict__ out,
                                                unsigned long long* __restrict__ total) {
    __shared__ unsigned long long part[1024];
    const uint64_t chunk = (n + blockDim.x - 1) / blockDim.x;
    const uint64_t b = threadIdx.x * chunk, e = min(n, b + chunk);
    unsigned long long s = 0;
    for (uint64_t i = b; i < e; ++i) s += in[i];
    part[threadIdx.x] = s;
    __syncthreads();
    for (uint32_t o = 1; o < blockDim.x; o <<= 1) { // inclusive scan
        const unsigned long long x = threadIdx.x >= o ? part[threadIdx.x - o] : 0ull;
        __syncthreads();
        part[threadIdx.x] += x;
        __syncthreads();
    }
    unsigned long long run = threadIdx.x ? part[threadIdx.x - 1] : 0ull;
    for (uint64_t i = b; i < e; ++i) {
        out[i] = run;
        run += in[i];
    }
    if (threadIdx.x == blockDim.x - 1) *total = part[threadIdx.x];
}

// Warp per datagram; lane r decodes record r (decode_raw_record,
// netflow.cpp:27-50) and resolve_times; accepted lanes are compacted in
// record order.
__global__ void __launch_bounds__(256) n3_decode(const uint8_t* __restrict__ d,
                                                 const uint64_t* __restrict__ off, uint64_t n,
                                                 const uint64_t* __restrict__ base,
                                                 uint8_t* __restrict__ out) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
    for (uint64_t i = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; i < n; i += nwarps) {
        const uint8_t* p = d + off[i];
        uint32_t count;
        if (check_header(p, off[i + 1] - off[i], count) != 0) continue; // warp-uniform
        const uint32_t uptime = be32(p + 4), secs = be32(p + 8), nsecs = be32(p + 12);
        const uint64_t wall = static_cast<uint64_t>(secs) * 1000u + nsecs / 1000000u;
        bool ok = false;
        uint4 w0{}, w1{}, w2{};
        uint64_t start = 0, end = 0;
        if (lane < count) {
            const uint8_t* q = p + kHdr + kRec * lane;
            const uint32_t pkts = be32(q + 16), oct = be32(q + 20);
            ok = pkts != 0 && oct >= pkts;
            const uint32_t first = be32(q + 24), last = be32(q + 28);
            // RawFlowRecord in memory order (netflow.hpp:32-57): u32 src, dst,
            // next_hop; u16 input_if, output_if; u32 d_pkts, d_octets, first,
            // last; u16 src_port, dst_port; u8 pad1, tcp_flags, protocol, tos;
            // u16 src_as, dst_as; u8 src_mask, dst_mask; u16 pad2.
            w0 = make_uint4(be32(q), be32(q + 4), be32(q + 8), be16(q + 12) | be16(q + 14) << 16);
            w1 = make_uint4(pkts, oct, first, last);
            w2 = make_uint4(be16(q + 32) | be16(q + 34) << 16,
                            static_cast<uint32_t>(q[36]) | static_cast<uint32_t>(q[37]) << 8 |
                                static_cast<uint32_t>(q[38]) << 16 | static_cast<uint32_t>(q[39]) << 24,
                            be16(q + 40) | be16(q + 42) << 16,
                            static_cast<uint32_t>(q[44]) | static_cast<uint32_t>(q[45]) << 8 | be16(q + 46) << 16);
            start = wall - wrap_diff(uptime, first);
            end = wall - wrap_diff(uptime, last);
            if (end < start) end = start; // degenerate record (netflow.cpp:157-159)
        }
        const unsigned m = __ballot_sync(0xFFFFFFFFu, ok);
        if (ok) {
            uint4* o = reinterpret_cast<uint4*>(out + (base[i] + __popc(m & ((1u << lane) - 1u))) * 64);
            o[0] = w0;
            o[1] = w1;
            o[2] = w2;
            o[3] = make_uint4(static_cast<uint32_t>(start), static_cast<uint32_t>(start >> 32),
                              static_cast<uint32_t>(end), static_cast<uint32_t>(end >> 32));
        }
    }
}

// FlowStore::load's entry decode (flow_store.cpp:194-200), thread per entry:
// be64 start/end and decode_raw_record of the big-endian raw record, written
// as the 64-byte little-endian FlowRecord (raw fields, start_ms, end_ms).
__global__ void __launch_bounds__(256) a1_decode(const uint32_t* __restrict__ e, uint64_t n,
                                                 uint4* __restrict__ out) {
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t* w = e + i * 16;
        uint32_t x[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) x[k] = __ldg(w + k);
        auto sw = [](uint32_t v) { return __byte_perm(v, 0, 0x0123); };  // be32
        auto sw16 = [](uint32_t v) { return __byte_perm(v, 0, 0x2301); }; // two be16
        uint4* o = out + i * 4;
        // raw record = entry words 4..15
        o[0] = make_uint4(sw(x[4]), sw(x[5]), sw(x[6]), sw16(x[7]));
        o[1] = make_uint4(sw(x[8]), sw(x[9]), sw(x[10]), sw(x[11]));
        o[2] = make_uint4(sw16(x[12]), x[13], sw16(x[14]), __byte_perm(x[15], 0, 0x2310));
        o[3] = make_uint4(sw(x[1]), sw(x[0]), sw(x[3]), sw(x[2])); // start_ms, end_ms (LE u64)
    }
}

} // namespace

cudaError_t launch_archive_decode(const uint8_t* entries, uint64_t n, uint8_t* out, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const uint32_t g = static_cast<uint32_t>(std::min<uint64_t>((n + 255) / 256, 148 * 16));
    a1_decode<<<g, 256, 0, s>>>(reinterpret_cast<const uint32_t*>(entries), n, reinterpret_cast<uint4*>(out));
    return cudaGetLastError();
}

cudaError_t launch_netflow_decode(const uint8_t* d, const uint64_t* off, uint64_t n, uint32_t* accepted,
                                  uint64_t* base, uint8_t* status, unsigned long long* stats,
                                  uint8_t* out, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const uint32_t g1 = static_cast<uint32_t>(std::min<uint64_t>((n + 255) / 256, 4096));
    n1_validate<<<g1, 256, 0, s>>>(d, off, n, accepted, status, stats);
    n2_scan<<<1, 1024, 0, s>>>(accepted, n, base, stats + 4);
    const uint32_t g3 = static_cast<uint32_t>(std::min<uint64_t>((n * 32 + 255) / 256, 65535));
    n3_decode<<<g3, 256, 0, s>>>(d, off, n, base, out);
    return cudaGetLastError();
}

} // namespace gnm
