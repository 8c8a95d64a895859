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
// N1 validates every datagram and counts its accepted records (thread per
// datagram), N2 turns the counts into output offsets (cub's decoupled
// look-back exclusive scan), N3 decodes (warp per datagram, lane = record)
// and compacts the accepted records with a ballot.
#include <cuda_runtime.h>

#include <cstdint>

#include <cub/device/device_scan.cuh>
#include <cuda/std/functional>

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

__device__ __forceinline__ uint32_t ld_be32(const uint8_t* q, bool words) {
    return words ? __byte_perm(__ldg(reinterpret_cast<const uint32_t*>(q)), 0, 0x0123) : be32(q);
}

// N1, warp per datagram: header checks (lane 0's view is every lane's), then
// lane r tests record r's reject rule; the ballot's popcount is the
// datagram's accepted count.
__global__ void __launch_bounds__(256) n1_validate(const uint8_t* __restrict__ d,
                                                   const uint64_t* __restrict__ off, uint64_t n,
                                                   uint32_t* __restrict__ accepted,
                                                   uint8_t* __restrict__ status,
                                                   unsigned long long* __restrict__ stats) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
    uint32_t err = 0, rej = 0, acc = 0; // lane 0's running totals
    for (uint64_t i = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; i < n; i += nwarps) {
        const uint8_t* p = d + off[i];
        uint32_t count;
        const uint32_t st = check_header(p, off[i + 1] - off[i], count); // warp-uniform
        bool ok = false;
        if (st == 0 && lane < count) {
            const uint8_t* q = p + kHdr + kRec * lane;
            const bool words = (reinterpret_cast<uintptr_t>(p) & 3u) == 0;
            const uint32_t pkts = ld_be32(q + 16, words), oct = ld_be32(q + 20, words);
            ok = pkts != 0 && oct >= pkts;
        }
        const uint32_t a = __popc(__ballot_sync(0xFFFFFFFFu, ok));
        if (lane == 0) {
            if (st == 0) rej += count - a;
            else ++err;
            acc += a;
            accepted[i] = a;
            if (status) status[i] = static_cast<uint8_t>(st);
        }
    }
    if (lane == 0) {
        if (err) atomicAdd(stats + 1, static_cast<unsigned long long>(err));
        if (rej) atomicAdd(stats + 2, static_cast<unsigned long long>(rej));
        if (acc) atomicAdd(stats + 3, static_cast<unsigned long long>(acc));
    }
}

__global__ void n2_total(const uint32_t* __restrict__ in, const uint64_t* __restrict__ base, uint64_t n,
                         unsigned long long* __restrict__ total) {
    *total = base[n - 1] + in[n - 1];
}

// Record fields of one 48-byte big-endian record (decode_raw_record,
// netflow.cpp:27-50) as the RawFlowRecord words in memory order
// (netflow.hpp:32-57): u32 src, dst, next_hop; u16 input_if, output_if; u32
// d_pkts, d_octets, first, last; u16 src_port, dst_port; u8 pad1,
// tcp_flags, protocol, tos; u16 src_as, dst_as; u8 src_mask, dst_mask; u16
// pad2. kWords: the record is 4-byte aligned, so 12 word loads and byte
// permutes replace 48 byte loads.
template <bool kWords>
__device__ __forceinline__ void load_raw(const uint8_t* q, uint4& w0, uint4& w1, uint4& w2) {
    if constexpr (kWords) {
        const uint32_t* u = reinterpret_cast<const uint32_t*>(q);
        uint32_t x[12];
#pragma unroll
        for (int k = 0; k < 12; ++k) x[k] = __ldg(u + k);
        auto sw = [](uint32_t v) { return __byte_perm(v, 0, 0x0123); };   // be32
        auto sw16 = [](uint32_t v) { return __byte_perm(v, 0, 0x2301); }; // two be16
        w0 = make_uint4(sw(x[0]), sw(x[1]), sw(x[2]), sw16(x[3]));
        w1 = make_uint4(sw(x[4]), sw(x[5]), sw(x[6]), sw(x[7]));
        w2 = make_uint4(sw16(x[8]), x[9], sw16(x[10]), __byte_perm(x[11], 0, 0x2310));
    } else {
        w0 = make_uint4(be32(q), be32(q + 4), be32(q + 8), be16(q + 12) | be16(q + 14) << 16);
        w1 = make_uint4(be32(q + 16), be32(q + 20), be32(q + 24), be32(q + 28));
        w2 = make_uint4(be16(q + 32) | be16(q + 34) << 16,
                        static_cast<uint32_t>(q[36]) | static_cast<uint32_t>(q[37]) << 8 |
                            static_cast<uint32_t>(q[38]) << 16 | static_cast<uint32_t>(q[39]) << 24,
                        be16(q + 40) | be16(q + 42) << 16,
                        static_cast<uint32_t>(q[44]) | static_cast<uint32_t>(q[45]) << 8 | be16(q + 46) << 16);
    }
}

// Warp per datagram; lane r decodes record r and resolve_times; accepted
// lanes are compacted in record order.
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
            if ((reinterpret_cast<uintptr_t>(p) & 3u) == 0) load_raw<true>(q, w0, w1, w2); // warp-uniform
            else load_raw<false>(q, w0, w1, w2);
            const uint32_t pkts = w1.x, oct = w1.y, first = w1.z, last = w1.w;
            ok = pkts != 0 && oct >= pkts;
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

// FlowStore::load's entry decode (flow_store.cpp:194-200): be64 start/end
// and decode_raw_record of the big-endian raw record, written as the 64-byte
// little-endian FlowRecord (raw fields, start_ms, end_ms). Entries sit at
// 20 + 64*i (4-byte aligned only), so a warp moves 32 entries at a time
// through shared memory: coalesced word loads in, a per-lane decode from a
// padded tile (stride 17 words: conflict-free), coalesced 16-byte stores out.
constexpr uint32_t kA1Block = 256;
__global__ void __launch_bounds__(kA1Block) a1_decode(const uint32_t* __restrict__ e, uint64_t n,
                                                      uint4* __restrict__ out) {
    __shared__ uint32_t tile[kA1Block / 32][32 * 17];
    __shared__ uint4 rows[kA1Block / 32][32 * 4];
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    uint32_t* t = tile[warp];
    uint4* o = rows[warp];
    const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
    for (uint64_t b = ((static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * 32; b < n;
         b += nwarps * 32) {
        const uint32_t cnt = n - b < 32 ? static_cast<uint32_t>(n - b) : 32u;
        const uint32_t* src = e + b * 16;
#pragma unroll
        for (uint32_t k = 0; k < 16; ++k) {
            const uint32_t idx = k * 32 + lane;
            if (idx < cnt * 16) t[(idx >> 4) * 17 + (idx & 15u)] = __ldcs(src + idx);
        }
        __syncwarp();
        if (lane < cnt) {
            uint32_t x[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) x[k] = t[lane * 17 + k];
            auto sw = [](uint32_t v) { return __byte_perm(v, 0, 0x0123); };  // be32
            auto sw16 = [](uint32_t v) { return __byte_perm(v, 0, 0x2301); }; // two be16
            // raw record = entry words 4..15
            o[lane * 4 + 0] = make_uint4(sw(x[4]), sw(x[5]), sw(x[6]), sw16(x[7]));
            o[lane * 4 + 1] = make_uint4(sw(x[8]), sw(x[9]), sw(x[10]), sw(x[11]));
            o[lane * 4 + 2] = make_uint4(sw16(x[12]), x[13], sw16(x[14]), __byte_perm(x[15], 0, 0x2310));
            o[lane * 4 + 3] = make_uint4(sw(x[1]), sw(x[0]), sw(x[3]), sw(x[2])); // start_ms, end_ms (LE u64)
        }
        __syncwarp();
        uint4* dst = out + b * 4;
#pragma unroll
        for (uint32_t k = 0; k < 4; ++k) {
            const uint32_t idx = k * 32 + lane;
            if (idx < cnt * 4) __stcs(dst + idx, o[idx]);
        }
        __syncwarp();
    }
}

} // namespace

cudaError_t launch_archive_decode(const uint8_t* entries, uint64_t n, uint8_t* out, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const uint32_t g = static_cast<uint32_t>(std::min<uint64_t>((n + kA1Block - 1) / kA1Block, 148 * 8));
    a1_decode<<<g, kA1Block, 0, s>>>(reinterpret_cast<const uint32_t*>(entries), n, reinterpret_cast<uint4*>(out));
    return cudaGetLastError();
}

cudaError_t launch_netflow_decode(const uint8_t* d, const uint64_t* off, uint64_t n, uint32_t* accepted,
                                  uint64_t* base, uint8_t* status, unsigned long long* stats,
                                  uint8_t* out, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const uint32_t g1 = static_cast<uint32_t>(std::min<uint64_t>((n * 32 + 255) / 256, 148 * 16));
    n1_validate<<<g1, 256, 0, s>>>(d, off, n, accepted, status, stats);
    // N2: exclusive scan (decoupled look-back) of the accepted counts into u64 offsets.
    size_t tb = 0;
    cudaError_t e = cub::DeviceScan::ExclusiveScan(nullptr, tb, accepted, base, ::cuda::std::plus<uint64_t>(),
                                                   static_cast<uint64_t>(0), n, s);
    if (e != cudaSuccess) return e;
    void* tmp = nullptr;
    if ((e = cudaMallocAsync(&tmp, std::max<size_t>(tb, 1), s)) != cudaSuccess) return e;
    e = cub::DeviceScan::ExclusiveScan(tmp, tb, accepted, base, ::cuda::std::plus<uint64_t>(),
                                       static_cast<uint64_t>(0), n, s);
    if (e != cudaSuccess) return e;
    if ((e = cudaFreeAsync(tmp, s)) != cudaSuccess) return e;
    n2_total<<<1, 1, 0, s>>>(accepted, base, n, stats + 4);
    const uint32_t g3 = static_cast<uint32_t>(std::min<uint64_t>((n * 32 + 255) / 256, 65535));
    n3_decode<<<g3, 256, 0, s>>>(d, off, n, base, out);
    return cudaGetLastError();
}

} // namespace gnm
