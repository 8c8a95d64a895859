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
// One kernel (nf_decode): validate and count, a chained scan across tiles
// of datagrams for the output offsets, then decode and compact.
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
    uint32_t version;
    if ((reinterpret_cast<uintptr_t>(p) & 3u) == 0) { // one word load instead of four byte loads
        const uint32_t w = __byte_perm(__ldg(reinterpret_cast<const uint32_t*>(p)), 0, 0x0123);
        version = w >> 16;
        count = w & 0xFFFFu;
    } else {
        version = be16(p);
        count = be16(p + 2);
    }
    if (version != 5) return 1;
    if (count == 0 || count > kMaxRec) return 3;
    if (len != kHdr + static_cast<uint64_t>(kRec) * count) return 2;
    return 0;
}


// Record fields of one 48-byte big-endian record (decode_raw_record,
// netflow.cpp:27-50), byte loads (datagrams that are not 4-byte aligned), as
// the RawFlowRecord words in memory order (netflow.hpp:32-57): u32 src, dst,
// next_hop; u16 input_if, output_if; u32 d_pkts, d_octets, first, last; u16
// src_port, dst_port; u8 pad1, tcp_flags, protocol, tos; u16 src_as, dst_as;
// u8 src_mask, dst_mask; u16 pad2.
__device__ __forceinline__ void load_raw_bytes(const uint8_t* q, uint4& w0, uint4& w1, uint4& w2) {
    w0 = make_uint4(be32(q), be32(q + 4), be32(q + 8), be16(q + 12) | be16(q + 14) << 16);
    w1 = make_uint4(be32(q + 16), be32(q + 20), be32(q + 24), be32(q + 28));
    w2 = make_uint4(be16(q + 32) | be16(q + 34) << 16,
                    static_cast<uint32_t>(q[36]) | static_cast<uint32_t>(q[37]) << 8 |
                        static_cast<uint32_t>(q[38]) << 16 | static_cast<uint32_t>(q[39]) << 24,
                    be16(q + 40) | be16(q + 42) << 16,
                    static_cast<uint32_t>(q[44]) | static_cast<uint32_t>(q[45]) << 8 | be16(q + 46) << 16);
}

// Single-pass decode with a chained scan (decoupled look-back). CTAs claim
// tiles of kNfTile consecutive datagrams in order from a counter. Phase 1:
// warp per datagram, the header checks of decode_packet and the collector's
// reject rule per record (lane = record), ballot counts. The tile's count
// total is published as an aggregate, the predecessors' are summed back to
// the first inclusive prefix, and the tile's inclusive prefix is published.
// Phase 2: warp per datagram again; a 4-byte-aligned datagram's record area
// (an L2 hit: phase 1 just read it) moves into shared memory with coalesced
// word loads (13-word record stride: conflict-free), others use byte loads;
// decode (byte permutes), resolve_times, accepted rows staged in shared
// memory and written with coalesced 16-byte stores at their final offsets.
#ifndef GNM_NF_PER_WARP
#define GNM_NF_PER_WARP 4
#endif
// kNfTile datagrams per tile, a multiple of 32 (warp 0 scans kNfPer per lane):
// bigger tiles amortise the look-back's CTA-wide barrier over more datagrams.
constexpr uint32_t kNfWarps = 8, kNfPerWarp = GNM_NF_PER_WARP, kNfTile = kNfWarps * kNfPerWarp;
constexpr uint32_t kNfPer = kNfTile / 32;
static_assert(kNfTile % 32 == 0, "tile = whole warps of datagrams");
constexpr unsigned long long kFlagAgg = 1ull << 62, kFlagPrefix = 2ull << 62, kValMask = (1ull << 62) - 1;

__global__ void __launch_bounds__(kNfWarps * 32) nf_decode(const uint8_t* __restrict__ d,
                                                           const uint64_t* __restrict__ off, uint64_t n,
                                                           unsigned long long* __restrict__ tiles,
                                                           uint8_t* __restrict__ status,
                                                           unsigned long long* __restrict__ stats,
                                                           uint8_t* __restrict__ out) {
    __shared__ uint32_t s_cnt[kNfTile];
    __shared__ unsigned long long s_base[kNfTile];
    __shared__ unsigned long long s_tile;
    __shared__ uint32_t s_rec[kNfWarps][kMaxRec * 13]; // a datagram's records, 13-word stride
    __shared__ uint4 s_out[kNfWarps][kMaxRec * 4];     // its accepted rows
    unsigned long long* counter = tiles; // tiles[0]: next tile; tiles[1 + t]: tile t's state
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const uint64_t n_tiles = (n + kNfTile - 1) / kNfTile;
    uint32_t err = 0, rej = 0, acc = 0; // lane 0's running totals
    while (true) {
        if (threadIdx.x == 0) s_tile = atomicAdd(counter, 1ull);
        __syncthreads();
        const uint64_t tile = s_tile;
        if (tile >= n_tiles) break; // CTA-uniform
        for (uint32_t k = 0; k < kNfPerWarp; ++k) {
            const uint32_t li = warp * kNfPerWarp + k;
            const uint64_t i = tile * kNfTile + li;
            uint32_t a = 0;
            if (i < n) { // warp-uniform
                const uint8_t* p = d + off[i];
                uint32_t count;
                const uint32_t st = check_header(p, off[i + 1] - off[i], count);
                const bool words = (reinterpret_cast<uintptr_t>(p) & 3u) == 0;
                bool ok = false;
                if (st == 0 && lane < count) {
                    const uint8_t* q = p + kHdr + kRec * lane;
                    uint32_t pkts, oct;
                    if (words) {
                        pkts = __byte_perm(__ldg(reinterpret_cast<const uint32_t*>(q + 16)), 0, 0x0123);
                        oct = __byte_perm(__ldg(reinterpret_cast<const uint32_t*>(q + 20)), 0, 0x0123);
                    } else {
                        pkts = be32(q + 16);
                        oct = be32(q + 20);
                    }
                    ok = pkts != 0 && oct >= pkts;
                }
                a = __popc(__ballot_sync(0xFFFFFFFFu, ok));
                if (lane == 0) {
                    if (st == 0) rej += count - a;
                    else ++err;
                    acc += a;
                    if (status) status[i] = static_cast<uint8_t>(st);
                }
            }
            if (lane == 0) s_cnt[li] = a;
        }
        __syncthreads();
        if (warp == 0) {
            // lane l owns datagrams [l*kNfPer, (l+1)*kNfPer) of the tile
            uint32_t vv[kNfPer], v = 0;
#pragma unroll
            for (uint32_t q = 0; q < kNfPer; ++q) {
                vv[q] = s_cnt[lane * kNfPer + q];
                v += vv[q];
            }
            uint32_t incl = v;
#pragma unroll
            for (uint32_t o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                if (lane >= o) incl += y;
            }
            const uint32_t total = __shfl_sync(0xFFFFFFFFu, incl, 31);
            unsigned long long prefix = 0;
            if (lane == 0) {
                if (tile == 0) {
                    atomicExch(tiles + 1, kFlagPrefix | total);
                } else {
                    atomicExch(tiles + 1 + tile, kFlagAgg | total);
                    for (uint64_t j = tile; j-- > 0;) { // predecessors were claimed earlier: they finish
                        unsigned long long stj;
                        do {
                            stj = *reinterpret_cast<volatile unsigned long long*>(tiles + 1 + j);
                        } while (stj == 0);
                        prefix += stj & kValMask;
                        if ((stj & ~kValMask) == kFlagPrefix) break;
                    }
                    atomicExch(tiles + 1 + tile, kFlagPrefix | (prefix + total));
                }
            }
            prefix = __shfl_sync(0xFFFFFFFFu, prefix, 0);
            unsigned long long b = prefix + incl - v;
#pragma unroll
            for (uint32_t q = 0; q < kNfPer; ++q) {
                s_base[lane * kNfPer + q] = b;
                b += vv[q];
            }
        }
        __syncthreads();
        for (uint32_t k = 0; k < kNfPerWarp; ++k) {
            const uint32_t li = warp * kNfPerWarp + k;
            const uint64_t i = tile * kNfTile + li;
            if (i >= n) break;
            const uint8_t* p = d + off[i];
            uint32_t count;
            if (check_header(p, off[i + 1] - off[i], count) != 0) continue; // warp-uniform
            const bool words = (reinterpret_cast<uintptr_t>(p) & 3u) == 0; // warp-uniform
            uint32_t uptime, secs, nsecs;
            if (words) {
                const uint32_t* h = reinterpret_cast<const uint32_t*>(p);
                uptime = __byte_perm(__ldg(h + 1), 0, 0x0123);
                secs = __byte_perm(__ldg(h + 2), 0, 0x0123);
                nsecs = __byte_perm(__ldg(h + 3), 0, 0x0123);
            } else {
                uptime = be32(p + 4), secs = be32(p + 8), nsecs = be32(p + 12);
            }
            const uint64_t wall = static_cast<uint64_t>(secs) * 1000u + nsecs / 1000000u;
            uint32_t* recw = s_rec[warp];
            if (words) { // coalesced word loads of the record area (an L2 hit) into a padded tile
                const uint32_t* src = reinterpret_cast<const uint32_t*>(p + kHdr);
                // word idx = 12 r + c; each step of 32 words is r += 2, c += 8
                uint32_t r = lane / 12, c = lane - r * 12;
                for (uint32_t idx = lane; idx < count * 12; idx += 32) {
                    recw[r * 13 + c] = __ldg(src + idx);
                    r += 2;
                    c += 8;
                    if (c >= 12) {
                        c -= 12;
                        ++r;
                    }
                }
                __syncwarp();
            }
            bool ok = false;
            uint4 w0{}, w1{}, w2{};
            uint64_t start = 0, end = 0;
            if (lane < count) {
                if (words) {
                    const uint32_t* x = recw + lane * 13;
                    auto sw = [](uint32_t v) { return __byte_perm(v, 0, 0x0123); };   // be32
                    auto sw16 = [](uint32_t v) { return __byte_perm(v, 0, 0x2301); }; // two be16
                    w0 = make_uint4(sw(x[0]), sw(x[1]), sw(x[2]), sw16(x[3]));
                    w1 = make_uint4(sw(x[4]), sw(x[5]), sw(x[6]), sw(x[7]));
                    w2 = make_uint4(sw16(x[8]), x[9], sw16(x[10]), __byte_perm(x[11], 0, 0x2310));
                } else {
                    load_raw_bytes(p + kHdr + kRec * lane, w0, w1, w2);
                }
                const uint32_t pkts = w1.x, oct = w1.y, first = w1.z, last = w1.w;
                ok = pkts != 0 && oct >= pkts;
                start = wall - wrap_diff(uptime, first);
                end = wall - wrap_diff(uptime, last);
                if (end < start) end = start; // degenerate record (netflow.cpp:157-159)
            }
            const unsigned m = __ballot_sync(0xFFFFFFFFu, ok);
            // Rows through shared memory, then coalesced 16-byte stores.
            uint4* rows = s_out[warp];
            __syncwarp();
            if (ok) {
                const uint32_t j = __popc(m & ((1u << lane) - 1u));
                rows[j * 4 + 0] = w0;
                rows[j * 4 + 1] = w1;
                rows[j * 4 + 2] = w2;
                rows[j * 4 + 3] = make_uint4(static_cast<uint32_t>(start), static_cast<uint32_t>(start >> 32),
                                             static_cast<uint32_t>(end), static_cast<uint32_t>(end >> 32));
            }
            __syncwarp();
            uint4* dst = reinterpret_cast<uint4*>(out + s_base[li] * 64);
            for (uint32_t idx = lane; idx < __popc(m) * 4; idx += 32) __stcs(dst + idx, rows[idx]);
            __syncwarp();
        }
        __syncthreads(); // s_tile, s_cnt and s_base are reused
    }
    if (lane == 0) {
        if (err) atomicAdd(stats + 1, static_cast<unsigned long long>(err));
        if (rej) atomicAdd(stats + 2, static_cast<unsigned long long>(rej));
        if (acc) atomicAdd(stats + 3, static_cast<unsigned long long>(acc));
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

uint64_t netflow_scratch_words(uint64_t n) { return 1 + (n + kNfTile - 1) / kNfTile; }

cudaError_t launch_netflow_decode(const uint8_t* d, const uint64_t* off, uint64_t n, unsigned long long* scratch,
                                  uint8_t* status, unsigned long long* stats, uint8_t* out, int device,
                                  cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    cudaError_t e = cudaMemsetAsync(scratch, 0, netflow_scratch_words(n) * 8, s);
    if (e != cudaSuccess) return e;
    int sms = 0, per_sm = 0;
    if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device)) != cudaSuccess) return e;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, nf_decode, kNfWarps * 32, 0)) != cudaSuccess)
        return e;
    const uint64_t n_tiles = (n + kNfTile - 1) / kNfTile;
    const uint32_t g = static_cast<uint32_t>(std::min<uint64_t>(n_tiles, static_cast<uint64_t>(sms) * std::max(per_sm, 1)));
    nf_decode<<<g, kNfWarps * 32, 0, s>>>(d, off, n, scratch, status, stats, out);
    return cudaGetLastError();
}

} // namespace gnm
