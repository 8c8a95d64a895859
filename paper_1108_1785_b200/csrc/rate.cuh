// rate.cuh — one flow's f64 rate and exact micro-bps on the device, shared by
// K2 (kernels.cu) and the per-host post-pass H1 (hosts.cu), which recomputes
// them from the logged (octets, duration) instead of reading them back.
//   flow_rate    rate_engine.cpp:88-94   RN(8000*oct / RN(dur)), one IEEE division
//   rate_ubps_of rate_engine.cpp:100-107 floor(oct * 8e9 / dur) as a 128-bit value
// Paths are relative to /root/reference/proj/core/src.
#pragma once
#include <cstdint>

namespace gnm {

static __device__ __forceinline__ double flow_rate_dev(uint32_t oct, uint64_t dur) {
    return __ddiv_rn(8000.0 * static_cast<double>(oct), __ull2double_rn(dur));
}

// Exact micro-bps (hi is non-zero only when dur is a few ms and octets are
// huge). Fast path: the f64 rate is within 2^-52 relative of 8000*oct/dur
// (2^-53 more when double(dur) rounds), so y = rate * 1e6 is within
// 3*X*2^-53 of X; below rate 1e9 (X < 2^50) that is < 0.375, and q = rint(y)
// satisfies |q - X| < 0.875. Hence floor(X) is q or q - 1, decided by the
// sign of the exact residual p - q*dur (|residual| < dur, so its 64-bit
// wrapped value is exact). Everything else takes the exact integer division.
static __device__ __noinline__ uint4 ubps_slow(uint32_t oct, uint64_t dur) {
    if (oct <= 2305843009u) {
        const uint64_t q = static_cast<uint64_t>(oct) * 8000000000ull / dur;
        return make_uint4(static_cast<uint32_t>(q), static_cast<uint32_t>(q >> 32), 0u, 0u);
    }
    const unsigned __int128 q = static_cast<unsigned __int128>(oct) * 8000000000ull / dur;
    const uint64_t lo = static_cast<uint64_t>(q), hi = static_cast<uint64_t>(q >> 64);
    return make_uint4(static_cast<uint32_t>(lo), static_cast<uint32_t>(lo >> 32),
                      static_cast<uint32_t>(hi), static_cast<uint32_t>(hi >> 32));
}

static __device__ __forceinline__ void ubps_of(uint32_t oct, uint64_t dur, double rate, uint64_t& lo,
                                               uint64_t& hi) {
    if (oct <= 2305843009u && rate < 1.0e9) {
        const uint64_t pp = static_cast<uint64_t>(oct) * 8000000000ull;
        const uint64_t q = __double2ull_rn(__dmul_rn(rate, 1.0e6));
        const int64_t r = static_cast<int64_t>(pp - q * dur);
        lo = r < 0 ? q - 1 : q;
        hi = 0;
        return;
    }
    const uint4 s = ubps_slow(oct, dur);
    lo = static_cast<uint64_t>(s.y) << 32 | s.x;
    hi = static_cast<uint64_t>(s.w) << 32 | s.z;
}

} // namespace gnm
