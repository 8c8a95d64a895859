// netflow.cuh — launch interface of the batched NetFlow v5 ingest (netflow.cu).
#pragma once

#include <algorithm>
#include <cstdint>
#include <cuda_runtime.h>

namespace gnm {

// d: concatenated datagrams; off[n+1]: datagram i is bytes [off[i], off[i+1]).
// scratch: netflow_scratch_words(n) u64 words (tile counter + tile states,
// zeroed here). status[n] (optional): 0 ok, 1 bad version, 2 truncated, 3
// bad count. stats[5] (zeroed by the caller): [1] decode errors, [2] records
// rejected, [3] records accepted. out: accepted FlowRecords (64 B each),
// datagram order.
uint64_t netflow_scratch_words(uint64_t n);
cudaError_t launch_netflow_decode(const uint8_t* d, const uint64_t* off, uint64_t n, unsigned long long* scratch,
                                  uint8_t* status, unsigned long long* stats, uint8_t* out, int device,
                                  cudaStream_t s);

// FLOWARC1 entries (64 B, big-endian, 4-byte aligned) -> FlowRecord rows.
cudaError_t launch_archive_decode(const uint8_t* entries, uint64_t n, uint8_t* out, cudaStream_t s);

} // namespace gnm
