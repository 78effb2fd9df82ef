// Host-side entry points of the device-wide primitives in sort.cu.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

namespace cvlg {

// Counts every kernel launch the library issues (reported as `gpu_launches` by the bench).
void count_launch();
uint64_t launch_count();

uint64_t scan_temp_words(uint64_t n);
// out[i] = sum(in[0..i)); *d_total (optional, device) = sum(in). d_tmp: scan_temp_words(n) u32.
void exclusive_scan_u32(const uint32_t* in, uint32_t* out, uint64_t n, uint32_t* d_total,
                        uint32_t* d_tmp, cudaStream_t s);

uint64_t radix_temp_bytes(uint64_t n);
// Stable LSD sort of (keys, vals) on key bits [begin_bit, end_bit). Result in (keys, vals).
// d_orand (2 x u64 device) + h_orand (2 x u64 pinned host) enable constant-digit skipping.
// With `in_alt` (host flag out), the one-sweep path does not copy a result that ended in the
// alternate buffers back: it waits for the pass plan and sets *in_alt instead (the caller swaps).
void radix_sort_pairs(uint64_t* keys, uint32_t* vals, uint64_t* keys_alt, uint32_t* vals_alt,
                      uint64_t n, int begin_bit, int end_bit, void* d_tmp, cudaStream_t s,
                      unsigned long long* d_orand, unsigned long long* h_orand,
                      bool* in_alt = nullptr);

}  // namespace cvlg
