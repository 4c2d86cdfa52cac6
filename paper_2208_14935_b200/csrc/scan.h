// scan.h -- the library's device scan and stable descending key sort (scan.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace hyt {
// bytes of temporary device memory exclusive_scan needs for n items
uint64_t scan_temp_bytes(uint64_t n);
// out[i] = sum_{j<i} in[j] (out may alias nothing); temp >= scan_temp_bytes(n)
template <class In, class Out>
void exclusive_scan(const In *in, Out *out, uint64_t n, void *temp, cudaStream_t st);
// sort (key, val) pairs by key descending, stable; key2/val2/flags/pos are n-item
// scratch, scan_temp >= scan_temp_bytes(n), mx_dev one u64 of device scratch
void sort_desc_stable(uint64_t *key, uint32_t *val, uint64_t *key2, uint32_t *val2, uint64_t n, uint32_t *flags,
                      uint32_t *pos, void *scan_temp, unsigned long long *mx_dev, cudaStream_t st);
}  // namespace hyt
