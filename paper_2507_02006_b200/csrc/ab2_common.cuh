// ab2_common.cuh -- shared device/host plumbing for the B200 AIRES SpGEMM path.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <string>

#include "aires_b200.h"

namespace ab2 {

// Status carrying error: thrown inside the library, converted to a C status at
// the ABI boundary (ab2_api.cu).  code = 1 + aires::errc, or >= 100.
struct Error {
  int code;
  std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg);
void check_cuda(cudaError_t e, const char* what, const char* file, int line);

#define AB2_CUDA(x) ::ab2::check_cuda((x), #x, __FILE__, __LINE__)

constexpr unsigned kFull = 0xffffffffu;
constexpr int kMaxDenseColsF32 = 8192;   // dense shared accumulator limit (fp32)
constexpr int kMaxDenseColsF64 = 4096;   // (fp64)

// Device control block, zeroed per product.
struct Ctl {
  unsigned long long light_next;      // light-row ticket (symbolic)
  unsigned long long heavy_next;      // heavy-row ticket (symbolic)
  unsigned long long n_num_heavy;     // rows appended to the numeric heavy list
  unsigned long long flops;           // total MACs
  unsigned long long num_light_next;  // light-row ticket (numeric)
  unsigned long long num_heavy_next;  // heavy-row ticket (numeric)
  unsigned long long n_sym_heavy;     // rows appended to the symbolic heavy list
  unsigned long long n_fix;           // rows needing the structural-zero fix-up path
  unsigned long long nnz;             // total C nnz (written by the scan)
  unsigned long long bad_row;         // robw: smallest oversized row
  unsigned long long pad[6];
};

// ---- warp / block helpers --------------------------------------------------
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ int warp_id() { return threadIdx.x >> 5; }

template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

template <class T>
__device__ __forceinline__ T warp_incl_scan(T v) {
  const int lane = lane_id();
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T n = __shfl_up_sync(kFull, v, o);
    if (lane >= o) v += n;
  }
  return v;
}

// Block-wide inclusive scan (blockDim.x <= 1024, multiple of 32).  `tmp` needs
// 32 entries of T in shared memory.  Returns inclusive value; *total = block sum.
template <class T>
__device__ __forceinline__ T block_incl_scan(T v, T* tmp, T* total) {
  const int lane = lane_id(), warp = warp_id(), nw = blockDim.x >> 5;
  T x = warp_incl_scan(v);
  if (lane == 31) tmp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    T w = lane < nw ? tmp[lane] : T(0);
    w = warp_incl_scan(w);
    if (lane < nw) tmp[lane] = w;
  }
  __syncthreads();
  T off = warp > 0 ? tmp[warp - 1] : T(0);
  T tot = tmp[nw - 1];
  __syncthreads();
  *total = tot;
  return x + off;
}

template <class T>
__device__ __forceinline__ T block_sum(T v, T* tmp) {
  T tot;
  block_incl_scan(v, tmp, &tot);
  return tot;
}

}  // namespace ab2
