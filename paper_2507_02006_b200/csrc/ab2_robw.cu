// ab2_robw.cu -- RoBW row-block-wise tiler (Alg. 1, partition.hpp:52-74) on the device.
//
// The reference walks the rows greedily.  Its cut sequence is equivalent to
//   cut_{j+1} = max e  with  calc_mem(e - cut_j, row_ptr[e] - row_ptr[cut_j]) <= m_a
// (calc_mem(k,q) = (k+1)*I + q*(I+V), memory_model.hpp:84-86), because calc_mem of a row
// range is monotone in its end.  So:
//   K_next   : for every row r, nxt[r] = that max e (binary search over row_ptr)
//   K_bad    : the smallest row that cannot fit alone -> row_too_large (partition.hpp:64-69)
//   K_mark   : pointer doubling marks the chain 0 -> nxt(0) -> ... -> n in ceil(log2(S+1))
//              rounds of O(n) work (S = segment count)
//   K_scan + K_emit : compaction of the marked rows into the ordered cut list.
#include <algorithm>
#include <climits>

#include "ab2_internal.h"
#include "ab2_kernels.cuh"

namespace ab2 {

namespace {

__device__ __forceinline__ unsigned __int128 calc_mem_dev(uint64_t k, uint64_t q, uint64_t I, uint64_t V) {
  return static_cast<unsigned __int128>(k + 1) * I + static_cast<unsigned __int128>(q) * (I + V);
}

__global__ void k_robw_bad(const uint64_t* __restrict__ ptr, int64_t n, uint64_t m_a, uint64_t I, uint64_t V,
                           Ctl* __restrict__ ctl) {
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < n;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (calc_mem_dev(1, ptr[r + 1] - ptr[r], I, V) > m_a)
      atomicMin(&ctl->bad_row, static_cast<unsigned long long>(r));
  }
}

__global__ void k_robw_next(const uint64_t* __restrict__ ptr, int64_t n, uint64_t m_a, uint64_t I, uint64_t V,
                            int64_t* __restrict__ nxt, int32_t* __restrict__ mark) {
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r <= n;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    mark[r] = r == 0 ? 1 : 0;
    if (r == n) {
      nxt[r] = n;
      continue;
    }
    const uint64_t base = ptr[r];
    int64_t lo = r + 1, hi = n;  // largest e in [r+1, n] that fits; r+1 fits (no bad rows)
    while (lo < hi) {
      int64_t mid = lo + (hi - lo + 1) / 2;
      if (calc_mem_dev(static_cast<uint64_t>(mid - r), ptr[mid] - base, I, V) <= m_a)
        lo = mid;
      else
        hi = mid - 1;
    }
    nxt[r] = lo;
  }
}

__global__ void k_robw_mark(const int64_t* __restrict__ jump, int64_t n, int32_t* __restrict__ mark,
                            int64_t* __restrict__ jump2) {
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r <= n;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t j = jump[r];
    if (mark[r]) mark[j] = 1;
    jump2[r] = jump[j];
  }
}

__global__ void k_robw_emit(const int32_t* __restrict__ mark, const int64_t* __restrict__ pos, int64_t n,
                            uint64_t* __restrict__ cuts) {
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r <= n;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x)
    if (mark[r]) cuts[pos[r]] = static_cast<uint64_t>(r);
}

}  // namespace

int robw_cuts(Ctx& ctx, const uint64_t* row_ptr, uint64_t n_rows, uint64_t m_a, uint64_t I, uint64_t V,
              uint32_t location, uint64_t* cuts, uint64_t cap, uint64_t* n_segs, uint64_t* bad_row) {
  const int64_t n = static_cast<int64_t>(n_rows);
  if (cap < 1) fail(AIRES_B200_CAPACITY_EXCEEDED, "cuts capacity is zero");
  cuts[0] = 0;
  *n_segs = 0;
  if (n == 0) return AIRES_B200_OK;
  const uint64_t* dptr = row_ptr;
  if (location == AIRES_B200_HOST) {
    uint64_t* up = ctx.a_ptr.as<uint64_t>(n + 1);
    AB2_CUDA(cudaMemcpyAsync(up, row_ptr, (n + 1) * 8, cudaMemcpyHostToDevice, ctx.stream));
    dptr = up;
  }
  Ctl* ctl = ctx.ctl.as<Ctl>(1);
  Ctl* h = static_cast<Ctl*>(ctx.h_ctl.get(sizeof(Ctl)));
  AB2_CUDA(cudaMemsetAsync(ctl, 0, sizeof(Ctl), ctx.stream));
  AB2_CUDA(cudaMemsetAsync(&ctl->bad_row, 0xff, sizeof(unsigned long long), ctx.stream));
  const int grid = static_cast<int>(std::min<int64_t>((n + 256) / 256, static_cast<int64_t>(ctx.sms) * 16));
  k_robw_bad<<<grid, 256, 0, ctx.stream>>>(dptr, n, m_a, I, V, ctl);
  AB2_CUDA(cudaGetLastError());
  AB2_CUDA(cudaMemcpyAsync(h, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, ctx.stream));
  AB2_CUDA(cudaStreamSynchronize(ctx.stream));
  if (h->bad_row != ULLONG_MAX) {
    if (bad_row) *bad_row = h->bad_row;
    return AIRES_B200_ROW_TOO_LARGE;
  }
  int64_t* nxt = ctx.rflops.as<int64_t>(n + 1);
  int64_t* nxt2 = ctx.sym_heavy.as<int64_t>(n + 1);
  int32_t* mark = ctx.cnt.as<int32_t>(n + 1);
  int64_t* pos = ctx.cptr.as<int64_t>(n + 2);
  k_robw_next<<<grid, 256, 0, ctx.stream>>>(dptr, n, m_a, I, V, nxt, mark);
  AB2_CUDA(cudaGetLastError());
  // Pointer doubling; stop once jump^(2^t)(0) reaches n (every chain node marked).
  for (int round = 0; round < 64; round++) {
    k_robw_mark<<<grid, 256, 0, ctx.stream>>>(nxt, n, mark, nxt2);
    AB2_CUDA(cudaGetLastError());
    std::swap(nxt, nxt2);
    int64_t j0 = 0;
    AB2_CUDA(cudaMemcpyAsync(&j0, nxt, 8, cudaMemcpyDeviceToHost, ctx.stream));
    AB2_CUDA(cudaStreamSynchronize(ctx.stream));
    if (j0 == n) {
      // one more marking pass with the final jump covers the last 2^t chain nodes
      k_robw_mark<<<grid, 256, 0, ctx.stream>>>(nxt, n, mark, nxt2);
      AB2_CUDA(cudaGetLastError());
      break;
    }
  }
  const int64_t m = n + 1;
  const int64_t nb = (m + kScanTile - 1) / kScanTile;
  int64_t* part = ctx.scan_part.as<int64_t>(std::max<int64_t>(nb, 1));
  k_scan_reduce<<<static_cast<unsigned>(nb), kScanThreads, 0, ctx.stream>>>(mark, m, part);
  k_scan_part<<<1, 1024, 0, ctx.stream>>>(part, nb, ctl);
  k_scan_down<<<static_cast<unsigned>(nb), kScanThreads, 0, ctx.stream>>>(mark, m, part, pos);
  AB2_CUDA(cudaGetLastError());
  AB2_CUDA(cudaMemcpyAsync(h, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, ctx.stream));
  AB2_CUDA(cudaStreamSynchronize(ctx.stream));
  const uint64_t count = h->nnz;  // marked rows = segments + 1
  if (count > cap) fail(AIRES_B200_CAPACITY_EXCEEDED, "cuts buffer too small for " + std::to_string(count));
  uint64_t* dcuts = reinterpret_cast<uint64_t*>(ctx.num_heavy.as<int64_t>(count));
  k_robw_emit<<<grid, 256, 0, ctx.stream>>>(mark, pos, n, dcuts);
  AB2_CUDA(cudaGetLastError());
  AB2_CUDA(cudaMemcpyAsync(cuts, dcuts, count * 8, cudaMemcpyDeviceToHost, ctx.stream));
  AB2_CUDA(cudaStreamSynchronize(ctx.stream));
  *n_segs = count - 1;
  return AIRES_B200_OK;
}

}  // namespace ab2
