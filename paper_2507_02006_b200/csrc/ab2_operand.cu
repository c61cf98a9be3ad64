// ab2_operand.cu -- builds the B200 feature layout of X (ab2_operand.cuh) on the device.
//
// Accepts X as CSR (spgemm_full(Csr,Csr), spgemm.hpp:148-151) or CSC (the form the
// reference kernel takes, spgemm.hpp:63); CSC is transposed on the device (the
// reference's csc_to_csr, sparse.hpp:142-163: columns ascend within each row).
#include <algorithm>
#include <cstring>

#include "ab2_internal.h"
#include "ab2_kernels.cuh"

namespace ab2 {

namespace {

// ptr holds absolute offsets into idx/val (spgemm.hpp:79-84); nnz = ptr[K] - ptr[0] is read
// on the device so a device-resident operand needs no host round trip.
template <class IdxT, class VIn, class V>
__global__ void k_x_from_csr(const uint64_t* __restrict__ ptr, int64_t K, const IdxT* __restrict__ idx,
                             const VIn* __restrict__ val, int64_t n_cols, int64_t* __restrict__ xptr,
                             int32_t* __restrict__ xcol, V* __restrict__ xval, Ctl* __restrict__ ctl) {
  const uint64_t p0 = ptr[0];
  const int64_t nnz = static_cast<int64_t>(ptr[K] - p0);
  int64_t n = max(K + 1, nnz);
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (i <= K) xptr[i] = static_cast<int64_t>(ptr[i] - p0);
    if (i < nnz) {
      uint64_t c = static_cast<uint64_t>(idx[p0 + i]);
      if (c >= static_cast<uint64_t>(n_cols)) ctl->bad_row = 1;
      xcol[i] = static_cast<int32_t>(c);
      xval[i] = static_cast<V>(val[p0 + i]);
    }
  }
}

template <class IdxT>
__global__ void k_csc_count(const IdxT* __restrict__ ridx, int64_t nnz, int64_t K,
                            int32_t* __restrict__ counts, Ctl* __restrict__ ctl) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nnz;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    uint64_t r = static_cast<uint64_t>(ridx[i]);
    if (r >= static_cast<uint64_t>(K)) {
      ctl->bad_row = 1;
      continue;
    }
    atomicAdd(&counts[r], 1);
  }
}

template <class IdxT, class VIn, class V>
__global__ void k_csc_scatter(const uint64_t* __restrict__ cptr, uint64_t p0, int64_t n_cols,
                              const IdxT* __restrict__ ridx, const VIn* __restrict__ val, int64_t nnz,
                              int64_t K, const int64_t* __restrict__ xptr, int32_t* __restrict__ cursor,
                              int32_t* __restrict__ xcol, V* __restrict__ xval) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nnz;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    uint64_t q = p0 + static_cast<uint64_t>(i);
    int64_t lo = 0, hi = n_cols + 1;  // upper_bound(q) over cptr[0..n_cols]
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (cptr[mid] <= q)
        lo = mid + 1;
      else
        hi = mid;
    }
    int64_t c = lo - 1;
    uint64_t r = static_cast<uint64_t>(ridx[i]);
    if (r >= static_cast<uint64_t>(K)) continue;
    int64_t pos = xptr[r] + atomicAdd(&cursor[r], 1);
    xcol[pos] = static_cast<int32_t>(c);
    xval[pos] = static_cast<V>(val[i]);
  }
}

// Rows of X are short on the dense path; insertion sort restores ascending columns
// after the unordered scatter (columns are unique per row, so the result is unique).
template <class V>
__global__ void k_row_sort(const int64_t* __restrict__ xptr, int64_t K, int32_t* __restrict__ xcol,
                           V* __restrict__ xval) {
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < K;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t s = xptr[k], e = xptr[k + 1];
    for (int64_t i = s + 1; i < e; i++) {
      int32_t c = xcol[i];
      V v = xval[i];
      int64_t j = i - 1;
      while (j >= s && xcol[j] > c) {
        xcol[j + 1] = xcol[j];
        xval[j + 1] = xval[j];
        j--;
      }
      xcol[j + 1] = c;
      xval[j + 1] = v;
    }
  }
}

__global__ void k_len_hist(const int64_t* __restrict__ xptr, int64_t K,
                           unsigned long long* __restrict__ h) {
  __shared__ int64_t tmp[32];
  int64_t c[5] = {0, 0, 0, 0, 0};
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < K;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t n = xptr[k + 1] - xptr[k];
    c[0] += n > 2;
    c[1] += n > 4;
    c[2] += n > 8;
    c[3] += n > 16;
    c[4] = max(c[4], n);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) h[5] = static_cast<unsigned long long>(xptr[K]);
  for (int j = 0; j < 4; j++) {
    int64_t s = block_sum<int64_t>(c[j], tmp);
    if (threadIdx.x == 0 && s) atomicAdd(&h[j], static_cast<unsigned long long>(s));
  }
  int64_t m = c[4];
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(kFull, m, o));
  __shared__ int64_t s_m[32];
  if ((threadIdx.x & 31) == 0) s_m[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < static_cast<int>(blockDim.x >> 5); i++) m = max(m, s_m[i]);
    atomicMax(&h[4], static_cast<unsigned long long>(m));
  }
}

// Slot rows 0..K-1 from the plain CSR, plus the dummy row K (see ab2_operand.cuh).
// Smallest nonzero |x| (bit patterns of non-negative floats order like the values) and an
// exact-zero flag: they decide how the product pass guards against zero products.
template <class V>
__global__ void k_x_val_stats(const V* __restrict__ xval, const int64_t* __restrict__ xptr, int64_t K,
                              unsigned long long* __restrict__ st) {
  const int64_t nnz = xptr[K];
  unsigned long long mn = ~0ull;
  int z = 0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nnz;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double v = fabs(static_cast<double>(xval[i]));
    if (v == 0.0)
      z = 1;
    else
      mn = min(mn, static_cast<unsigned long long>(__double_as_longlong(v)));
  }
  for (int o = 16; o > 0; o >>= 1) {
    mn = min(mn, __shfl_xor_sync(kFull, mn, o));
    z |= __shfl_xor_sync(kFull, z, o);
  }
  // one atomic per block (every warp of every block hitting one word serialised ~30 us at cfg2)
  __shared__ unsigned long long s_mn[32];
  __shared__ int s_z[32];
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    s_mn[w] = mn;
    s_z[w] = z;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < nw; i++) {
      mn = min(mn, s_mn[i]);
      z |= s_z[i];
    }
    if (mn != ~0ull) atomicMin(&st[0], mn);
    if (z) st[1] = 1;
  }
}

template <class V, int W>
__global__ void k_x_slots(const int64_t* __restrict__ xptr, const int32_t* __restrict__ xcol,
                          const V* __restrict__ xval, int64_t K, uint32_t trash,
                          typename SlotOf<V>::type* __restrict__ slots, uint16_t* __restrict__ xlen) {
  using S = typename SlotOf<V>::type;
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k <= K;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t s = k < K ? xptr[k] : 0, n = k < K ? xptr[k + 1] - s : 0;
    S* out = slots + k * W;
    xlen[k] = static_cast<uint16_t>(n);
    const bool ovf = n > W;
    const int inl = ovf ? W - 1 : static_cast<int>(n);
#pragma unroll
    for (int e = 0; e < W; e++) {
      S en{};
      en.val = V(1);
      en.col = trash;
      if (e < inl) {
        en.col = static_cast<uint32_t>(xcol[s + e]);
        en.val = xval[s + e];
      } else if (ovf && e == W - 1) {
        const uint32_t tail = static_cast<uint32_t>(n - (W - 1));
        const uint32_t off = static_cast<uint32_t>(s + W - 1);
        en.col = kSlotOvf | (tail << 16) | trash;
        if constexpr (sizeof(V) == 4)
          en.val = __uint_as_float(kOneBits + off);
        else
          en.pad = off;
      }
      out[e] = en;
    }
  }
}

// Padded fp32 layout for the step-list product pass (ab2_numeric5.cuh): X row k occupies
// nslot = ceil(len / W5) consecutive W5-entry slots starting at slot pstart[k]; an entry is
// {accumulator byte offset col * 4, value bits}; entries past len point at the trash column
// (value 1.0), so a W5-lane group always loads and adds a full slot.  The last slot is an
// all-trash dummy used to pad step lists.
// desc[k] = {pstart[k], nslot | len << 16}; desc[K] = {0, 0} (the dummy row).
__global__ void k_x_pcount(const int64_t* __restrict__ xptr, int64_t K, int w5, int32_t* __restrict__ cnt) {
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < K;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    cnt[k] = static_cast<int32_t>((xptr[k + 1] - xptr[k] + w5 - 1) / w5);
}

__global__ void k_x_pfill(const int64_t* __restrict__ xptr, const int32_t* __restrict__ xcol,
                          const float* __restrict__ xval, int64_t K, int w5, uint32_t trash,
                          const uint32_t* __restrict__ pstart, uint2* __restrict__ desc, uint2* __restrict__ ent,
                          int64_t dummy) {
  if (blockIdx.x == 0 && threadIdx.x < w5) ent[dummy * w5 + threadIdx.x] = make_uint2(trash * 4u, kOneBits);
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k <= K;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (k == K) {
      desc[k] = make_uint2(0u, 0u);
      continue;
    }
    const int64_t s = xptr[k], len = xptr[k + 1] - s;
    const int64_t ns = (len + w5 - 1) / w5;
    const int64_t p = pstart[k];
    desc[k] = make_uint2(static_cast<uint32_t>(p), static_cast<uint32_t>(ns | (len << 16)));
    uint2* o = ent + p * w5;
    for (int64_t e = 0; e < ns * w5; e++)
      o[e] = e < len ? make_uint2(static_cast<uint32_t>(xcol[s + e]) * 4u, __float_as_uint(xval[s + e]))
                     : make_uint2(trash * 4u, kOneBits);
  }
}

// Column-only slots for the symbolic pass (kCSlotW entries, one 32 B sector per row).
__global__ void k_x_cslots(const int64_t* __restrict__ xptr, const int32_t* __restrict__ xcol, int64_t K,
                           uint16_t* __restrict__ cslots) {
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < K;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t s = xptr[k], n = xptr[k + 1] - s;
    const bool ovf = n > kCSlotW;
    const int inl = ovf ? kCSlotW - 1 : static_cast<int>(n);
    uint16_t v[kCSlotW];
#pragma unroll
    for (int e = 0; e < kCSlotW; e++)
      v[e] = e < inl ? static_cast<uint16_t>(xcol[s + e]) : (ovf && e == kCSlotW - 1 ? kCOvf : kCEmpty);
    uint4* o = reinterpret_cast<uint4*>(cslots + k * kCSlotW);
    const uint32_t* w = reinterpret_cast<const uint32_t*>(v);
    o[0] = make_uint4(w[0], w[1], w[2], w[3]);
    o[1] = make_uint4(w[4], w[5], w[6], w[7]);
  }
}

int grid_for(int64_t n, int threads, int sms) {
  int64_t b = (n + threads - 1) / threads;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(b, static_cast<int64_t>(sms) * 32)));
}

template <class V>
void build_slots(Ctx& ctx, XOperand& x) {
  int g = grid_for(x.K + 1, 256, ctx.sms);
  using S = typename SlotOf<V>::type;
  auto* sl = static_cast<S*>(x.slots);
  auto* cs = static_cast<uint16_t*>(x.cslots);
  auto* xp = static_cast<int64_t*>(x.ptr);
  auto* xc = static_cast<int32_t*>(x.col);
  auto* xv = static_cast<V*>(x.val);
  const uint32_t trash = static_cast<uint32_t>(x.n_cols);
  if (x.slots) switch (x.W) {
    case 2: k_x_slots<V, 2><<<g, 256, 0, ctx.stream>>>(xp, xc, xv, x.K, trash, sl, static_cast<uint16_t*>(x.xlen)); break;
    case 4: k_x_slots<V, 4><<<g, 256, 0, ctx.stream>>>(xp, xc, xv, x.K, trash, sl, static_cast<uint16_t*>(x.xlen)); break;
    case 8: k_x_slots<V, 8><<<g, 256, 0, ctx.stream>>>(xp, xc, xv, x.K, trash, sl, static_cast<uint16_t*>(x.xlen)); break;
    default: k_x_slots<V, 16><<<g, 256, 0, ctx.stream>>>(xp, xc, xv, x.K, trash, sl, static_cast<uint16_t*>(x.xlen)); break;
  }
  if (x.cslots) k_x_cslots<<<g, 256, 0, ctx.stream>>>(xp, xc, x.K, cs);
  AB2_CUDA(cudaGetLastError());
}

template <class IdxT, class VIn, class V>
void fill_plain(Ctx& ctx, XOperand& x, const aires_b200_matrix& b, const uint64_t* dptr, uint64_t p0,
                const void* didx, const void* dval, Ctl* ctl) {
  const IdxT* idx = static_cast<const IdxT*>(didx);
  const VIn* val = static_cast<const VIn*>(dval);
  auto* xp = static_cast<int64_t*>(x.ptr);
  auto* xc = static_cast<int32_t*>(x.col);
  auto* xv = static_cast<V*>(x.val);
  if (b.layout == AIRES_B200_CSR) {
    int g = grid_for(std::max<int64_t>(x.K + 1, x.nnz), 256, ctx.sms);
    k_x_from_csr<IdxT, VIn, V><<<g, 256, 0, ctx.stream>>>(dptr, x.K, idx, val, x.n_cols, xp, xc, xv, ctl);
    AB2_CUDA(cudaGetLastError());
    return;
  }
  // CSC -> CSR: count, scan, scatter, sort (entries addressed from p0).
  idx += p0;
  val += p0;
  int32_t* counts = ctx.cnt.as<int32_t>(std::max<int64_t>(x.K, 1));
  int32_t* cursor = reinterpret_cast<int32_t*>(ctx.rflops.as<int64_t>(std::max<int64_t>(x.K, 1)));
  AB2_CUDA(cudaMemsetAsync(counts, 0, sizeof(int32_t) * std::max<int64_t>(x.K, 1), ctx.stream));
  AB2_CUDA(cudaMemsetAsync(cursor, 0, sizeof(int32_t) * std::max<int64_t>(x.K, 1), ctx.stream));
  if (x.nnz > 0) {
    k_csc_count<IdxT><<<grid_for(x.nnz, 256, ctx.sms), 256, 0, ctx.stream>>>(idx, x.nnz, x.K, counts, ctl);
    AB2_CUDA(cudaGetLastError());
  }
  int64_t nb = (x.K + kScanTile - 1) / kScanTile;
  int64_t* part = ctx.scan_part.as<int64_t>(std::max<int64_t>(nb, 1));
  if (x.K > 0) {
    k_scan_reduce<<<static_cast<unsigned>(nb), kScanThreads, 0, ctx.stream>>>(counts, x.K, part);
    k_scan_part<<<1, 1024, 0, ctx.stream>>>(part, nb, ctl);
    k_scan_down<<<static_cast<unsigned>(nb), kScanThreads, 0, ctx.stream>>>(counts, x.K, part, xp);
  } else {
    AB2_CUDA(cudaMemsetAsync(xp, 0, sizeof(int64_t), ctx.stream));
  }
  AB2_CUDA(cudaGetLastError());
  if (x.nnz > 0) {
    k_csc_scatter<IdxT, VIn, V><<<grid_for(x.nnz, 256, ctx.sms), 256, 0, ctx.stream>>>(
        dptr, p0, x.n_cols, idx, val, x.nnz, x.K, xp, cursor, xc, xv);
    k_row_sort<V><<<grid_for(x.K, 128, ctx.sms), 128, 0, ctx.stream>>>(xp, x.K, xc, xv);
    AB2_CUDA(cudaGetLastError());
  }
}

template <class V>
void fill_dispatch(Ctx& ctx, XOperand& x, const aires_b200_matrix& b, const uint64_t* dptr, uint64_t p0,
                   const void* didx, const void* dval, Ctl* ctl) {
  if (b.idx_bytes == 4 && b.val_bytes == 4)
    fill_plain<uint32_t, float, V>(ctx, x, b, dptr, p0, didx, dval, ctl);
  else if (b.idx_bytes == 4)
    fill_plain<uint32_t, double, V>(ctx, x, b, dptr, p0, didx, dval, ctl);
  else if (b.val_bytes == 4)
    fill_plain<uint64_t, float, V>(ctx, x, b, dptr, p0, didx, dval, ctl);
  else
    fill_plain<uint64_t, double, V>(ctx, x, b, dptr, p0, didx, dval, ctl);
}

void* dmalloc(size_t bytes, size_t* total) {
  void* p = nullptr;
  bytes = std::max<size_t>(bytes, 16);
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    fail(AIRES_B200_INSUFFICIENT_DEVICE_MEMORY, "cudaMalloc of operand failed");
  }
  AB2_CUDA(e);
  *total += bytes;
  return p;
}

}  // namespace

XOperand::~XOperand() {
  if (!owned) return;
  int prev = -1;
  cudaGetDevice(&prev);
  if (prev != device) cudaSetDevice(device);
  for (void* p : {ptr, col, val, slots, cslots, xlen, xdesc, xent})
    if (p) cudaFree(p);
  if (prev != device && prev >= 0) cudaSetDevice(prev);
}

int64_t wide_threshold(uint32_t mode) {
  const int64_t dense_max = mode == AIRES_B200_MODE_FP32 ? kMaxDenseColsF32 : kMaxDenseColsF64;
  return std::max<int64_t>(32, std::min<int64_t>(dense_max, option("wide_at", dense_max)));
}

std::unique_ptr<XOperand> make_operand(Ctx& ctx, const aires_b200_matrix& b, uint32_t mode, bool temp, uint32_t plan,
                                       Region* rg) {
  if (b.layout != AIRES_B200_CSR && b.layout != AIRES_B200_CSC)
    fail(AIRES_B200_INVALID_ARGUMENT, "operand layout must be CSR or CSC");
  if ((b.idx_bytes != 4 && b.idx_bytes != 8) || (b.val_bytes != 4 && b.val_bytes != 8))
    fail(AIRES_B200_INVALID_ARGUMENT, "operand idx_bytes/val_bytes must be 4 or 8");
  if (mode == AIRES_B200_MODE_AUTO) mode = b.val_bytes == 8 ? AIRES_B200_MODE_FP64_EXACT : AIRES_B200_MODE_FP32;
  if (mode != AIRES_B200_MODE_FP32 && mode != AIRES_B200_MODE_FP64_EXACT)
    fail(AIRES_B200_INVALID_ARGUMENT, "unknown arithmetic mode");
  auto x = std::make_unique<XOperand>();
  x->device = ctx.device;
  x->mode = mode;
  x->owned = !temp;
  x->K = static_cast<int64_t>(b.n_rows);
  x->n_cols = static_cast<int64_t>(b.n_cols);
  const uint64_t nptr = (b.layout == AIRES_B200_CSR ? b.n_rows : b.n_cols) + 1;
  const int64_t dense_max = wide_threshold(mode);
  // wide X: only the plain CSR is built; the product runs in column tiles (wide_product)
  x->wide = x->n_cols > dense_max;
  if (x->wide && (plan & (kPlanStep | kPlanCSlots)))
    fail(AIRES_B200_UNSUPPORTED_FORMAT, "feature matrix has " + std::to_string(x->n_cols) +
                                            " columns; the out-of-core path supports " + std::to_string(dense_max));
  if (b.ptr == nullptr) fail(AIRES_B200_INVALID_ARGUMENT, "operand ptr is null");
  if (b.span >= (uint64_t(1) << 31)) fail(AIRES_B200_CAPACITY_EXCEEDED, "operand span exceeds 2^31 entries");

  // Host operands: stage the used span.  Device CSR operands are read in place (the
  // kernels read ptr[0] / ptr[K] themselves); device CSC needs the span ends on the host.
  uint64_t p0 = 0, p1 = b.span;
  const uint64_t* dptr = b.ptr;
  const void* didx = b.idx;
  const void* dval = b.val;
  // a budgeted lean build from a host CSR already in the canonical widths (u32 columns, fp32 values,
  // ptr[0] = 0) converts the raw upload in place: it is the plain CSR the step list is built from
  const bool lean = rg && (plan & kPlanLean) && (plan & kPlanStep) && !(plan & (kPlanSlots | kPlanCSlots));
  bool in_place = false;
  if (b.location == AIRES_B200_HOST) {
    p0 = b.ptr[0];
    p1 = b.ptr[nptr - 1];
    if (p1 < p0 || p1 > b.span) fail(AIRES_B200_INDEX_OUT_OF_RANGE, "operand pointer array exceeds its span");
    in_place = lean && p0 == 0 && b.layout == AIRES_B200_CSR && b.idx_bytes == 4 && b.val_bytes == 4 &&
               mode == AIRES_B200_MODE_FP32;
    uint64_t* up = rg ? static_cast<uint64_t*>(rg->temp(nptr * 8)) : ctx.x_ptr.as<uint64_t>(nptr);
    void* ui = rg ? rg->temp(std::max<uint64_t>(p1, 1) * b.idx_bytes) : ctx.x_idx.get(std::max<uint64_t>(p1, 1) * b.idx_bytes);
    void* uv = rg ? rg->temp(std::max<uint64_t>(p1, 1) * b.val_bytes) : ctx.x_val.get(std::max<uint64_t>(p1, 1) * b.val_bytes);
    AB2_CUDA(cudaMemcpyAsync(up, b.ptr, nptr * 8, cudaMemcpyHostToDevice, ctx.stream));
    if (p1 > p0) {  // same absolute positions as on the host
      AB2_CUDA(cudaMemcpyAsync(static_cast<char*>(ui) + p0 * b.idx_bytes,
                               static_cast<const char*>(b.idx) + p0 * b.idx_bytes, (p1 - p0) * b.idx_bytes,
                               cudaMemcpyHostToDevice, ctx.stream));
      AB2_CUDA(cudaMemcpyAsync(static_cast<char*>(uv) + p0 * b.val_bytes,
                               static_cast<const char*>(b.val) + p0 * b.val_bytes, (p1 - p0) * b.val_bytes,
                               cudaMemcpyHostToDevice, ctx.stream));
    }
    dptr = up;
    didx = ui;
    dval = uv;
    x->bytes += nptr * 8 + std::max<uint64_t>(p1, 1) * (b.idx_bytes + b.val_bytes);  // raw upload
  } else if (b.layout == AIRES_B200_CSC) {
    AB2_CUDA(cudaMemcpyAsync(&p0, b.ptr, 8, cudaMemcpyDeviceToHost, ctx.stream));
    AB2_CUDA(cudaMemcpyAsync(&p1, b.ptr + nptr - 1, 8, cudaMemcpyDeviceToHost, ctx.stream));
    AB2_CUDA(cudaStreamSynchronize(ctx.stream));
    if (p1 < p0 || p1 > b.span) fail(AIRES_B200_INDEX_OUT_OF_RANGE, "operand pointer array exceeds its span");
  }
  // nnz upper bound until the histogram readback reports the exact count
  x->nnz = static_cast<int64_t>(b.location == AIRES_B200_HOST || b.layout == AIRES_B200_CSC ? p1 - p0 : b.span);

  Ctl* ctl = ctx.ctl.as<Ctl>(1);
  AB2_CUDA(cudaMemsetAsync(ctl, 0, sizeof(Ctl), ctx.stream));
  const size_t vb = mode == AIRES_B200_MODE_FP32 ? 4 : 8;
  if (plan == kPlanAuto)
    plan = mode == AIRES_B200_MODE_FP32 && option("numeric_kernel", 3) == 5 ? kPlanStep : kPlanSlots;
  if (mode != AIRES_B200_MODE_FP32) plan &= ~static_cast<uint32_t>(kPlanStep);
  auto alloc = [&](DevBuf& cache, size_t bytes) -> void* {
    if (rg) {
      x->bytes += Region::up(bytes);
      return rg->keep(bytes);
    }
    if (temp) {
      x->bytes += std::max<size_t>(bytes, 256);
      return cache.get(bytes);
    }
    return dmalloc(bytes, &x->bytes);
  };
  if (in_place) {  // the raw upload (same positions, p0 = 0) becomes the plain CSR
    x->ptr = const_cast<uint64_t*>(dptr);
    x->col = const_cast<void*>(didx);
    x->val = const_cast<void*>(dval);
  } else if (lean) {  // the plain CSR is a build temporary
    x->ptr = rg->temp((x->K + 1) * 8);
    x->col = rg->temp(std::max<int64_t>(x->nnz, 1) * 4);
    x->val = rg->temp(std::max<int64_t>(x->nnz, 1) * vb);
  } else {
    x->ptr = alloc(ctx.xo_ptr, (x->K + 1) * 8);
    x->col = alloc(ctx.xo_col, std::max<int64_t>(x->nnz, 1) * 4);
    x->val = alloc(ctx.xo_val, std::max<int64_t>(x->nnz, 1) * vb);
  }
  if (mode == AIRES_B200_MODE_FP32)
    fill_dispatch<float>(ctx, *x, b, dptr, p0, didx, dval, ctl);
  else
    fill_dispatch<double>(ctx, *x, b, dptr, p0, didx, dval, ctl);

  // choose the slot width from the row-length histogram (one readback)
  unsigned long long* hist = reinterpret_cast<unsigned long long*>(&ctl->pad[0]);
  AB2_CUDA(cudaMemsetAsync(&ctl->bad_row + 0, 0, 8, ctx.stream));
  AB2_CUDA(cudaMemsetAsync(&ctl->flops, 0xff, 8, ctx.stream));  // min |x| bits
  {
    const int g = std::min(grid_for(std::max<int64_t>(x->nnz, 1), 256, ctx.sms), ctx.sms * 8);
    auto* xp = static_cast<const int64_t*>(x->ptr);
    if (mode == AIRES_B200_MODE_FP32)
      k_x_val_stats<float><<<g, 256, 0, ctx.stream>>>(static_cast<float*>(x->val), xp, x->K, &ctl->flops);
    else
      k_x_val_stats<double><<<g, 256, 0, ctx.stream>>>(static_cast<double*>(x->val), xp, x->K, &ctl->flops);
  }
  k_len_hist<<<std::min(grid_for(std::max<int64_t>(x->K, 1), 256, ctx.sms), ctx.sms * 8), 256, 0, ctx.stream>>>(
      static_cast<int64_t*>(x->ptr), x->K, hist);
  AB2_CUDA(cudaGetLastError());
  Ctl* h = static_cast<Ctl*>(ctx.h_ctl.get(sizeof(Ctl)));
  AB2_CUDA(cudaMemcpyAsync(h, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, ctx.stream));
  AB2_CUDA(cudaStreamSynchronize(ctx.stream));
  if (h->bad_row) fail(AIRES_B200_INDEX_OUT_OF_RANGE, "operand index outside its dimensions");
  x->nnz = static_cast<int64_t>(h->pad[5]);
  {
    const unsigned long long bits = h->flops;
    double mn;
    std::memcpy(&mn, &bits, 8);
    x->xmin = bits == ~0ull ? 0.0 : mn;
    x->has_zero = h->num_light_next != 0;
  }
  if (static_cast<int64_t>(h->pad[4]) > kMaxTail)
    fail(AIRES_B200_UNSUPPORTED_FORMAT, "feature row longer than " + std::to_string(kMaxTail) + " entries");
  x->max_row_len = static_cast<int64_t>(h->pad[4]);
  const double K = static_cast<double>(std::max<int64_t>(x->K, 1));
  const double frac[4] = {h->pad[0] / K, h->pad[1] / K, h->pad[2] / K, h->pad[3] / K};
  int W = 16;
  const int widths[4] = {2, 4, 8, 16};
  // Tails cost a dependent round trip for the whole warp step, so the slot must hold
  // all but ~1% of rows (measured: 8-wide slots on the Reddit shape put a tail in 48%
  // of warp steps and doubled the numeric pass's instruction count).
  for (int i = 0; i < 4; i++)
    if (frac[i] <= 0.01) {
      W = widths[i];
      break;
    }
  int64_t forced = option("slot_w", 0);
  if (forced == 2 || forced == 4 || forced == 8 || forced == 16) W = static_cast<int>(forced);
  x->W = W;
  if (x->wide) plan = 0;
  if (plan & kPlanSlots) {
    const size_t sb = mode == AIRES_B200_MODE_FP32 ? sizeof(SlotF) : sizeof(SlotD);
    x->slots = alloc(ctx.xo_slots, (x->K + 1) * W * sb);
    x->xlen = alloc(ctx.xo_len, (x->K + 1) * 2);
    x->prep_launches += 1;
  }
  if (plan & kPlanCSlots) {
    x->cslots = alloc(ctx.xo_cslots, std::max<int64_t>(x->K, 1) * kCSlotW * 2);
    x->prep_launches += 1;
  }
  if (mode == AIRES_B200_MODE_FP32)
    build_slots<float>(ctx, *x);
  else
    build_slots<double>(ctx, *x);
  if (plan & kPlanStep) {
    // step-list layout: W5 ~ the mean row length, copies = 32 / W5 accumulators per warp
    const double mean = static_cast<double>(x->nnz) / K;
    int w5 = mean >= 4.0 ? 8 : (mean >= 2.0 ? 4 : 2);
    const int64_t stride = (x->n_cols + 1 + 31) & ~int64_t(31);
    while (w5 < 32 && (32 / w5) * stride * 4 > 24 * 1024) w5 *= 2;
    const int64_t fw = option("w5", 0);
    if (fw == 2 || fw == 4 || fw == 8 || fw == 16 || fw == 32) w5 = static_cast<int>(fw);
    x->W5 = w5;
    const int64_t nb = (x->K + kScanTile - 1) / kScanTile;
    int32_t* pc = rg ? static_cast<int32_t*>(rg->temp(std::max<int64_t>(x->K, 1) * 4))
                     : ctx.cnt.as<int32_t>(std::max<int64_t>(x->K, 1));
    uint32_t* ps = rg ? static_cast<uint32_t*>(rg->temp((x->K + 1) * 4))
                      : reinterpret_cast<uint32_t*>(ctx.cptr.as<int64_t>(x->K / 2 + 1));
    int64_t* part = rg ? static_cast<int64_t*>(rg->temp(std::max<int64_t>(nb, 1) * 8))
                       : ctx.scan_part.as<int64_t>(std::max<int64_t>(nb, 1));
    const int g = grid_for(std::max<int64_t>(x->K + 1, 1), 256, ctx.sms);
    k_x_pcount<<<g, 256, 0, ctx.stream>>>(static_cast<const int64_t*>(x->ptr), x->K, w5, pc);
    int64_t n_slots = 0;
    if (x->K > 0) {
      k_scan_reduce<<<static_cast<unsigned>(nb), kScanThreads, 0, ctx.stream>>>(pc, x->K, part);
      k_scan_part<<<1, 1024, 0, ctx.stream>>>(part, nb, ctl);
      k_scan_down<uint32_t><<<static_cast<unsigned>(nb), kScanThreads, 0, ctx.stream>>>(pc, x->K, part, ps);
      // the exact slot count (one readback) sizes the entry array
      AB2_CUDA(cudaMemcpyAsync(&h->nnz, &ctl->nnz, 8, cudaMemcpyDeviceToHost, ctx.stream));
      AB2_CUDA(cudaStreamSynchronize(ctx.stream));
      n_slots = static_cast<int64_t>(h->nnz);
    }
    if (n_slots >= (int64_t(1) << 32) - 1) fail(AIRES_B200_CAPACITY_EXCEEDED, "feature step list exceeds 2^32 slots");
    const int64_t slots_ub = n_slots + 1;  // + the dummy slot
    x->dummy_slot = slots_ub - 1;
    x->xdesc = alloc(ctx.xo_desc, (x->K + 1) * sizeof(uint2));
    x->xent = alloc(ctx.xo_ent, slots_ub * w5 * sizeof(uint2));
    k_x_pfill<<<g, 256, 0, ctx.stream>>>(static_cast<const int64_t*>(x->ptr), static_cast<const int32_t*>(x->col),
                                           static_cast<const float*>(x->val), x->K, w5,
                                           static_cast<uint32_t>(x->n_cols), ps, static_cast<uint2*>(x->xdesc),
                                           static_cast<uint2*>(x->xent), x->dummy_slot);
    AB2_CUDA(cudaGetLastError());
    x->prep_launches += x->K > 0 ? 5 : 2;
  }
  x->prep_launches += (b.layout == AIRES_B200_CSR ? 1 : 6) + 2;
  if (rg) {
    // the build's temporaries (raw upload, scratch, and the plain CSR of a lean build) go back to
    // the region once the kernels reading them are done
    AB2_CUDA(cudaStreamSynchronize(ctx.stream));
    rg->drop_temps();
    if (lean) x->ptr = x->col = x->val = nullptr;
  } else if ((plan & kPlanLean) && (plan & kPlanStep) && x->xdesc && !x->slots && !x->cslots && temp) {
    // tight budgets: the step list is the only layout the product and the sizing kernels read, so
    // the plain CSR (the build's input) is released rather than held through the run
    AB2_CUDA(cudaStreamSynchronize(ctx.stream));
    const size_t csr = ctx.xo_ptr.cap + ctx.xo_col.cap + ctx.xo_val.cap;
    ctx.xo_ptr.release();
    ctx.xo_col.release();
    ctx.xo_val.release();
    x->ptr = x->col = x->val = nullptr;
    x->bytes = x->bytes > csr ? x->bytes - csr : 0;
  }
  if (!temp) AB2_CUDA(cudaStreamSynchronize(ctx.stream));
  return x;
}

}  // namespace ab2
