// Probe of the tcgen05 (kind::tf32) path the cfg5 H·W kernel uses: one 128x48 tile, K = 64, operands
// in shared memory in the K-major 128-byte-swizzled canonical layout, 3xTF32 split (hi*hi + hi*lo +
// lo*hi), accumulator in TMEM.  Prints the max relative error against an fp64 host product.
#include <cstdint>
#include <cstdio>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

constexpr int M = 128, N = 48, K = 64;

__device__ __forceinline__ uint32_t swz(int m, int k) {  // byte offset of (m, k) in one 32-wide K atom
  return (m >> 3) * 1024 + (m & 7) * 128 + ((((k >> 2) ^ (m & 7)) & 7) << 4) + (k & 3) * 4;
}
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4);
  d |= static_cast<uint64_t>(1) << 16;             // LBO (unused for swizzled K-major)
  d |= static_cast<uint64_t>(1024 >> 4) << 32;     // SBO: 8-row groups 1024 B apart
  d |= static_cast<uint64_t>(1) << 46;             // version (sm100)
  d |= static_cast<uint64_t>(2) << 61;             // SWIZZLE_128B
  return d;
}
__device__ __forceinline__ void split_tf32(float a, float& hi, float& lo) {
  hi = __uint_as_float(__float_as_uint(a) & 0xFFFFE000u);
  lo = a - hi;
}

__global__ void k_probe(const float* __restrict__ A, const float* __restrict__ B /* K x N */, float* __restrict__ D,
                        int* flag) {
  extern __shared__ __align__(1024) unsigned char sm[];
  // layout: A_hi [2 atoms x 16 KB], A_lo [2 x 16 KB], B_hi [2 x 6 KB], B_lo [2 x 6 KB], mbar, tmem slot
  unsigned char* a_hi = sm;
  unsigned char* a_lo = sm + 32768;
  unsigned char* b_hi = sm + 65536;
  unsigned char* b_lo = sm + 65536 + 12288;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(sm + 65536 + 24576);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(sm + 65536 + 24576 + 8);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < M * K; i += blockDim.x) {
    const int m = i / K, k = i % K;
    float h, l;
    split_tf32(A[i], h, l);
    const uint32_t off = (k >> 5) * 16384 + swz(m, k & 31);
    *reinterpret_cast<float*>(a_hi + off) = h;
    *reinterpret_cast<float*>(a_lo + off) = l;
  }
  for (int i = tid; i < N * K; i += blockDim.x) {
    const int n = i / K, k = i % K;  // B^T row n = column n of B
    float h, l;
    split_tf32(B[k * N + n], h, l);
    const uint32_t off = (k >> 5) * 6144 + swz(n, k & 31);
    *reinterpret_cast<float*>(b_hi + off) = h;
    *reinterpret_cast<float*>(b_lo + off) = l;
  }
  const uint32_t mbar_s = static_cast<uint32_t>(__cvta_generic_to_shared(mbar));
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar_s));
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(
        static_cast<uint32_t>(__cvta_generic_to_shared(tslot))));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tslot;
  if (tid == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
    const uint32_t ah = static_cast<uint32_t>(__cvta_generic_to_shared(a_hi));
    const uint32_t al = static_cast<uint32_t>(__cvta_generic_to_shared(a_lo));
    const uint32_t bh = static_cast<uint32_t>(__cvta_generic_to_shared(b_hi));
    const uint32_t bl = static_cast<uint32_t>(__cvta_generic_to_shared(b_lo));
    int first = 1;
    for (int kk = 0; kk < K / 8; kk++) {
      const uint32_t ao = (kk >> 2) * 16384 + (kk & 3) * 32, bo = (kk >> 2) * 6144 + (kk & 3) * 32;
      const uint64_t d_ah = sw128_desc(ah + ao), d_al = sw128_desc(al + ao);
      const uint64_t d_bh = sw128_desc(bh + bo), d_bl = sw128_desc(bl + bo);
      const uint64_t as[3] = {d_ah, d_ah, d_al}, bs[3] = {d_bh, d_bl, d_bh};
      for (int q = 0; q < 3; q++) {
        const uint32_t acc = first ? 0u : 1u;
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
                     "l"(as[q]), "l"(bs[q]), "r"(idesc), "r"(acc));
        first = 0;
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mbar_s)
                 : "memory");
  }
  // wait for the accumulator (phase 0)
  {
    uint32_t done = 0;
    while (!done) {
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
                   : "=r"(done) : "r"(mbar_s) : "memory");
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int m = warp * 32 + lane;
  for (int c0 = 0; c0 < N; c0 += 8) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 8; j++) D[m * N + c0 + j] = __uint_as_float(r[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem));
  if (tid == 0) *flag = 1;
}

int main() {
  std::vector<float> A(M * K), B(K * N), D(M * N);
  uint64_t s = 12345;
  auto rnd = [&] { s = s * 6364136223846793005ull + 1442695040888963407ull; return static_cast<float>((s >> 40) * (1.0 / (1ull << 24)) - 0.5); };
  for (auto& v : A) v = rnd();
  for (auto& v : B) v = rnd();
  float *dA, *dB, *dD;
  int* dflag;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  cudaMalloc(&dflag, 4);
  cudaMemset(dflag, 0, 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  const int smem = 65536 + 24576 + 64;
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_probe<<<1, 128, smem>>>(dA, dB, dD, dflag);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  double maxrel = 0, maxabs = 0;
  for (int m = 0; m < M; m++)
    for (int n = 0; n < N; n++) {
      double ref = 0, sc = 0;
      for (int k = 0; k < K; k++) {
        ref += static_cast<double>(A[m * K + k]) * B[k * N + n];
        sc += std::fabs(static_cast<double>(A[m * K + k]) * B[k * N + n]);
      }
      maxabs = std::max(maxabs, std::fabs(ref - D[m * N + n]));
      maxrel = std::max(maxrel, std::fabs(ref - D[m * N + n]) / sc);
    }
  printf("max abs err %.3e  max err / sum|terms| %.3e  D[0]=%f D[last]=%f\n", maxabs, maxrel, D[0], D[M * N - 1]);
  return 0;
}
