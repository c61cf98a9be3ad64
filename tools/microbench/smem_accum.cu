// Microbenchmark: cost of the candidate per-product accumulation primitives on B200
// (shared-memory fp32 CAS add, ATOMS.OR, MATCH.ANY-resolved LDS/FADD/STS, plain
// LDS/FADD/STS), random columns in [0, NC). One warp-private accumulator per warp.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define NC 602
#define ITERS 4096
__device__ __forceinline__ uint32_t hsh(uint32_t x){x^=x>>16;x*=0x7feb352d;x^=x>>15;x*=0x846ca68b;x^=x>>16;return x;}
template<int MODE>
__global__ void kern(float* out, int seed) {
  extern __shared__ float sm[];
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* acc = sm + warp * 640;
  uint32_t* bm = reinterpret_cast<uint32_t*>(acc);
  for (int i = lane; i < 640; i += 32) acc[i] = 0.f;
  __syncwarp();
  uint32_t s = hsh(seed ^ (blockIdx.x * 1024 + threadIdx.x));
  for (int it = 0; it < ITERS; it++) {
    s = hsh(s + it);
    int j = s % NC;
    float p = (s & 255) * 1e-3f;
    if (MODE == 0) { atomicAdd(&acc[j], p); }
    else if (MODE == 1) { atomicOr(&bm[j >> 5], 1u << (j & 31)); }
    else if (MODE == 2) {
      unsigned peers = __match_any_sync(0xffffffffu, j);
      int rank = __popc(peers & ((1u << lane) - 1));
      int maxr = __reduce_max_sync(0xffffffffu, rank);
      for (int q = 0; q <= maxr; q++) { if (rank == q) acc[j] += p; __syncwarp(); }
    } else if (MODE == 3) { acc[j] += p; }  // racy, cost floor
    else if (MODE == 4) {  // tag-based: write lane, read back
      int* tag = reinterpret_cast<int*>(acc + 320);
      bool pend = true;
      while (__any_sync(0xffffffffu, pend)) {
        if (pend) tag[j >> 1] = lane;
        __syncwarp();
        bool win = pend && tag[j >> 1] == lane;
        if (win) { acc[j & 255] += p; pend = false; }
        __syncwarp();
      }
    }
  }
  __syncwarp();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc[lane];
}
__global__ void gather(const uint2* __restrict__ x, const int* __restrict__ ptr, int K, float* out, int seed) {
  uint32_t s = hsh(seed ^ (blockIdx.x * 1024 + threadIdx.x)); float a = 0;
  for (int it = 0; it < 256; it++) { s = hsh(s + it); int k = s % K; int b = ptr[k], e = ptr[k+1];
    for (int t = b; t < e; t++) { uint2 v = x[t]; a += __int_as_float(v.y) * (v.x & 1); } }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a;
}
template<int M> float run(float* out, int blocks, int threads) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int smem = (threads / 32) * 640 * 4;
  cudaFuncSetAttribute(kern<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  kern<M><<<blocks, threads, smem>>>(out, 1);
  cudaEventRecord(a); kern<M><<<blocks, threads, smem>>>(out, 2); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); return ms;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int threads = 512, blocks = sms * 3; float* out; cudaMalloc(&out, blocks * threads * 4 * 4);
  double ops = double(blocks) * threads * ITERS;
  const char* names[] = {"atomicAdd f32 (CAS loop)", "atomicOr u32", "match_any ordered LDS/FADD/STS", "plain LDS/FADD/STS (racy floor)", "tag write/readback"};
  float t[5] = {run<0>(out, blocks, threads), run<1>(out, blocks, threads), run<2>(out, blocks, threads), run<3>(out, blocks, threads), run<4>(out, blocks, threads)};
  for (int i = 0; i < 5; i++) printf("%-34s %8.3f ms  %7.2f Gop/s  %6.2f SM-cycles/warp-op @1.9GHz\n", names[i], t[i], ops / t[i] / 1e6, t[i] * 1e-3 * 1.9e9 * sms / (ops / 32));
  // L2 gather of X rows: K rows of ~6 (col,val) pairs
  int K = 233000, nnz = K * 6; int* ptr; uint2* x; cudaMalloc(&ptr, (K + 1) * 4); cudaMalloc(&x, nnz * 8);
  int* hp = new int[K + 1]; for (int i = 0; i <= K; i++) hp[i] = i * 6; cudaMemcpy(ptr, hp, (K + 1) * 4, cudaMemcpyHostToDevice); cudaMemset(x, 0, nnz * 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int rep = 0; rep < 2; rep++) { cudaEventRecord(a); gather<<<sms * 4, 512>>>(x, ptr, K, out, rep); cudaEventRecord(b); cudaEventSynchronize(b); }
  float ms; cudaEventElapsedTime(&ms, a, b); double rows = double(sms) * 4 * 512 * 256;
  printf("X-row gather (6 x 8B, random k)    %8.3f ms  %7.2f G rows/s  (114M rows -> %.3f ms)\n", ms, rows / ms / 1e6, 114e6 / (rows / ms));
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
