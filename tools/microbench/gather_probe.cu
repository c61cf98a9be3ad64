// Random-row gather ceiling for the fused layer's Ã·T kernel (k_agg_t_cp): T is R rows of P floats
// (pitch P*4 bytes), G row indices drawn uniformly; every gathered row is read in full (16-byte
// loads, half a warp per row) and summed so the loads are live.  Prints the achieved GB/s of
// gathered row bytes for a few loads-in-flight settings -- the roofline the aggregation is held to
// (cfg5: R = 2.45M, P = 48, G = 126M).
#include <cstdint>
#include <cstdio>
#include <vector>

#include <cuda_runtime.h>

#define CK(x)                                                                           \
  do {                                                                                  \
    cudaError_t e_ = (x);                                                               \
    if (e_ != cudaSuccess) {                                                            \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));        \
      return 1;                                                                         \
    }                                                                                   \
  } while (0)

template <int P, int U>
__global__ void __launch_bounds__(256) k_gather(const float4* __restrict__ t, const uint32_t* __restrict__ idx,
                                                int64_t g, float* __restrict__ out) {
  constexpr int P4 = P / 4;
  const int lane = threadIdx.x & 31, half = lane >> 4, piece = lane & 15;
  const int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int64_t b = w * 2 * U; b < g; b += nw * 2 * U) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int64_t i = b + 2 * u + half;
      v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (i < g && piece < P4) v[u] = __ldg(t + static_cast<int64_t>(idx[i]) * P4 + piece);
    }
#pragma unroll
    for (int u = 0; u < U; u++) s.x += v[u].x, s.y += v[u].y, s.z += v[u].z, s.w += v[u].w;
  }
  if (s.x + s.y + s.z + s.w == 12345.f) out[0] = s.x;
}

template <int P, int U>
int run(const float4* t, const uint32_t* idx, int64_t g, float* out, int sms) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  int nb = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_gather<P, U>, 256, 0));
  const int grid = nb * sms;
  for (int i = 0; i < 2; i++) k_gather<P, U><<<grid, 256>>>(t, idx, g, out);
  CK(cudaEventRecord(a));
  const int reps = 5;
  for (int i = 0; i < reps; i++) k_gather<P, U><<<grid, 256>>>(t, idx, g, out);
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, a, b));
  ms /= reps;
  printf("P=%d loads-in-flight/lane=%d  %.3f ms  %.0f GB/s of gathered rows\n", P, U, ms,
         g * P * 4.0 / ms / 1e6);
  return 0;
}

int main(int argc, char** argv) {
  const int64_t R = argc > 1 ? atoll(argv[1]) : 2449029, G = argc > 2 ? atoll(argv[2]) : 126167053;
  constexpr int P = 48;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  std::vector<uint32_t> h(G);
  uint64_t x = 88172645463325252ull;
  for (int64_t i = 0; i < G; i++) {
    x ^= x << 13, x ^= x >> 7, x ^= x << 17;
    h[i] = static_cast<uint32_t>(x % R);
  }
  float4* t;
  uint32_t* idx;
  float* out;
  CK(cudaMalloc(&t, R * P * 4));
  CK(cudaMalloc(&idx, G * 4));
  CK(cudaMalloc(&out, 4));
  CK(cudaMemset(t, 0, R * P * 4));
  CK(cudaMemcpy(idx, h.data(), G * 4, cudaMemcpyHostToDevice));
  printf("R=%lld rows x %d floats (%.0f MB), G=%lld gathers\n", (long long)R, P, R * P * 4 / 1e6, (long long)G);
  if (run<P, 2>(t, idx, G, out, sms) || run<P, 4>(t, idx, G, out, sms) || run<P, 8>(t, idx, G, out, sms) ||
      run<P, 16>(t, idx, G, out, sms))
    return 1;
  return 0;
}
