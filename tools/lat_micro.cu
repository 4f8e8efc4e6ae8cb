// lat_micro.cu — single-warp dependent-chain latencies on the B200 (cycles per
// op) for the instructions on the latency-mode critical path: DADD, DMUL,
// DFMA, sqrt (double), __drcp_rn, SHFL, LDS, VOTE, WARPSYNC.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false tools/lat_micro.cu -o /tmp/lat_micro
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 4096;

__global__ void lat(double* out, long long* cyc, double a, double b) {
  __shared__ double sm[64];
  const int l = threadIdx.x;
  sm[l] = a + l;
  sm[l + 32] = b;
  __syncwarp();
  double x = a + l * 1e-9;
  long long t0, t1;
  int k = 0;
#define RUN(name, body)                      \
  t0 = clock64();                            \
  for (int i = 0; i < N; ++i) { body; }      \
  t1 = clock64();                            \
  if (l == 0) cyc[k] = t1 - t0;              \
  ++k;
  RUN("dadd", x = x + b)
  RUN("dmul", x = x * b)
  RUN("dfma", x = __fma_rn(x, b, a))
  RUN("dsqrt", x = sqrt(x) + 1.0)
  RUN("drcp", x = __drcp_rn(x) + 1.0)
  RUN("shfl", x = __shfl_sync(0xffffffffu, x, (l + 1) & 31))
  int idx = l;
  RUN("lds", idx = static_cast<int>(sm[idx & 63]) & 63)
  x += idx;
  unsigned m = l;
  RUN("vote", m = __ballot_sync(0xffffffffu, (m & 1u) != 0u) + l)
  x += m;
  RUN("syncwarp+lds", __syncwarp(); idx = static_cast<int>(sm[idx & 63]) & 63)
  x += idx;
  RUN("dsetp+sel", x = (x > b) ? x - a : x + a)
  out[l] = x;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 32 * 8);
  cudaMallocManaged(&cyc, 64 * 8);
  lat<<<1, 32>>>(out, cyc, 1.0000001, 0.9999999);
  cudaDeviceSynchronize();
  lat<<<1, 32>>>(out, cyc, 1.0000001, 0.9999999);
  cudaDeviceSynchronize();
  const char* names[] = {"dadd", "dmul", "dfma", "dsqrt(+dadd)", "drcp(+dadd)", "shfl", "lds(+cvt)", "vote(+iadd)",
                         "syncwarp+lds(+cvt)", "dsetp+sel(+dadd)"};
  for (int k = 0; k < 10; ++k) printf("%-20s %7.1f cycles/op\n", names[k], static_cast<double>(cyc[k]) / N);
  return 0;
}
