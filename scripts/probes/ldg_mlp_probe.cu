// L2 gather throughput vs resident warps per SM and loads in flight per lane
// (LDG.E.256 non-coherent, 256 B rows = 8 lanes x 32 B, hashed rows from a
// 64 MiB L2-resident footprint).  Is the attention kernels' gap to the probe
// peak an MLP (latency-hiding) gap?
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

template <int U>
__global__ void __launch_bounds__(256) probe(const float* __restrict__ buf, uint32_t rows,
                                             uint32_t iters, float* sink) {
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t grp = tid / 8, sub = tid % 8;
  uint32_t x = grp * 2654435761u + 12345u;
  float acc = 0.f;
  for (uint32_t i = 0; i < iters; i += U) {
    float v[U][8];
#pragma unroll
    for (int t = 0; t < U; ++t) {
      x = x * 1664525u + 1013904223u;
      const float* p = buf + (static_cast<size_t>(x % rows) * 8 + sub) * 8;
      asm volatile("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=f"(v[t][0]), "=f"(v[t][1]), "=f"(v[t][2]), "=f"(v[t][3]), "=f"(v[t][4]),
                     "=f"(v[t][5]), "=f"(v[t][6]), "=f"(v[t][7])
                   : "l"(p));
    }
#pragma unroll
    for (int t = 0; t < U; ++t) acc += v[t][0] + v[t][7];
  }
  if (acc == 12345.678f) sink[tid] = acc;
}

template <int U>
void run(const float* buf, uint32_t rows, float* sink) {
  for (int bps : {2, 3, 4, 6, 8}) {
    const int blocks = 148 * bps;
    const uint32_t iters = 2048;
    probe<U><<<blocks, 256>>>(buf, rows, iters, sink);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int r = 0; r < 3; ++r) probe<U><<<blocks, 256>>>(buf, rows, iters, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double bytes = 3.0 * blocks * 256 * double(iters) * 32;
    printf("U %2d  warps/SM %2d  %8.0f GB/s\n", U, bps * 8, bytes / (ms * 1e-3) / 1e9);
  }
}

int main() {
  const size_t fp = 64u << 20;
  const uint32_t rows = fp / 256;
  float *buf, *sink;
  cudaMalloc(&buf, fp);
  cudaMalloc(&sink, 148 * 8 * 256 * 4);
  cudaMemset(buf, 0, fp);
  run<1>(buf, rows, sink);
  run<2>(buf, rows, sink);
  run<4>(buf, rows, sink);
  run<8>(buf, rows, sink);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
