// Design probe: does a software prefetch of the NEXT iteration's gathered rows
// into L1 (prefetch.global.L1) raise the gather rate of a latency-bound,
// register-limited loop like fwd_fast's?  Rows of 256 B from a 64 MiB
// L2-resident table in hashed order; lanes in groups of 8 read one row's
// consecutive 32 B sectors (LDG.E.256), U rows per group per iteration, a
// little FMA work per row; 3 CTAs x 256 threads per SM (80 registers).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l1pf l1_prefetch_probe.cu
#include <cstdint>
#include <cstdio>

constexpr int U = 4;

__device__ __forceinline__ uint32_t row_of(uint32_t g, uint32_t i, uint32_t rows) {
  uint32_t x = (g * 2654435761u) ^ (i * 0x9E3779B9u);
  x ^= x >> 15;
  x *= 0x2C1B3C6Du;
  x ^= x >> 12;
  return x % rows;
}

template <int MODE>  // 0: no_allocate loads; 1: L1-allocating loads; 2: 1 + prefetch.L1 of the next iteration
__global__ void __launch_bounds__(256, 3) probe(const float* __restrict__ buf, uint32_t rows,
                                                uint32_t iters, float* __restrict__ sink) {
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t grp = tid / 8, sub = tid % 8;
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  float w[8];
  for (int k = 0; k < 8; ++k) w[k] = 0.001f * (k + sub);
  if (MODE == 2) {
    for (int t = 0; t < U; ++t) {
      const float* p = buf + (static_cast<size_t>(row_of(grp, t, rows)) * 8 + sub) * 8;
      asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
    }
  }
#pragma unroll 1
  for (uint32_t i = 0; i < iters; ++i) {
    float v[U][8];
#pragma unroll
    for (int t = 0; t < U; ++t) {
      const float* p = buf + (static_cast<size_t>(row_of(grp, i * U + t, rows)) * 8 + sub) * 8;
      if (MODE == 0)
        asm volatile("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(v[t][0]), "=f"(v[t][1]), "=f"(v[t][2]), "=f"(v[t][3]), "=f"(v[t][4]),
                       "=f"(v[t][5]), "=f"(v[t][6]), "=f"(v[t][7])
                     : "l"(p));
      else
        asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(v[t][0]), "=f"(v[t][1]), "=f"(v[t][2]), "=f"(v[t][3]), "=f"(v[t][4]),
                       "=f"(v[t][5]), "=f"(v[t][6]), "=f"(v[t][7])
                     : "l"(p));
    }
    if (MODE == 2) {
#pragma unroll
      for (int t = 0; t < U; ++t) {
        const float* p =
            buf + (static_cast<size_t>(row_of(grp, (i + 1) * U + t, rows)) * 8 + sub) * 8;
        asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
      }
    }
#pragma unroll
    for (int t = 0; t < U; ++t) {
      float s = 0.f;
#pragma unroll
      for (int k = 0; k < 8; ++k) s = fmaf(v[t][k], w[k], s);
      const float pr = exp2f(s);
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] = fmaf(pr, v[t][k], acc[k]);
    }
  }
  float s = 0.f;
  for (int k = 0; k < 8; ++k) s += acc[k];
  if (s == 12345.678f) sink[tid] = s;
}

template <int MODE>
double run(const float* buf, uint32_t rows, float* sink, int sms) {
  const int blocks = sms * 3 * 8;
  const uint32_t iters = 256;
  probe<MODE><<<blocks, 256>>>(buf, rows, iters, sink);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) probe<MODE><<<blocks, 256>>>(buf, rows, iters, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double bytes = 5.0 * blocks * 256 / 8 * iters * U * 256.0;
  return bytes / (ms * 1e-3) / 1e9;
}

int main() {
  const size_t foot = 64u << 20;
  const uint32_t rows = foot / 256;
  float *buf, *sink;
  cudaMalloc(&buf, foot);
  cudaMemset(buf, 0, foot);
  cudaMalloc(&sink, 1 << 24);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int rep = 0; rep < 2; ++rep) {
    printf("no_allocate loads           %8.0f GB/s\n", run<0>(buf, rows, sink, sms));
    printf("L1-allocating loads         %8.0f GB/s\n", run<1>(buf, rows, sink, sms));
    printf("+ prefetch.global.L1 next   %8.0f GB/s\n", run<2>(buf, rows, sink, sms));
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
