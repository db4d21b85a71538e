// Design probe: the floor of a 3-kernel step on B200 — what C1's 18 us step
// (fwd + pass A + pass B, PDL-chained) would cost with no work at all, and
// with one cold dependent-load chain per kernel (schedule entry -> id ->
// gathered row, as the fast kernels' first iteration).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lf launch_floor_probe.cu
#include <cstdint>
#include <cstdio>

__global__ void empty_k(int* sink) {
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (sink && threadIdx.x == 1023) sink[0] = 1;
}

// three dependent loads per warp (sched -> idx -> row), like a row prologue
__global__ void chain_k(const int4* sched, const int* idx, const float* rows, float* out) {
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int4 s = __ldcg(sched + w);
  const int u = __ldcg(idx + s.y + (threadIdx.x & 31));
  const float v = __ldcg(rows + static_cast<size_t>(u) * 64 + (threadIdx.x & 31));
  if (v == 1234.5f) out[w] = v;
}

template <class F>
float time_steps(F&& step, cudaStream_t s, int n, const void* flush_buf, size_t flush_bytes) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float total = 0.f;
  for (int i = 0; i < n; ++i) {
    if (flush_buf) cudaMemsetAsync(const_cast<void*>(flush_buf), 0, flush_bytes, s);
    cudaEventRecord(a, s);
    step();
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    if (i >= 5) total += ms;
  }
  return total / (n - 5) * 1e3f;  // us
}

int main() {
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  const int warps = 2708, blocks = (warps * 32 + 255) / 256;
  int4* sched;
  int* idx;
  float *rows, *out;
  void* flush;
  const size_t fb = 256u << 20;
  cudaMalloc(&sched, sizeof(int4) * warps);
  cudaMalloc(&idx, sizeof(int) * (warps * 4 + 64));
  cudaMalloc(&rows, sizeof(float) * 64 * 4096);
  cudaMalloc(&out, sizeof(float) * warps);
  cudaMalloc(&flush, fb);
  cudaMemset(sched, 0, sizeof(int4) * warps);
  cudaMemset(idx, 0, sizeof(int) * (warps * 4 + 64));
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr.val.programmaticStreamSerializationAllowed = 1;
  auto launch = [&](bool pdl, auto kern, auto... args) {
    cudaLaunchConfig_t c = {};
    c.gridDim = dim3(blocks);
    c.blockDim = dim3(256);
    c.stream = s;
    c.attrs = pdl ? &attr : nullptr;
    c.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&c, kern, args...);
  };
  for (int pdl = 0; pdl < 2; ++pdl) {
    const float e1 = time_steps([&] { launch(pdl, empty_k, (int*)nullptr); }, s, 200, nullptr, 0);
    const float e3 = time_steps([&] { for (int k = 0; k < 3; ++k) launch(pdl, empty_k, (int*)nullptr); },
                               s, 200, nullptr, 0);
    const float c3 = time_steps([&] { for (int k = 0; k < 3; ++k) launch(pdl, chain_k, (const int4*)sched, (const int*)idx, (const float*)rows, out); },
                               s, 200, flush, fb);
    printf("pdl=%d  1 empty kernel %.2f us | 3 empty kernels %.2f us | 3 cold 3-load chains %.2f us\n",
           pdl, e1, e3, c3);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
