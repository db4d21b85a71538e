// Measured L2 gather bandwidth: the denominator for the gather kernels whose
// node tables are L2-resident (C4: V 60 MB + el 7.5 MB), where the HBM
// roofline is exceeded by design (SURVEY §7 hard part 5).  Same instruction
// as the hot kernels' gathers (LDG.E.256 non-coherent, L1 no-allocate, L2
// evict-last), rows of `row_bytes` of a `footprint`-byte buffer in a hashed
// order, all SMs, after one warm-up pass.
#include <algorithm>

#include "gf_device.cuh"
#include "gf_internal.cuh"

namespace gfb {
namespace {

// Lanes in groups of `cpr` (chunks per row) read the consecutive 32 B chunks
// of one randomly chosen row, like the hot kernels' per-edge row gathers
// (GAT 8x8: 8 lanes x 32 B = one 256 B V row).
__global__ void __launch_bounds__(256) l2_gather_probe(const float* __restrict__ buf,
                                                       uint32_t rows, uint32_t cpr,
                                                       uint32_t per_thread,
                                                       float* __restrict__ sink) {
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t grp = tid / cpr, sub = tid % cpr;
  float acc = 0.f;
  uint32_t x = grp * 2654435761u + 12345u;
#pragma unroll 4
  for (uint32_t i = 0; i < per_thread; ++i) {
    x = x * 1664525u + 1013904223u;  // the group's LCG walk over the rows
    float v[8];
    ld_gather<float, 32>(buf + (static_cast<size_t>(x % rows) * cpr + sub) * 8, v);
    acc += v[0] + v[7];
  }
  if (acc == 12345.678f) sink[tid] = acc;  // keeps the loads alive
}

}  // namespace
}  // namespace gfb

extern "C" int gf_measure_l2_gather(size_t footprint_bytes, int32_t row_bytes, int32_t iters,
                                    double* gbs_out, void* stream) {
  if (!gbs_out || footprint_bytes < 32 || iters < 1 || row_bytes < 32 || row_bytes % 32 ||
      row_bytes > 1024 || (32 % (row_bytes / 32) && (row_bytes / 32) % 32)) {
    gfb::set_error("gf_measure_l2_gather: invalid arguments");
    return GF_ERR_INVALID;
  }
  auto s = static_cast<cudaStream_t>(stream);
  const uint32_t cpr = static_cast<uint32_t>(row_bytes / 32);
  const uint32_t rows = static_cast<uint32_t>(footprint_bytes / row_bytes);
  const uint32_t chunks = rows * cpr;
  const int blocks = 148 * 8, threads = 256;
  const uint32_t per_thread = 1024;
  float *buf = nullptr, *sink = nullptr;
  GF_CHECK_CUDA(cudaMalloc(&buf, static_cast<size_t>(chunks) * 32));
  GF_CHECK_CUDA(cudaMalloc(&sink, sizeof(float) * blocks * threads));
  cudaMemsetAsync(buf, 0, static_cast<size_t>(chunks) * 32, s);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  gfb::l2_gather_probe<<<blocks, threads, 0, s>>>(buf, rows, cpr, per_thread, sink);  // warm L2
  cudaEventRecord(a, s);
  for (int i = 0; i < iters; ++i)
    gfb::l2_gather_probe<<<blocks, threads, 0, s>>>(buf, rows, cpr, per_thread, sink);
  cudaEventRecord(b, s);
  int rc = GF_OK;
  if (cudaEventSynchronize(b) != cudaSuccess) {
    gfb::set_error("gf_measure_l2_gather: kernel failed");
    rc = GF_ERR_CUDA;
  }
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  const double bytes = 32.0 * blocks * threads * static_cast<double>(per_thread) * iters;
  *gbs_out = ms > 0 ? bytes / (ms * 1e-3) / 1e9 : 0.0;
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(buf);
  cudaFree(sink);
  return rc;
}

// Scatter-reduction probe (design measurement, not on the product path): per
// CSC edge u -> v, 8 lanes add one fp32 per head into table[v][0..7] (the
// shape of a GAT der[v] update issued from a source-owned pass), as scalar
// red.add.f32 (mode 0), red.add.v4.f32 from 2 lanes (mode 1), plain stores
// (mode 2) or 32 B gathers (mode 3).  Warp per column, 4 edges per step.
namespace gfb {
namespace {
__global__ void __launch_bounds__(256) scatter_probe(int n, const int32_t* __restrict__ ptr,
                                                     const int32_t* __restrict__ idx,
                                                     float* __restrict__ table, int mode,
                                                     float* __restrict__ sink) {
  const int lane = threadIdx.x & 31;
  const int sub = lane >> 3, h = lane & 7;
  float acc = 0.f;
  for (int u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < n;
       u += (gridDim.x * blockDim.x) >> 5) {
    const int b = __ldg(ptr + u), e = __ldg(ptr + u + 1);
    for (int j = b + sub; j < e; j += 4) {
      const int v = ld_idx(idx + j);
      float* p = table + static_cast<size_t>(v) * 8;
      const float x = 1e-3f * (h + 1);
      if (mode == 0) {
        asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p + h), "f"(x) : "memory");
      } else if (mode == 1) {
        if ((h & 3) == 0)
          asm volatile("red.global.add.v4.f32 [%0], {%1,%1,%1,%1};" ::"l"(p + h), "f"(x) : "memory");
      } else if (mode == 4) {
        unsigned long long* q = reinterpret_cast<unsigned long long*>(table) + static_cast<size_t>(v) * 8;
        asm volatile("red.global.add.u64 [%0], %1;" ::"l"(q + h), "l"(static_cast<unsigned long long>(h + 1)) : "memory");
      } else if (mode == 2) {
        p[h] = x;
      } else {
        acc += __ldg(p + h);
      }
    }
  }
  if (acc == 12345.678f) sink[threadIdx.x] = acc;
}
__global__ void policy_word_probe(uint64_t* out) { out[0] = pol_keep(); }

}  // namespace
}  // namespace gfb

extern "C" int gf_l2_policy_word(uint64_t* device_word, uint64_t* host_word) {
  if (!device_word || !host_word) {
    gfb::set_error("gf_l2_policy_word: null output");
    return GF_ERR_INVALID;
  }
  *host_word = gfb::kPolicyEvictLast;
  uint64_t* d = nullptr;
  GF_CHECK_CUDA(cudaMalloc(&d, sizeof(uint64_t)));
  gfb::policy_word_probe<<<1, 1>>>(d);
  const int rc = cudaMemcpy(device_word, d, sizeof(uint64_t), cudaMemcpyDeviceToHost) == cudaSuccess
                     ? GF_OK : GF_ERR_CUDA;
  cudaFree(d);
  if (rc) gfb::set_error("gf_l2_policy_word: kernel failed");
  return rc;
}

extern "C" int gf_probe_scatter(int64_t n, const int32_t* csc_ptr, const int32_t* csc_row,
                                float* table, int32_t mode, int32_t iters, float* ms_out,
                                void* stream) {
  auto s = static_cast<cudaStream_t>(stream);
  float* sink = nullptr;
  GF_CHECK_CUDA(cudaMalloc(&sink, sizeof(float) * 256));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int blocks = 148 * 8;
  gfb::scatter_probe<<<blocks, 256, 0, s>>>(static_cast<int>(n), csc_ptr, csc_row, table, mode, sink);
  cudaEventRecord(a, s);
  for (int i = 0; i < iters; ++i)
    gfb::scatter_probe<<<blocks, 256, 0, s>>>(static_cast<int>(n), csc_ptr, csc_row, table, mode,
                                              sink);
  cudaEventRecord(b, s);
  int rc = cudaEventSynchronize(b) == cudaSuccess ? GF_OK : GF_ERR_CUDA;
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  *ms_out = ms / iters;
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(sink);
  if (rc) gfb::set_error("gf_probe_scatter: kernel failed");
  return rc;
}
