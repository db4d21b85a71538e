// L2 gather bandwidth through TMA tile::gather4 (cp.async.bulk.tensor.2d
// .tile::gather4): one elected thread per CTA keeps S gathers of 4 hashed
// rows in flight into a shared-memory ring; compares with the LDG.E.256 probe
// (gf_measure_l2_gather).  Standalone: nvcc -gencode arch=compute_100a,code=sm_100a
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                    \
  do {                                                                           \
    cudaError_t e_ = (x);                                                        \
    if (e_ != cudaSuccess) {                                                     \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                   \
    }                                                                            \
  } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W;\n}\n" ::"r"(smem_u32(b)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void gather4(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                        int r0, int r1, int r2, int r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
      : "memory");
}

template <int S>
__global__ void __launch_bounds__(32) tma_probe(const __grid_constant__ CUtensorMap map,
                                                uint32_t rows, uint32_t row_bytes, int iters,
                                                int* err, int check) {
  extern __shared__ __align__(128) unsigned char ring[];
  __shared__ uint64_t full[S];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  uint32_t x = blockIdx.x * 2654435761u + 777u;
  const uint32_t stage_bytes = 4 * row_bytes;
  int rr[S][4];
  for (int i = 0; i < iters; ++i) {
    const int s = i % S;
    if (i >= S) {
      mbar_wait(&full[s], ((i / S) - 1) & 1);
      if (check && i < 2 * S) {
        const int* d = reinterpret_cast<const int*>(ring + s * stage_bytes);
        const int cols = row_bytes / 4;
        for (int k = 0; k < 4; ++k)
          for (int c = 0; c < cols; ++c)
            if (d[k * cols + c] != rr[s][k] * cols + c) atomicAdd(err, 1);
      }
    }
    int r[4];
    for (int k = 0; k < 4; ++k) {
      x = x * 1664525u + 1013904223u;
      r[k] = static_cast<int>((x >> 3) % rows);
      rr[s][k] = r[k];
    }
    mbar_expect(&full[s], stage_bytes);
    gather4(ring + s * stage_bytes, &map, &full[s], 0, r[0], r[1], r[2], r[3]);
  }
  for (int i = iters; i < iters + S; ++i) {
    const int s = i % S;
    if (i >= S) mbar_wait(&full[s], ((i / S) - 1) & 1);
  }
}

int main(int argc, char** argv) {
  const size_t footprint = (argc > 1 ? atol(argv[1]) : 64) << 20;
  void* fnp = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q));
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fnp);
  for (int row_bytes : {32, 64, 128, 256, 512}) {
    const uint32_t cols = row_bytes / 4, rows = footprint / row_bytes;
    std::vector<int> h(static_cast<size_t>(rows) * cols);
    for (size_t i = 0; i < h.size(); ++i) h[i] = static_cast<int>(i);
    int *buf, *err;
    CK(cudaMalloc(&buf, h.size() * 4));
    CK(cudaMalloc(&err, 4));
    CK(cudaMemcpy(buf, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemset(err, 0, 4));
    CUtensorMap map;
    const cuuint64_t dims[2] = {cols, rows};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(row_bytes)};
    const cuuint32_t box[2] = {cols, 1};
    const cuuint32_t es[2] = {1, 1};
    CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_INT32, 2, buf, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      printf("row %d: encode failed %d\n", row_bytes, static_cast<int>(r));
      continue;
    }
    constexpr int S = 32;
    const int smem = S * 4 * row_bytes;
    CK(cudaFuncSetAttribute(tma_probe<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    for (int cps : {4, 8, 16}) {
      const int blocks = 148 * cps, iters = 4096;
      if (cps * (smem + 1024) > 200 * 1024) continue;
      tma_probe<S><<<blocks, 32, smem>>>(map, rows, row_bytes, 256, err, 1);
      CK(cudaDeviceSynchronize());
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      tma_probe<S><<<blocks, 32, smem>>>(map, rows, row_bytes, iters, err, 0);
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      int e = 0;
      CK(cudaMemcpy(&e, err, 4, cudaMemcpyDeviceToHost));
      const double bytes = double(blocks) * iters * 4 * row_bytes;
      printf("row %4d B  footprint %zu MB  CTAs/SM %2d  %8.0f GB/s  %.2f Grows/s  errors %d\n",
             row_bytes, footprint >> 20, cps, bytes / (ms * 1e-3) / 1e9,
             double(blocks) * iters * 4 / (ms * 1e-3) / 1e9, e);
    }
    cudaFree(buf);
    cudaFree(err);
  }
  return 0;
}
