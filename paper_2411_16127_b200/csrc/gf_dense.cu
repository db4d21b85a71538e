// Dense layer pieces around the fused pipeline (models.hpp:58-86, 104-158):
// the X*W projections, their weight gradients X^T*dY, the GAT attention
// logits el/er and the GAT fan-in.  All deterministic (fixed reduction
// orders, split-K partials reduced in order; no atomics).
//
// gf_gemm dispatches fp32 X·W and X^T·dY to the tcgen05 3xTF32 tensor-core
// kernels (gf_tc_gemm.cu); fp64 and other shapes use the register-tiled SIMT
// GEMM below (64x64 tile, 4x4 per thread, deterministic split-K).
#include <algorithm>
#include <cstdlib>

#include "gf_device.cuh"
#include "gf_internal.cuh"

namespace gfb {

// gf_tc_gemm.cu
bool tc_gemm_eligible(int dtype, int trans_a, int64_t M, int64_t N, int64_t K, const void* A,
                      const void* C);
int tc_gemm(int64_t M, int64_t N, int64_t K, const float* A, const float* B, float* C,
            int accumulate, cudaStream_t s);
// gf_tc_gemm_tma.cu (warp-specialised TMA + tcgen05 pipeline)
bool tma_gemm_eligible(int dtype, int trans_a, int64_t M, int64_t N, int64_t K, const void* A,
                       const void* C);
int tma_gemm(int64_t M, int64_t N, int64_t K, const float* A, const float* B, float* C,
             int accumulate, cudaStream_t s, float* const* peer_c = nullptr, int n_peers = 0,
             int split_w = 0);
bool tc_gemm_tn_eligible(int dtype, int64_t M, int64_t N, int64_t K, const void* A,
                         const void* B);
int tc_gemm_tn(int64_t M, int64_t N, int64_t K, const float* A, const float* B, float* C,
               int accumulate, cudaStream_t s);

namespace {

constexpr int BM = 64, BN = 64, BK = 16;

// C_part[z] = op(A)[M x Kslice] * B[Kslice x N] over k in [k0, k1).
template <typename T, bool TRANS>
__global__ void __launch_bounds__(256) gemm_tile(int M, int N, int K, int kper,
                                                 const T* __restrict__ A, const T* __restrict__ B,
                                                 T* __restrict__ C, int accumulate,
                                                 T* __restrict__ part) {
  __shared__ T As[BK][BM + 4];
  __shared__ T Bs[BK][BN + 4];
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int k0 = blockIdx.z * kper, k1 = min(K, k0 + kper);
  T acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = T(0);
  for (int kb = k0; kb < k1; kb += BK) {
    // A tile: As[k][m] = op(A)[m0+m][kb+k]
    for (int x = tid; x < BK * BM; x += 256) {
      int k, m;
      if (TRANS) {  // A is K x M row-major: coalesced along m
        k = x / BM, m = x % BM;
      } else {  // A is M x K row-major: coalesced along k
        m = x / BK, k = x % BK;
      }
      const int gm = m0 + m, gk = kb + k;
      T val = T(0);
      if (gm < M && gk < k1) val = TRANS ? A[static_cast<size_t>(gk) * M + gm] : A[static_cast<size_t>(gm) * K + gk];
      As[k][m] = val;
    }
    for (int x = tid; x < BK * BN; x += 256) {
      const int k = x / BN, nn = x % BN;
      const int gk = kb + k, gn = n0 + nn;
      Bs[k][nn] = (gk < k1 && gn < N) ? B[static_cast<size_t>(gk) * N + gn] : T(0);
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      T a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[k][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[k][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] += a[i] * b[j];
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gm = m0 + ty * 4 + i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gn = n0 + tx * 4 + j;
      if (gn >= N) continue;
      const size_t o = static_cast<size_t>(gm) * N + gn;
      if (part) {
        part[static_cast<size_t>(blockIdx.z) * M * N + o] = acc[i][j];
      } else {
        C[o] = accumulate ? C[o] + acc[i][j] : acc[i][j];
      }
    }
  }
}

template <typename T>
__global__ void splitk_reduce(const T* __restrict__ part, int splits, size_t mn, T* __restrict__ C,
                              int accumulate) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < mn;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    T s = T(0);
    for (int z = 0; z < splits; ++z) s += part[z * mn + i];
    C[i] = accumulate ? C[i] + s : s;
  }
}

template <typename T>
int gemm_impl(int trans, int64_t M, int64_t N, int64_t K, const T* A, const T* B, T* C, int acc,
              cudaStream_t s) {
  if (M == 0 || N == 0) return GF_OK;
  const int tm = static_cast<int>((M + BM - 1) / BM), tn = static_cast<int>((N + BN - 1) / BN);
  // Split K when the output tile grid cannot fill the 148 SMs (X^T dY shapes).
  int splits = 1;
  if (static_cast<int64_t>(tm) * tn < 296 && K > 4096) {
    splits = static_cast<int>(std::min<int64_t>((K + 2047) / 2048, std::max(1, 592 / (tm * tn))));
  }
  int kper = static_cast<int>((K + splits - 1) / splits);
  kper = ((kper + BK - 1) / BK) * BK;
  splits = static_cast<int>((K + kper - 1) / kper);
  if (splits < 1) splits = 1;
  T* part = nullptr;
  if (splits > 1) GF_CHECK_CUDA(gfb::scratch_alloc(&part, sizeof(T) * splits * M * N, s));
  dim3 grid(tn, tm, splits);
  if (trans)
    gemm_tile<T, true><<<grid, 256, 0, s>>>(static_cast<int>(M), static_cast<int>(N),
                                            static_cast<int>(K), kper, A, B, C, acc, part);
  else
    gemm_tile<T, false><<<grid, 256, 0, s>>>(static_cast<int>(M), static_cast<int>(N),
                                             static_cast<int>(K), kper, A, B, C, acc, part);
  GF_CHECK_LAUNCH("gemm_tile");
  if (splits > 1) {
    const size_t mn = static_cast<size_t>(M) * N;
    splitk_reduce<T><<<static_cast<int>(std::min<size_t>(4096, (mn + 255) / 256)), 256, 0, s>>>(
        part, splits, mn, C, acc);
    GF_CHECK_LAUNCH("splitk_reduce");
    cudaFreeAsync(part, s);
  }
  return GF_OK;
}

template <typename T>
__global__ void gat_logits_kernel(int64_t n, int H, int D, const T* __restrict__ Hf,
                                  const T* __restrict__ al, const T* __restrict__ ar,
                                  T* __restrict__ el, T* __restrict__ er) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n * H;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / H;
    const int h = static_cast<int>(i % H);
    const T* x = Hf + r * H * D + static_cast<int64_t>(h) * D;
    T a = T(0), b = T(0);
    for (int d = 0; d < D; ++d) {
      a += x[d] * al[h * D + d];
      b += x[d] * ar[h * D + d];
    }
    el[i] = a;
    er[i] = b;
  }
}

template <typename T>
__global__ void gat_dh_kernel(int64_t n, int H, int D, const T* __restrict__ al,
                              const T* __restrict__ ar, const T* __restrict__ dV,
                              const T* __restrict__ del, const T* __restrict__ der,
                              T* __restrict__ dH) {
  const int64_t F = static_cast<int64_t>(H) * D;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n * F;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / F;
    const int f = static_cast<int>(i % F);
    const int h = f / D;
    dH[i] = dV[i] + del[r * H + h] * al[f] + der[r * H + h] * ar[f];
  }
}

// Stage 1 of da = Hf^T (x) dl: block b sums rows [b*R, (b+1)*R) per column.
template <typename T>
__global__ void gat_da_partial(int64_t n, int H, int D, int64_t rows_per_block,
                               const T* __restrict__ Hf, const T* __restrict__ del,
                               const T* __restrict__ der, T* __restrict__ part) {
  const int F = H * D;
  const int64_t r0 = blockIdx.x * rows_per_block, r1 = min(n, r0 + rows_per_block);
  for (int f = threadIdx.x; f < F; f += blockDim.x) {
    const int h = f / D;
    T a = T(0), b = T(0);
    for (int64_t r = r0; r < r1; ++r) {
      const T x = Hf[r * F + f];
      a += x * del[r * H + h];
      b += x * der[r * H + h];
    }
    part[static_cast<size_t>(blockIdx.x) * 2 * F + f] = a;
    part[static_cast<size_t>(blockIdx.x) * 2 * F + F + f] = b;
  }
}

template <typename T>
__global__ void gat_da_reduce(int blocks, int F, const T* __restrict__ part, T* __restrict__ dal,
                              T* __restrict__ dar) {
  for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < 2 * F; f += gridDim.x * blockDim.x) {
    T s = T(0);
    for (int b = 0; b < blocks; ++b) s += part[static_cast<size_t>(b) * 2 * F + f];
    if (f < F)
      dal[f] = s;
    else
      dar[f - F] = s;
  }
}

int grid_for(int64_t work) { return static_cast<int>(std::min<int64_t>(8192, (work + 255) / 256 + 1)); }

// ---- fp32 fast paths (D % 4 == 0, F <= 256): float4 rows, one pass ----------
// el/er: thread per (row, head), the head's D values as float4s.
__global__ void gat_logits_vec(int64_t n, int H, int D, const float* __restrict__ Hf,
                               const float* __restrict__ al, const float* __restrict__ ar,
                               float* __restrict__ el, float* __restrict__ er) {
  const int F = H * D;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n * H;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / H;
    const int h = static_cast<int>(i - r * H);
    const float4* x = reinterpret_cast<const float4*>(Hf + r * F + h * D);
    const float4* a = reinterpret_cast<const float4*>(al + h * D);
    const float4* b = reinterpret_cast<const float4*>(ar + h * D);
    float sa = 0.f, sb = 0.f;
    for (int d = 0; d < D / 4; ++d) {
      const float4 v = __ldg(x + d), p = __ldg(a + d), q = __ldg(b + d);
      sa += v.x * p.x + v.y * p.y + v.z * p.z + v.w * p.w;
      sb += v.x * q.x + v.y * q.y + v.z * q.z + v.w * q.w;
    }
    el[i] = sa;
    er[i] = sb;
  }
}

// GAT fan-in in one pass (models.hpp:143-150): dH = dV + del (x) a_l + der (x)
// a_r and the da_l / da_r column sums Hf^T del, Hf^T der.  Thread -> fixed
// float4 column chunk (blockDim = rows_per_iter * F/4), grid-stride over rows;
// per-block partials reduced in shared memory in a fixed order, then across
// blocks by gat_da_reduce_par (deterministic).
__global__ void __launch_bounds__(256) gat_fanin_vec(int64_t n, int H, int D,
                                                     const float* __restrict__ Hf,
                                                     const float* __restrict__ al,
                                                     const float* __restrict__ ar,
                                                     const float* __restrict__ dV,
                                                     const float* __restrict__ del,
                                                     const float* __restrict__ der,
                                                     float* __restrict__ dH,
                                                     float* __restrict__ part) {
  extern __shared__ float red[];  // [rows_per_iter][2F]
  const int F = H * D, C4 = F / 4;
  const int rpi = blockDim.x / C4;  // rows per iteration
  const int c = threadIdx.x % C4, rr = threadIdx.x / C4;
  const int h = (4 * c) / D;
  const float4 a = __ldg(reinterpret_cast<const float4*>(al) + c);
  const float4 b = __ldg(reinterpret_cast<const float4*>(ar) + c);
  float4 sa = make_float4(0.f, 0.f, 0.f, 0.f), sb = sa;
  if (rr < rpi) {
    for (int64_t r = blockIdx.x * static_cast<int64_t>(rpi) + rr; r < n;
         r += static_cast<int64_t>(gridDim.x) * rpi) {
      const float l = __ldg(del + r * H + h), q = __ldg(der + r * H + h);
      const float4 v = __ldg(reinterpret_cast<const float4*>(dV + r * F) + c);
      const float4 x = __ldg(reinterpret_cast<const float4*>(Hf + r * F) + c);
      reinterpret_cast<float4*>(dH + r * F)[c] =
          make_float4(v.x + l * a.x + q * b.x, v.y + l * a.y + q * b.y, v.z + l * a.z + q * b.z,
                      v.w + l * a.w + q * b.w);
      sa.x += x.x * l, sa.y += x.y * l, sa.z += x.z * l, sa.w += x.w * l;
      sb.x += x.x * q, sb.y += x.y * q, sb.z += x.z * q, sb.w += x.w * q;
    }
    float* o = red + rr * 2 * F;
    o[4 * c + 0] = sa.x, o[4 * c + 1] = sa.y, o[4 * c + 2] = sa.z, o[4 * c + 3] = sa.w;
    o[F + 4 * c + 0] = sb.x, o[F + 4 * c + 1] = sb.y, o[F + 4 * c + 2] = sb.z,
    o[F + 4 * c + 3] = sb.w;
  }
  __syncthreads();
  for (int f = threadIdx.x; f < 2 * F; f += blockDim.x) {
    float acc = 0.f;
    for (int k = 0; k < rpi; ++k) acc += red[k * 2 * F + f];  // fixed order
    part[static_cast<size_t>(blockIdx.x) * 2 * F + f] = acc;
  }
}

// Sum `blocks` partials of 2F values in a fixed order with one warp per
// output: lanes stride the partials, then a fixed-shape shuffle tree.
__global__ void gat_da_reduce_par(int blocks, int F, const float* __restrict__ part,
                                  float* __restrict__ dal, float* __restrict__ dar) {
  const int lane = threadIdx.x & 31;
  const int f = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (f >= 2 * F) return;
  float s = 0.f;
  for (int b = lane; b < blocks; b += 32) s += part[static_cast<size_t>(b) * 2 * F + f];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) {
    if (f < F)
      dal[f] = s;
    else
      dar[f - F] = s;
  }
}

}  // namespace
}  // namespace gfb

extern "C" int gf_gemm(int32_t dtype, int32_t trans_a, int64_t M, int64_t N, int64_t K,
                       const void* A, const void* B, void* C, int32_t accumulate, void* stream) {
  if (M < 0 || N < 0 || K < 0 || M >= (1LL << 31) || N >= (1LL << 31) || K >= (1LL << 31) ||
      (dtype != GF_F32 && dtype != GF_F64)) {
    gfb::set_error("gf_gemm: invalid arguments");
    return GF_ERR_INVALID;
  }
  auto s = static_cast<cudaStream_t>(stream);
  // fp32 X*W: tcgen05 3xTF32 tensor-core kernel (gf_tc_gemm.cu).  GF_GEMM_SIMT=1
  // forces the SIMT kernel (A/B measurements only).
  static const bool force_simt = [] {
    const char* e = std::getenv("GF_GEMM_SIMT");
    return e && e[0] == '1';
  }();
  static const bool no_tma = [] {
    const char* e = std::getenv("GF_GEMM_NO_TMA");
    return e && e[0] == '1';
  }();
  if (!force_simt && !no_tma && gfb::tma_gemm_eligible(dtype, trans_a, M, N, K, A, C))
    return gfb::tma_gemm(M, N, K, static_cast<const float*>(A), static_cast<const float*>(B),
                         static_cast<float*>(C), accumulate, s);
  if (!force_simt && gfb::tc_gemm_eligible(dtype, trans_a, M, N, K, A, C))
    return gfb::tc_gemm(M, N, K, static_cast<const float*>(A), static_cast<const float*>(B),
                        static_cast<float*>(C), accumulate, s);
  if (!force_simt && trans_a && gfb::tc_gemm_tn_eligible(dtype, M, N, K, A, B))
    return gfb::tc_gemm_tn(M, N, K, static_cast<const float*>(A), static_cast<const float*>(B),
                           static_cast<float*>(C), accumulate, s);
  if (dtype == GF_F32)
    return gfb::gemm_impl<float>(trans_a, M, N, K, static_cast<const float*>(A),
                                 static_cast<const float*>(B), static_cast<float*>(C), accumulate, s);
  return gfb::gemm_impl<double>(trans_a, M, N, K, static_cast<const double*>(A),
                                static_cast<const double*>(B), static_cast<double*>(C), accumulate,
                                s);
}

extern "C" int gf_gat_logits(int32_t dtype, int64_t n, int32_t H, int32_t D, const void* Hf,
                             const void* a_l, const void* a_r, void* el, void* er, void* stream) {
  if (n < 0 || H < 1 || D < 1 || (dtype != GF_F32 && dtype != GF_F64)) {
    gfb::set_error("gf_gat_logits: invalid arguments");
    return GF_ERR_INVALID;
  }
  if (n == 0) return GF_OK;
  auto s = static_cast<cudaStream_t>(stream);
  const int grid = gfb::grid_for(n * H);
  const bool vec = D % 4 == 0 && ((reinterpret_cast<uintptr_t>(Hf) | reinterpret_cast<uintptr_t>(a_l) |
                                   reinterpret_cast<uintptr_t>(a_r)) & 15u) == 0;
  if (dtype == GF_F32 && vec) {
    const int g2 = static_cast<int>(std::min<int64_t>(148 * 32, (n * H + 255) / 256));
    gfb::gat_logits_vec<<<g2, 256, 0, s>>>(n, H, D, static_cast<const float*>(Hf),
                                           static_cast<const float*>(a_l),
                                           static_cast<const float*>(a_r), static_cast<float*>(el),
                                           static_cast<float*>(er));
  } else if (dtype == GF_F32)
    gfb::gat_logits_kernel<float><<<grid, 256, 0, s>>>(
        n, H, D, static_cast<const float*>(Hf), static_cast<const float*>(a_l),
        static_cast<const float*>(a_r), static_cast<float*>(el), static_cast<float*>(er));
  else
    gfb::gat_logits_kernel<double><<<grid, 256, 0, s>>>(
        n, H, D, static_cast<const double*>(Hf), static_cast<const double*>(a_l),
        static_cast<const double*>(a_r), static_cast<double*>(el), static_cast<double*>(er));
  GF_CHECK_LAUNCH("gat_logits");
  return GF_OK;
}

namespace {
template <typename T>
int fanin_impl(int64_t n, int H, int D, const T* Hf, const T* al, const T* ar, const T* dV,
               const T* del, const T* der, T* dH, T* dal, T* dar, cudaStream_t s) {
  const int F = H * D;
  if constexpr (sizeof(T) == 4) {
    const bool al16 = ((reinterpret_cast<uintptr_t>(Hf) | reinterpret_cast<uintptr_t>(al) |
                        reinterpret_cast<uintptr_t>(ar) | reinterpret_cast<uintptr_t>(dV) |
                        reinterpret_cast<uintptr_t>(dH)) & 15u) == 0;
    if (D % 4 == 0 && F <= 256 && al16) {
      const int c4 = F / 4, rpi = 256 / c4;
      const int threads = rpi * c4;
      const int blocks = static_cast<int>(std::max<int64_t>(
          1, std::min<int64_t>(148 * 8, (n + rpi - 1) / rpi)));
      const size_t smem = sizeof(float) * rpi * 2 * F;
      T* part = nullptr;
      GF_CHECK_CUDA(gfb::scratch_alloc(&part, sizeof(T) * blocks * 2 * F, s));
      gfb::gat_fanin_vec<<<blocks, threads, smem, s>>>(n, H, D, Hf, al, ar, dV, del, der, dH, part);
      GF_CHECK_LAUNCH("gat_fanin_vec");
      gfb::gat_da_reduce_par<<<(2 * F * 32 + 255) / 256, 256, 0, s>>>(blocks, F, part, dal, dar);
      GF_CHECK_LAUNCH("gat_da_reduce_par");
      cudaFreeAsync(part, s);
      return GF_OK;
    }
  }
  gfb::gat_dh_kernel<T><<<gfb::grid_for(n * F), 256, 0, s>>>(n, H, D, al, ar, dV, del, der, dH);
  GF_CHECK_LAUNCH("gat_dh");
  const int64_t rpb = 512;
  const int blocks = static_cast<int>(std::max<int64_t>(1, (n + rpb - 1) / rpb));
  T* part = nullptr;
  GF_CHECK_CUDA(gfb::scratch_alloc(&part, sizeof(T) * blocks * 2 * F, s));
  gfb::gat_da_partial<T><<<blocks, 128, 0, s>>>(n, H, D, rpb, Hf, del, der, part);
  GF_CHECK_LAUNCH("gat_da_partial");
  gfb::gat_da_reduce<T><<<(2 * F + 255) / 256, 256, 0, s>>>(blocks, F, part, dal, dar);
  GF_CHECK_LAUNCH("gat_da_reduce");
  cudaFreeAsync(part, s);
  return GF_OK;
}
}  // namespace

extern "C" int gf_gat_fanin(int32_t dtype, int64_t n, int32_t H, int32_t D, const void* Hf,
                            const void* a_l, const void* a_r, const void* dV, const void* del,
                            const void* der, void* dH, void* da_l, void* da_r, void* stream) {
  if (n < 0 || H < 1 || D < 1 || (dtype != GF_F32 && dtype != GF_F64)) {
    gfb::set_error("gf_gat_fanin: invalid arguments");
    return GF_ERR_INVALID;
  }
  auto s = static_cast<cudaStream_t>(stream);
  if (dtype == GF_F32)
    return fanin_impl<float>(n, H, D, static_cast<const float*>(Hf), static_cast<const float*>(a_l),
                             static_cast<const float*>(a_r), static_cast<const float*>(dV),
                             static_cast<const float*>(del), static_cast<const float*>(der),
                             static_cast<float*>(dH), static_cast<float*>(da_l),
                             static_cast<float*>(da_r), s);
  return fanin_impl<double>(n, H, D, static_cast<const double*>(Hf),
                            static_cast<const double*>(a_l), static_cast<const double*>(a_r),
                            static_cast<const double*>(dV), static_cast<const double*>(del),
                            static_cast<const double*>(der), static_cast<double*>(dH),
                            static_cast<double*>(da_l), static_cast<double*>(da_r), s);
}

// Projection fused with its all-gather: C = A·B written to
// n_dst row-major M x N destinations, dst[0] local and dst[1..] the same rows
// of the other ranks' tables through peer-mapped addresses — the TMA-store
// epilogue sends every finished tile to all of them, so the exchange
// overlaps the remaining tiles' MMAs instead of following the GEMM.
extern "C" int gf_gemm_bcast(int32_t dtype, int64_t M, int64_t N, int64_t K, const void* A,
                             const void* B, void* const* dst, int32_t n_dst, void* stream) {
  if (!dst || n_dst < 1 || n_dst > 8 || M < 0 || N < 0 || K < 0 || M >= (1LL << 31) ||
      N >= (1LL << 31) || K >= (1LL << 31)) {
    gfb::set_error("gf_gemm_bcast: invalid arguments (1 <= n_dst <= 8)");
    return GF_ERR_INVALID;
  }
  for (int i = 0; i < n_dst; ++i)
    if (!dst[i] || (reinterpret_cast<uintptr_t>(dst[i]) & 15u)) {
      gfb::set_error("gf_gemm_bcast: destinations must be non-null and 16 B aligned");
      return GF_ERR_INVALID;
    }
  if (M == 0 || N == 0) return GF_OK;
  if (!gfb::tma_gemm_eligible(dtype, 0, M, N, K, A, dst[0]) || N % 32) {
    gfb::set_error("gf_gemm_bcast: needs fp32, K % 4 == 0, N % 32 == 0, 16 B aligned operands");
    return GF_ERR_INVALID;
  }
  float* peers[8];
  for (int i = 1; i < n_dst; ++i) peers[i - 1] = static_cast<float*>(dst[i]);
  return gfb::tma_gemm(M, N, K, static_cast<const float*>(A), static_cast<const float*>(B),
                       static_cast<float*>(dst[0]), 0, static_cast<cudaStream_t>(stream), peers,
                       n_dst - 1);
}

// C = A·B with column block j (N / n_dst wide) stored to dst[j] (row-major M x
// N / n_dst): the GT / AGNN projections X·[W_q | W_k | W_v] as ONE tcgen05
// GEMM (X read once) whose TMA epilogue writes Q, K and V into their own
// tables (models.hpp:116-125).
extern "C" int gf_gemm_split(int32_t dtype, int64_t M, int64_t N, int64_t K, const void* A,
                             const void* B, void* const* dst, int32_t n_dst, void* stream) {
  if (!dst || n_dst < 1 || n_dst > 8 || M < 0 || N < 0 || K < 0 || M >= (1LL << 31) ||
      N >= (1LL << 31) || K >= (1LL << 31) || (n_dst > 0 && N % n_dst)) {
    gfb::set_error("gf_gemm_split: invalid arguments (1 <= n_dst <= 8, N % n_dst == 0)");
    return GF_ERR_INVALID;
  }
  for (int i = 0; i < n_dst; ++i)
    if (!dst[i] || (reinterpret_cast<uintptr_t>(dst[i]) & 15u)) {
      gfb::set_error("gf_gemm_split: destinations must be non-null and 16 B aligned");
      return GF_ERR_INVALID;
    }
  if (M == 0 || N == 0) return GF_OK;
  const int64_t w = N / n_dst;
  if (!gfb::tma_gemm_eligible(dtype, 0, M, N, K, A, dst[0]) || w % 32) {
    gfb::set_error("gf_gemm_split: needs fp32, K % 4 == 0, (N / n_dst) % 32 == 0, 16 B aligned");
    return GF_ERR_INVALID;
  }
  float* rest[8];
  for (int i = 1; i < n_dst; ++i) rest[i - 1] = static_cast<float*>(dst[i]);
  return gfb::tma_gemm(M, N, K, static_cast<const float*>(A), static_cast<const float*>(B),
                       static_cast<float*>(dst[0]), 0, static_cast<cudaStream_t>(stream), rest,
                       n_dst - 1, static_cast<int>(w));
}
