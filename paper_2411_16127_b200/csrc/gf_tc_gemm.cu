// K0 — the dense projection C = A·B (X·W) on the 5th-generation tensor cores
// (tcgen05.mma kind::tf32, accumulator in TMEM), with the 3xTF32 split so the
// fp32 result keeps ~fp32 accuracy (plain TF32 would give ~5e-4 relative per
// dot at K = 64..128, failing the 1e-4 parity bar; SURVEY §7 hard part 1):
//     a = a_hi + a_lo,  b = b_hi + b_lo  (hi = top 19 bits, lo = remainder)
//     a·b ≈ a_hi·b_hi + a_hi·b_lo + a_lo·b_hi            (3 MMAs per k-step)
// Replaces the reference's naive serial matmul (models.hpp:58-72) on the
// X·W / QKV projection path of conv_forward (models.hpp:119-128).
//
// One CTA of 128 threads per 128-row tile of A and one N tile (N <= 256,
// multiple of 16).  K is streamed in chunks of 32: every thread converts one
// A row (and B columns) to hi/lo tf32 and stores them in shared memory in the
// UMMA K-major "interleave" canonical layout (8-row x 16-byte core matrices);
// after fence.proxy.async + barrier one elected thread issues the
// tcgen05.mma instructions (M=128, N=n_tile, K=8 each) and commits to an
// mbarrier.  The epilogue reads the accumulator with tcgen05.ld (32x32b:
// thread = row) and writes C.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "gf_internal.cuh"

namespace gfb {
namespace {

constexpr int TC_M = 128;   // rows per CTA (UMMA M)
constexpr int TC_KC = 32;   // K elements per smem chunk (4 MMA k-steps of 8)
constexpr int TC_THREADS = 128;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// UMMA shared-memory matrix descriptor, K-major, no swizzle (cute
// SmemDescriptor: start>>4 [0,14), LBO>>4 [16,30), SBO>>4 [32,46),
// version=1 [46,48), layout SWIZZLE_NONE=0 [61,64)).
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((addr >> 4) & 0x3FFF) |
         (static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

// Instruction descriptor: D f32, A/B tf32, both K-major, N>>3, M>>4.
__host__ __device__ constexpr uint32_t instr_desc_tf32(int m, int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(m >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void split_tf32(float x, float& hi, float& lo) {
  hi = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
  lo = x - hi;
#if GF_TF32_RAW_HI  // experiment: hand the tensor core the raw fp32 as "hi"
  hi = x;
#endif
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(bar),
      "r"(phase)
      : "memory");
}

// tcgen05.ld (32x32b, 16 columns: thread = TMEM lane) and its wait in ONE asm
// statement: as separate statements the compiler may consume the destination
// registers before tcgen05.wait::ld (it did: the drained values read as 0).
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
}

// C[M x N] = A[M x K] * B[K x N], all row-major fp32.  1-D grid over
// (m tile, n tile) with the n tile fastest, so the CTAs that share an A tile
// run together and all but the first read it from L2.  The next 32-K chunk
// of A and B is loaded into registers while the tensor core works on the
// current one (software pipelining across the smem stage).
__global__ void __launch_bounds__(TC_THREADS, 1)
    tc_gemm_3xtf32(int M, int N, int K, int n_tile, const float* __restrict__ A,
                   const float* __restrict__ B, float* __restrict__ C, int accumulate) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int n_tiles = N / n_tile;
  const int m0 = (blockIdx.x / n_tiles) * TC_M, n0 = (blockIdx.x % n_tiles) * n_tile;
  const int NT = n_tile;
  // smem: A_hi, A_lo (128 x 32 tf32 each, 16 KB), B_hi, B_lo (NT x 32, NT*128 B each)
  float* a_hi = reinterpret_cast<float*>(smem);
  float* a_lo = a_hi + TC_M * TC_KC;
  float* b_hi = a_lo + TC_M * TC_KC;
  float* b_lo = b_hi + NT * TC_KC;
  const uint32_t ncols = NT <= 32 ? 32 : NT <= 64 ? 64 : NT <= 128 ? 128 : 256;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  const uint32_t idesc = instr_desc_tf32(TC_M, NT);
  // Core-matrix geometry (bytes): A core (rg, kc) at (kc*16 + rg)*128;
  // B core (ng, kc) at (kc*NT/8 + ng)*128.  One MMA k-step = 2 kc.
  const uint32_t lbo_a = 16 * 128, lbo_b = (NT / 8) * 128, sbo = 128;

  const int row = m0 + t;
  // register stage: thread t holds row m0+t of the A chunk and columns
  // n0+t, n0+t+128 of the B chunk
  float4 av[TC_KC / 4];
  float bv[2][TC_KC];
  auto load_chunk = [&](int k0) {
#pragma unroll
    for (int kc = 0; kc < TC_KC / 4; ++kc) {
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      const int k = k0 + kc * 4;
      if (row < M) {
        const float* src = A + static_cast<size_t>(row) * K + k;
        if (k + 3 < K) {
          v = *reinterpret_cast<const float4*>(src);
        } else {
          v.x = k < K ? src[0] : 0.f;
          v.y = k + 1 < K ? src[1] : 0.f;
          v.z = k + 2 < K ? src[2] : 0.f;
        }
      }
      av[kc] = v;
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int n = t + i * TC_THREADS;
#pragma unroll
      for (int j = 0; j < TC_KC; ++j) {
        const int k = k0 + j;
        bv[i][j] = (n < NT && k < K) ? __ldg(B + static_cast<size_t>(k) * N + n0 + n) : 0.f;
      }
    }
  };

  uint32_t phase = 0;
  load_chunk(0);
  for (int k0 = 0; k0 < K; k0 += TC_KC) {
    // ---- A chunk (row m0+t) and B chunk (columns t, t+128) -> hi/lo tf32 in smem
#pragma unroll
    for (int kc = 0; kc < TC_KC / 4; ++kc) {
      const float4 v = av[kc];
      float4 h, l;
      split_tf32(v.x, h.x, l.x);
      split_tf32(v.y, h.y, l.y);
      split_tf32(v.z, h.z, l.z);
      split_tf32(v.w, h.w, l.w);
      const int off = (kc * 16 + t / 8) * 32 + (t % 8) * 4;  // floats
      *reinterpret_cast<float4*>(a_hi + off) = h;
      *reinterpret_cast<float4*>(a_lo + off) = l;
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int n = t + i * TC_THREADS;
      if (n >= NT) continue;
#pragma unroll
      for (int kc = 0; kc < TC_KC / 4; ++kc) {
        float4 h, l;
        split_tf32(bv[i][kc * 4 + 0], h.x, l.x);
        split_tf32(bv[i][kc * 4 + 1], h.y, l.y);
        split_tf32(bv[i][kc * 4 + 2], h.z, l.z);
        split_tf32(bv[i][kc * 4 + 3], h.w, l.w);
        const int off = (kc * (NT / 8) + n / 8) * 32 + (n % 8) * 4;
        *reinterpret_cast<float4*>(b_hi + off) = h;
        *reinterpret_cast<float4*>(b_lo + off) = l;
      }
    }
    // generic-proxy smem writes -> visible to the tensor core (async proxy)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (t == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t ah = smem_u32(a_hi), al = smem_u32(a_lo), bh = smem_u32(b_hi),
                     bl = smem_u32(b_lo);
#pragma unroll
      for (int s = 0; s < TC_KC / 8; ++s) {
        const uint32_t da = s * 2 * lbo_a, db = s * 2 * lbo_b;
        const uint64_t dah = smem_desc(ah + da, lbo_a, sbo), dal = smem_desc(al + da, lbo_a, sbo);
        const uint64_t dbh = smem_desc(bh + db, lbo_b, sbo), dbl = smem_desc(bl + db, lbo_b, sbo);
        mma_tf32(tmem, dah, dbh, idesc, (k0 > 0 || s > 0) ? 1u : 0u);
        mma_tf32(tmem, dah, dbl, idesc, 1u);
        mma_tf32(tmem, dal, dbh, idesc, 1u);
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(&mbar)) : "memory");
    }
    if (k0 + TC_KC < K) load_chunk(k0 + TC_KC);  // in flight under the MMAs
    mbar_wait(smem_u32(&mbar), phase);  // MMAs done: smem reusable, accumulator final
    phase ^= 1;
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

  // ---- epilogue: warp w reads TMEM lanes [32w, 32w+32): thread = row
  const uint32_t lane_base = static_cast<uint32_t>(warp * 32) << 16;
  for (int c = 0; c < NT; c += 16) {
    uint32_t r[16];
    tmem_ld16(tmem + lane_base + c, r);
    if (row < M) {
      float* dst = C + static_cast<size_t>(row) * N + n0 + c;
#pragma unroll
      for (int j = 0; j < 16; j += 4) {
        float4 o = make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]),
                               __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3]));
        if (accumulate) {
          const float4 p = *reinterpret_cast<const float4*>(dst + j);
          o.x += p.x, o.y += p.y, o.z += p.z, o.w += p.w;
        }
        *reinterpret_cast<float4*>(dst + j) = o;
      }
    }
  }
  (void)lane;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(ncols));
}

// ---------------------------------------------------------------------------
// Weight gradients C[M x N] = A^T·B with A = X (K x M) and B = dY (K x N), both
// row-major, K = number of nodes (millions), M = F_in (<= 128), N = F_out
// (<= 256).  The staging transposes: thread m loads X[k..k+3][m] (coalesced
// across threads: one 512 B row segment per k) and stores the 4 K values as
// one float4 in the same K-major core-matrix layout as tc_gemm_3xtf32, so both
// kernels issue identical K-major UMMA descriptors.  (MN-major descriptors
// were tried first and produced all-zero accumulators on B200.)
// Deterministic split-K: CTA z owns K rows [z*Ks, (z+1)*Ks) and writes its
// M x N partial; a fixed-order reduction sums the partials.
__global__ void __launch_bounds__(TC_THREADS, 3)
    tc_gemm_tn_3xtf32(int M, int N, int K, int ks, const float* __restrict__ A,
                      const float* __restrict__ B, float* __restrict__ part) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int t = threadIdx.x, warp = t >> 5;
  const int NP = N;                 // multiple of 16 (UMMA N)
  float* a_hi = reinterpret_cast<float*>(smem);
  float* a_lo = a_hi + TC_M * TC_KC;
  float* b_hi = a_lo + TC_M * TC_KC;
  float* b_lo = b_hi + NP * TC_KC;
  const uint32_t ncols = NP <= 32 ? 32 : NP <= 64 ? 64 : NP <= 128 ? 128 : 256;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  const uint32_t idesc = instr_desc_tf32(TC_M, NP);  // both operands K-major
  const uint32_t lbo_a = 16 * 128, lbo_b = (NP / 8) * 128, sbo = 128;
  // The launcher caps the K slice at kTnMaxSlice rows: the tensor core's
  // truncating accumulation then spans <= 1024 products per element, and the
  // fp32 partials are summed round-to-nearest in a fixed order (tn_reduce*).
  const int kb = blockIdx.x * ks, ke = min(K, kb + ks);
  uint32_t phase = 0;
  const uint32_t lane_base = static_cast<uint32_t>(warp * 32) << 16;
  // register stage (next chunk prefetched under the current MMAs): thread t
  // holds column t of X^T (= X[k][t]) and columns t, t+128 of dY
  float xa[TC_KC], yb[2][TC_KC];
  auto load_chunk = [&](int k0) {
#pragma unroll
    for (int j = 0; j < TC_KC; ++j) {
      const int k = k0 + j;
      xa[j] = (t < M && k < ke) ? __ldg(A + static_cast<size_t>(k) * M + t) : 0.f;
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int n = t + i * TC_THREADS;
#pragma unroll
      for (int j = 0; j < TC_KC; ++j) {
        const int k = k0 + j;
        yb[i][j] = (n < NP && k < ke) ? __ldg(B + static_cast<size_t>(k) * N + n) : 0.f;
      }
    }
  };
  load_chunk(kb);
  for (int k0 = kb; k0 < ke; k0 += TC_KC) {
    // A^T chunk: thread t = output row m, 4 K rows per float4 (K-major cores)
#pragma unroll
    for (int kc = 0; kc < TC_KC / 4; ++kc) {
      float4 h, l;
      split_tf32(xa[kc * 4 + 0], h.x, l.x);
      split_tf32(xa[kc * 4 + 1], h.y, l.y);
      split_tf32(xa[kc * 4 + 2], h.z, l.z);
      split_tf32(xa[kc * 4 + 3], h.w, l.w);
      const int off = (kc * 16 + t / 8) * 32 + (t % 8) * 4;
      *reinterpret_cast<float4*>(a_hi + off) = h;
      *reinterpret_cast<float4*>(a_lo + off) = l;
    }
    // dY chunk: column n of B, 4 K rows per float4 (same layout as the NN kernel)
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int n = t + i * TC_THREADS;
      if (n >= NP) continue;
#pragma unroll
      for (int kc = 0; kc < TC_KC / 4; ++kc) {
        float4 h, l;
        split_tf32(yb[i][kc * 4 + 0], h.x, l.x);
        split_tf32(yb[i][kc * 4 + 1], h.y, l.y);
        split_tf32(yb[i][kc * 4 + 2], h.z, l.z);
        split_tf32(yb[i][kc * 4 + 3], h.w, l.w);
        const int off = (kc * (NP / 8) + n / 8) * 32 + (n % 8) * 4;
        *reinterpret_cast<float4*>(b_hi + off) = h;
        *reinterpret_cast<float4*>(b_lo + off) = l;
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (t == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t ah = smem_u32(a_hi), al = smem_u32(a_lo), bh = smem_u32(b_hi),
                     bl = smem_u32(b_lo);
#pragma unroll
      for (int s = 0; s < TC_KC / 8; ++s) {
        const uint32_t da = s * 2 * lbo_a, db = s * 2 * lbo_b;
        const uint64_t dah = smem_desc(ah + da, lbo_a, sbo), dal = smem_desc(al + da, lbo_a, sbo);
        const uint64_t dbh = smem_desc(bh + db, lbo_b, sbo), dbl = smem_desc(bl + db, lbo_b, sbo);
        mma_tf32(tmem, dah, dbh, idesc, (k0 > kb || s > 0) ? 1u : 0u);
        mma_tf32(tmem, dah, dbl, idesc, 1u);
        mma_tf32(tmem, dal, dbh, idesc, 1u);
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(&mbar)) : "memory");
    }
    if (k0 + TC_KC < ke) load_chunk(k0 + TC_KC);  // in flight under the MMAs
    mbar_wait(smem_u32(&mbar), phase);
    phase ^= 1;
  }
  // epilogue: TMEM -> this split's partial (thread = output row m)
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int row = t;
  float* dst = part + static_cast<size_t>(blockIdx.x) * M * N + static_cast<size_t>(row) * N;
  for (int c = 0; c < NP; c += 16) {
    uint32_t r[16];
    tmem_ld16(tmem + lane_base + c, r);
    if (row < M) {
#pragma unroll
      for (int j = 0; j < 16; j += 4)
        *reinterpret_cast<float4*>(dst + c + j) =
            make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]),
                        __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3]));
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(ncols));
}

__global__ void tn_reduce(const float* __restrict__ part, int splits, size_t mn,
                          float* __restrict__ C, int accumulate) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < mn;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    float s = 0.f;
    for (int z = 0; z < splits; ++z) s += part[z * mn + i];  // fixed order: deterministic
    C[i] = accumulate ? C[i] + s : s;
  }
}

// First level of the fixed-order reduction for many splits: block (x, g)
// sums splits [g*per, (g+1)*per) of its elements into part2[g].
__global__ void tn_reduce_group(const float* __restrict__ part, int splits, int per, size_t mn,
                                float* __restrict__ part2) {
  const int g = blockIdx.y;
  const int z0 = g * per, z1 = min(splits, z0 + per);
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < mn;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    float s = 0.f;
    for (int z = z0; z < z1; ++z) s += part[z * mn + i];
    part2[g * mn + i] = s;
  }
}

}  // namespace

bool tc_gemm_tn_eligible(int dtype, int64_t M, int64_t N, int64_t K, const void* A,
                         const void* B) {
  if (dtype != GF_F32 || M <= 0 || M > TC_M || M % 4 || N <= 0 || N > 256 || N % 16 ||
      K <= 0)
    return false;
  return ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15u) == 0;
}

int tc_gemm_tn(int64_t M, int64_t N, int64_t K, const float* A, const float* B, float* C,
               int accumulate, cudaStream_t s) {
  // K slices: enough CTAs for ~4 per SM, each <= kTnMaxSlice rows (a multiple
  // of the 32-row chunk); every CTA writes one fp32 partial
  constexpr int64_t kTnMaxSlice = 1024;
  int64_t ks = (K + 148 * 4 - 1) / (148 * 4);
  ks = std::min<int64_t>(kTnMaxSlice, std::max<int64_t>(TC_KC, (ks + TC_KC - 1) / TC_KC * TC_KC));
  const int splits = static_cast<int>((K + ks - 1) / ks);
  constexpr int kPer = 64;  // splits summed per first-level group
  const int groups = splits > kPer ? (splits + kPer - 1) / kPer : 0;
  float* part = nullptr;
  GF_CHECK_CUDA(gfb::scratch_alloc(&part, sizeof(float) * (splits + groups) * M * N, s));
  const size_t smem = sizeof(float) * (2 * TC_M * TC_KC + 2 * static_cast<size_t>(N) * TC_KC);
  GF_CHECK_CUDA(cudaFuncSetAttribute(tc_gemm_tn_3xtf32,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
  tc_gemm_tn_3xtf32<<<splits, TC_THREADS, smem, s>>>(static_cast<int>(M), static_cast<int>(N),
                                                     static_cast<int>(K), static_cast<int>(ks), A,
                                                     B, part);
  GF_CHECK_LAUNCH("tc_gemm_tn_3xtf32");
  const size_t mn = static_cast<size_t>(M) * N;
  const int rblocks = static_cast<int>(std::min<size_t>(1024, (mn + 255) / 256));
  if (groups) {  // two fixed-order levels: groups of kPer splits, then the groups
    float* part2 = part + static_cast<size_t>(splits) * mn;
    tn_reduce_group<<<dim3(rblocks, groups), 256, 0, s>>>(part, splits, kPer, mn, part2);
    GF_CHECK_LAUNCH("tn_reduce_group");
    tn_reduce<<<rblocks, 256, 0, s>>>(part2, groups, mn, C, accumulate);
  } else {
    tn_reduce<<<rblocks, 256, 0, s>>>(part, splits, mn, C, accumulate);
  }
  GF_CHECK_LAUNCH("tn_reduce");
  cudaFreeAsync(part, s);
  return GF_OK;
}

// Tensor-core eligibility: fp32, C = A·B (not transposed), N a multiple of 16,
// 16-byte aligned rows.  N is tiled by the largest multiple of 16 <= 256 that
// divides it.
bool tc_gemm_eligible(int dtype, int trans_a, int64_t M, int64_t N, int64_t K, const void* A,
                      const void* C) {
  if (dtype != GF_F32 || trans_a || M <= 0 || N <= 0 || K <= 0) return false;
  if (N % 16 || K % 4) return false;
  if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(C)) & 15u) return false;
  return true;
}

int tc_gemm(int64_t M, int64_t N, int64_t K, const float* A, const float* B, float* C,
            int accumulate, cudaStream_t s) {
  int nt = 16;
  for (int cand = 256; cand >= 16; cand -= 16)
    if (N % cand == 0) {
      nt = cand;
      break;
    }
  const size_t smem = sizeof(float) * (2 * TC_M * TC_KC + 2 * static_cast<size_t>(nt) * TC_KC);
  GF_CHECK_CUDA(cudaFuncSetAttribute(tc_gemm_3xtf32, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
  const int64_t grid = (M + TC_M - 1) / TC_M * (N / nt);
  tc_gemm_3xtf32<<<static_cast<unsigned>(grid), TC_THREADS, smem, s>>>(static_cast<int>(M), static_cast<int>(N),
                                                static_cast<int>(K), nt, A, B, C, accumulate);
  GF_CHECK_LAUNCH("tc_gemm_3xtf32");
  return GF_OK;
}

}  // namespace gfb
