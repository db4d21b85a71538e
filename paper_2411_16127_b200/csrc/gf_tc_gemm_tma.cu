// K0, the dense projection C = A·B (X·W), as a warp-specialised, TMA-fed
// tcgen05 pipeline (3xTF32 for fp32 parity).
//
// The tensor core reads kind::tf32 operands by truncating the fp32 bit
// pattern to tf32 (measured: handing it raw fp32 instead of the masked "hi"
// gives bit-identical results, scripts/tf32_trunc_probe.py).  So the raw A
// tile that TMA lands in shared memory IS the "hi" operand, and only
// lo = x - trunc(x) has to be computed — elementwise, in place of layout, by
// four converter warps.  B (the small weight matrix) is transposed and split
// once per call into K-major [raw | lo] arrays that TMA streams per chunk.
//
//   warp 8 lane 0   TMA producer: A chunk (128 rows x 32 K, 128B-swizzled),
//                   B raw and B lo chunks (NT x 32 K) -> stage s
//   warps 4-7       converters: A_lo = A - trunc(A) into the stage's lo slot
//   warp 9 lane 0   MMA issuer: per chunk 4 k-steps x 3 tcgen05.mma
//                   (Ah Bh + Ah Bl + Al Bh) into a TMEM accumulator
//   warps 0-3       epilogue: tcgen05.ld the accumulator (thread = row) -> C
// Barriers: full[s] (TMA bytes), lo[s] (128 converter arrivals), empty[s]
// (MMA commit), tfull[a] / tempty[a] for the two TMEM accumulators, so the
// epilogue of tile i overlaps the MMAs of tile i+1.  Persistent CTAs, each on
// one n tile, walking the m tiles.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>

#include "gf_internal.cuh"

namespace gfb {
namespace {

constexpr int TM = 128;        // rows per tile (UMMA M)
constexpr int KC = 32;         // K per chunk: 32 fp32 = one 128 B swizzle row
constexpr int NUM_THREADS = 320;

__device__ __forceinline__ uint32_t saddr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// K-major, 128B-swizzled UMMA descriptor: SBO = 1024 B (8 rows x 128 B),
// LBO unused (1), version 1, layout SWIZZLE_128B (2).
__device__ __forceinline__ uint64_t desc_sw128(uint32_t addr) {
  return static_cast<uint64_t>((addr >> 4) & 0x3FFF) | (1ull << 16) |
         (static_cast<uint64_t>(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}

__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(m >> 4) << 24);
}

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(b)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(saddr(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
          "r"(saddr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(saddr(bar))
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   saddr(bar))
               : "memory");
}
__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
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
// TMA tensor store / reduce-add of a [32 cols x 128 rows] box from smem.
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, int c0, int c1, const void* src,
                                             bool add) {
  if (add)
    asm volatile(
        "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2}], [%3];" ::
            "l"(reinterpret_cast<uint64_t>(map)),
        "r"(c0), "r"(c1), "r"(saddr(src))
        : "memory");
  else
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(c0), "r"(c1), "r"(saddr(src))
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void epi_bar() {  // the 4 epilogue warps only
  asm volatile("bar.sync 1, 128;" ::: "memory");
}

__device__ __forceinline__ float lo_of(float x) {
  return x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}

// Extra destinations of the output tile (projection -> all-gather fused):
// the same C rows in other ranks' tables, reached through peer-mapped
// (NVLink / NVSwitch) addresses; the epilogue's TMA stores go to every one.
constexpr int kMaxPeers = 7;
struct PeerMaps {
  CUtensorMap map[kMaxPeers];
  int n;
};

struct Layout {  // byte offsets of one stage inside the dynamic smem
  uint32_t a_raw, a_lo, b_raw, b_lo, bytes;
};
// bres: B is resident for the whole kernel (all chunks, after the stages) and
// a stage carries only the A chunk; otherwise B chunks stream with A.
__host__ __device__ inline Layout stage_layout(int nt, bool bres) {
  Layout l;
  l.a_raw = 0;
  l.a_lo = TM * KC * 4;
  l.b_raw = 2 * TM * KC * 4;
  l.b_lo = l.b_raw + nt * KC * 4;
  const uint32_t b = bres ? l.b_raw : l.b_lo + nt * KC * 4;
  l.bytes = (b + 1023) / 1024 * 1024;  // 1024 B aligned (swizzle atom)
  return l;
}

__global__ void __launch_bounds__(NUM_THREADS, 1)
    tma_gemm_kernel(const __grid_constant__ CUtensorMap map_a,
                    const __grid_constant__ CUtensorMap map_braw,
                    const __grid_constant__ CUtensorMap map_blo,
                    const __grid_constant__ CUtensorMap map_c,
                    const __grid_constant__ PeerMaps peers, int M, int N, int K, int nt,
                    int stages, int bres, int tma_out, float* __restrict__ C, int accumulate,
                    int split_w) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024 B-align the stage area (the swizzle pattern assumes it)
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  __shared__ __align__(8) uint64_t full[4], lor[4], empty[4], tfull[2], tempty[2], bfull;
  __shared__ uint32_t tmem_base;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const Layout L = stage_layout(nt, bres);
  const int n_tiles = N / nt;
  const int m_tiles = (M + TM - 1) / TM;
  const int n_idx = blockIdx.x % n_tiles;
  const int m_first = blockIdx.x / n_tiles, m_step = gridDim.x / n_tiles;
  const int chunks = (K + KC - 1) / KC;
  const uint32_t acc_cols = static_cast<uint32_t>(nt);
  const uint32_t ncols = 2 * nt <= 32 ? 32 : 2 * nt <= 64 ? 64 : 2 * nt <= 128 ? 128 : 256;
  // resident B: chunk c's raw / lo blocks (nt x 128 B each) after the stages;
  // then two 16 KB epilogue staging buffers (128 rows x 32 fp32, 128B-swizzled)
  unsigned char* bres_base = smem + stages * L.bytes;
  const uint32_t bchunk = static_cast<uint32_t>(nt) * KC * 4;
  unsigned char* stage_out = bres_base + (bres ? 2 * bchunk * chunks : 0);

  if (warp == 9) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     saddr(&tmem_base)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&lor[s], 128);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 128);
    }
    mbar_init(&bfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;

  if (warp == 8) {
    // ===== TMA producer =====
    if (lane == 0) {
      if (bres) {  // all of this n tile's B, once
        mbar_expect_tx(&bfull, 2 * bchunk * chunks);
        for (int c = 0; c < chunks; ++c) {
          tma_load_2d(bres_base + c * bchunk, &map_braw, c * KC, n_idx * nt, &bfull);
          tma_load_2d(bres_base + (chunks + c) * bchunk, &map_blo, c * KC, n_idx * nt, &bfull);
        }
      }
      const uint32_t bytes = (TM + (bres ? 0 : 2 * nt)) * KC * 4;
      int it = 0;
      for (int m = m_first; m < m_tiles; m += m_step)
        for (int c = 0; c < chunks; ++c, ++it) {
          const int s = it % stages;
          mbar_wait(&empty[s], ((it / stages) & 1) ^ 1);
          unsigned char* st = smem + s * L.bytes;
          mbar_expect_tx(&full[s], bytes);
          tma_load_2d(st + L.a_raw, &map_a, c * KC, m * TM, &full[s]);
          if (!bres) {
            tma_load_2d(st + L.b_raw, &map_braw, c * KC, n_idx * nt, &full[s]);
            tma_load_2d(st + L.b_lo, &map_blo, c * KC, n_idx * nt, &full[s]);
          }
        }
    }
  } else if (warp >= 4 && warp < 8) {
    // ===== converters: A_lo = A - trunc(A), same (swizzled) byte offsets =====
    const int ct = t - 128;
    int it = 0;
    for (int m = m_first; m < m_tiles; m += m_step)
      for (int c = 0; c < chunks; ++c, ++it) {
        const int s = it % stages;
        mbar_wait(&full[s], (it / stages) & 1);
        unsigned char* st = smem + s * L.bytes;
        const float4* src = reinterpret_cast<const float4*>(st + L.a_raw);
        float4* dst = reinterpret_cast<float4*>(st + L.a_lo);
#pragma unroll
        for (int i = 0; i < TM * KC / 4 / 128; ++i) {
          const float4 x = src[ct + i * 128];
          dst[ct + i * 128] = make_float4(lo_of(x.x), lo_of(x.y), lo_of(x.z), lo_of(x.w));
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive(&lor[s]);
      }
  } else if (warp == 9) {
    // ===== MMA issuer =====
    if (lane == 0) {
      const uint32_t idesc = idesc_tf32(TM, nt);
      if (bres) mbar_wait(&bfull, 0);
      int it = 0, tile = 0;
      for (int m = m_first; m < m_tiles; m += m_step, ++tile) {
        const int a = tile & 1;
        mbar_wait(&tempty[a], ((tile >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tmem + a * acc_cols;
        for (int c = 0; c < chunks; ++c, ++it) {
          const int s = it % stages;
          mbar_wait(&lor[s], (it / stages) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          unsigned char* st = smem + s * L.bytes;
          const uint32_t ah = saddr(st + L.a_raw), al = saddr(st + L.a_lo);
          const uint32_t bh = bres ? saddr(bres_base + c * bchunk) : saddr(st + L.b_raw);
          const uint32_t bl = bres ? saddr(bres_base + (chunks + c) * bchunk) : saddr(st + L.b_lo);
#pragma unroll
          for (int k = 0; k < KC / 8; ++k) {  // 8 tf32 = 32 B per k-step inside the 128 B row
            const uint32_t o = k * 32;
            mma_tf32(d, desc_sw128(ah + o), desc_sw128(bh + o), idesc, (c > 0 || k > 0) ? 1u : 0u);
            mma_tf32(d, desc_sw128(ah + o), desc_sw128(bl + o), idesc, 1u);
            mma_tf32(d, desc_sw128(al + o), desc_sw128(bh + o), idesc, 1u);
          }
          umma_commit(&empty[s]);  // frees the stage when these MMAs complete
        }
        umma_commit(&tfull[a]);  // accumulator a complete
      }
    }
  } else {
    // ===== epilogue (warps 0-3: TMEM lanes 32w..32w+31 = tile rows) =====
    const uint32_t lane_base = static_cast<uint32_t>(warp * 32) << 16;
    int tile = 0, grp = 0;
    for (int m = m_first; m < m_tiles; m += m_step, ++tile) {
      const int a = tile & 1;
      mbar_wait(&tfull[a], (tile >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int row = m * TM + t;
      if (tma_out) {
        // 32-column slices: TMEM -> swizzled smem (conflict-free) -> one TMA
        // store (or reduce-add) per slice, double-buffered through bulk groups
        for (int c0 = 0; c0 < nt; c0 += 32, ++grp) {
          float* buf = reinterpret_cast<float*>(stage_out + (grp & 1) * (TM * 32 * 4));
          if (t == 0) bulk_wait_read<1>();  // the store that used this buffer has read it
          epi_bar();
          uint32_t r[2][16];
          tmem_ld16(tmem + a * acc_cols + lane_base + c0, r[0]);
          tmem_ld16(tmem + a * acc_cols + lane_base + c0 + 16, r[1]);
#pragma unroll
          for (int j = 0; j < 8; ++j) {  // 16 B chunk j of row t at chunk j ^ (t % 8)
            const uint32_t* q = &r[j >> 2][(j & 3) * 4];
            *reinterpret_cast<float4*>(buf + t * 32 + ((j ^ (t & 7)) * 4)) =
                make_float4(__uint_as_float(q[0]), __uint_as_float(q[1]), __uint_as_float(q[2]),
                            __uint_as_float(q[3]));
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          epi_bar();
          if (t == 0) {
            const int col = n_idx * nt + c0;
            if (split_w > 0) {  // column block j of C goes to destination j
              const int j = col / split_w;
              tma_store_2d(j == 0 ? &map_c : &peers.map[j - 1], col - j * split_w, m * TM, buf,
                           accumulate != 0);
            } else {
              tma_store_2d(&map_c, col, m * TM, buf, accumulate != 0);
              for (int p = 0; p < peers.n; ++p)  // same tile into the peers' tables
                tma_store_2d(&peers.map[p], col, m * TM, buf, accumulate != 0);
            }
            bulk_commit();
          }
        }
      } else {
        float* out = C + static_cast<size_t>(row) * N + n_idx * nt;
        for (int c0 = 0; c0 < nt; c0 += 16) {
          uint32_t r[16];
          tmem_ld16(tmem + a * acc_cols + lane_base + c0, r);
          if (row < M) {
#pragma unroll
            for (int j = 0; j < 16; j += 4) {
              float4 o = make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]),
                                     __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3]));
              if (accumulate) {
                const float4 p = *reinterpret_cast<const float4*>(out + c0 + j);
                o.x += p.x, o.y += p.y, o.z += p.z, o.w += p.w;
              }
              *reinterpret_cast<float4*>(out + c0 + j) = o;
            }
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(&tempty[a]);
    }
    if (tma_out && t == 0) bulk_wait_all();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 9)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(ncols));
}

// B (K x N row-major) -> K-major [raw | lo] (N x K): Bt_raw[n][k] = B[k][n],
// Bt_lo[n][k] = B[k][n] - trunc_tf32(B[k][n]).
__global__ void split_b_kernel(const float* __restrict__ B, int K, int N, float* __restrict__ braw,
                               float* __restrict__ blo) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < K * N; i += gridDim.x * blockDim.x) {
    const int k = i / N, n = i % N;
    const float x = B[i];
    braw[static_cast<size_t>(n) * K + k] = x;
    blo[static_cast<size_t>(n) * K + k] = lo_of(x);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// 2-D fp32 tensor [rows x cols] (cols contiguous), box [box_rows x 32 cols],
// 128 B swizzle, out-of-bounds elements read as 0.
bool make_map(CUtensorMap* map, const float* base, int64_t rows, int64_t cols, int box_rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols) * 4};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(KC), static_cast<cuuint32_t>(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int pick_nt(int64_t N) {
  for (int c = 128; c >= 16; c -= 16)
    if (N % c == 0) return c;
  return 0;
}

}  // namespace

bool tma_gemm_eligible(int dtype, int trans_a, int64_t M, int64_t N, int64_t K, const void* A,
                       const void* C) {
  if (dtype != GF_F32 || trans_a || M <= 0 || K <= 0 || K % 4 || !pick_nt(N)) return false;
  if (M >= (1LL << 31) || K >= (1LL << 31)) return false;
  if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(C)) & 15u) return false;
  return encode_fn() != nullptr;
}

int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e && *e ? std::atoi(e) : dflt;
}

int tma_gemm(int64_t M, int64_t N, int64_t K, const float* A, const float* B, float* C,
             int accumulate, cudaStream_t s, float* const* peer_c, int n_peers, int split_w) {
  if (n_peers < 0 || n_peers > kMaxPeers) {
    set_error("gf_gemm_bcast: at most 8 destinations");
    return GF_ERR_INVALID;
  }
  // GF_TMA_NT / GF_TMA_BRES: A/B overrides of the tile width and B residency
  int nt = pick_nt(N);
  const int nt_env = env_int("GF_TMA_NT", 0);
  if (nt_env >= 16 && nt_env <= 128 && nt_env % 16 == 0 && N % nt_env == 0) nt = nt_env;
  if (split_w > 0 && (split_w % 32 || N != static_cast<int64_t>(split_w) * (n_peers + 1) || nt % 32)) {
    set_error("gf_gemm_split: every destination must be a multiple of 32 columns wide");
    return GF_ERR_INVALID;
  }
  float* bsplit = nullptr;
  GF_CHECK_CUDA(scratch_alloc(&bsplit, sizeof(float) * 2 * N * K, s));
  float *braw = bsplit, *blo = bsplit + N * K;
  split_b_kernel<<<static_cast<int>(std::min<int64_t>(1024, (N * K + 255) / 256)), 256, 0, s>>>(
      B, static_cast<int>(K), static_cast<int>(N), braw, blo);
  GF_CHECK_LAUNCH("split_b_kernel");
  CUtensorMap ma, mbr, mbl, mc;
  const bool tma_out = nt % 32 == 0 && N % 4 == 0;  // C rows 16 B aligned for the TMA store
  PeerMaps pm;
  pm.n = n_peers;
  if (n_peers > 0 && !tma_out) {
    cudaFreeAsync(bsplit, s);
    set_error("gf_gemm_bcast: N must be a multiple of 32 (TMA-store epilogue)");
    return GF_ERR_INVALID;
  }
  bool peer_ok = true;
  const int64_t cw = split_w > 0 ? split_w : N;  // columns of each destination
  for (int p = 0; p < n_peers; ++p) peer_ok = peer_ok && make_map(&pm.map[p], peer_c[p], M, cw, TM);
  if (!peer_ok || !make_map(&ma, A, M, K, TM) || !make_map(&mbr, braw, N, K, nt) ||
      !make_map(&mbl, blo, N, K, nt) || (tma_out && !make_map(&mc, C, M, cw, TM))) {
    cudaFreeAsync(bsplit, s);
    set_error("gf_gemm: cuTensorMapEncodeTiled failed");
    return GF_ERR_CUDA;
  }
  const int chunks = static_cast<int>((K + KC - 1) / KC);
  const size_t bres_bytes = 2ull * nt * KC * 4 * chunks;
  const size_t out_bytes = tma_out ? 2 * TM * 32 * 4 : 0;
  // B resident only while >= 3 A stages still fit (A/B on B200: C5 GT QKV
  // 3 streamed stages 1.39 ms vs resident B + 2 stages 1.56 ms)
  const size_t a_stage = stage_layout(nt, true).bytes;
  const bool bres = env_int("GF_TMA_BRES", 1) && bres_bytes <= 128 * 1024 &&
                    224 * 1024 >= bres_bytes + out_bytes + 3 * a_stage;
  const Layout L = stage_layout(nt, bres);
  const size_t budget = 224 * 1024 - (bres ? bres_bytes : 0) - out_bytes;
  const int stages = static_cast<int>(std::max<size_t>(2, std::min<size_t>(4, budget / L.bytes)));
  const size_t smem =
      static_cast<size_t>(stages) * L.bytes + (bres ? bres_bytes : 0) + out_bytes + 1024;
  GF_CHECK_CUDA(cudaFuncSetAttribute(tma_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
  const int n_tiles = static_cast<int>(N / nt);
  const int64_t m_tiles = (M + TM - 1) / TM;
  int grid = static_cast<int>(std::min<int64_t>(m_tiles * n_tiles, 148));
  grid = std::max(n_tiles, grid / n_tiles * n_tiles);
  if (!tma_out) mc = ma;  // unused
  tma_gemm_kernel<<<grid, NUM_THREADS, smem, s>>>(ma, mbr, mbl, mc, pm, static_cast<int>(M),
                                                  static_cast<int>(N), static_cast<int>(K), nt,
                                                  stages, bres ? 1 : 0, tma_out ? 1 : 0, C,
                                                  accumulate, split_w);
  GF_CHECK_LAUNCH("tma_gemm_kernel");
  cudaFreeAsync(bsplit, s);
  return GF_OK;
}

}  // namespace gfb
