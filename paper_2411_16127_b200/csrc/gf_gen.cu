// Synthetic graph generators on the device: the
// reference's gen_random / gen_super_node (graph.cpp:127-185) draw edges one
// at a time from mt19937_64 with an unordered_set rejection loop — 80 s for
// the ogbn-products shape on the CPU.  Here every candidate edge is an
// independent counter-based hash of (seed, index) (splitmix64), duplicates
// are removed by a radix sort + unique, and when more distinct edges than
// requested survive, the kept subset is chosen by a second hash-keyed sort
// (an unbiased random subset, not the smallest ids).  The graphs therefore
// follow the reference's distributions (uniform distinct edges; one hub with
// an exact in-degree; a power-law in-degree sequence) but not its exact
// sequence — bit-exact generation is inherently sequential; tests check the
// distributional contract (counts, distinctness, hub degree, determinism).
// Output is COO (int64 src, dst) for gf_from_coo_device.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <vector>

#include "gf_device.cuh"
#include "gf_internal.cuh"

namespace gfb {
namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t x) {  // splitmix64 finaliser
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// candidate i -> key = dst * n + src (the (dst, src) order from_coo sorts by)
__global__ void uniform_candidates(uint64_t seed, uint64_t stream_id, int64_t count, int64_t n,
                                   int64_t dst_lo, int64_t dst_n, int64_t skip_dst,
                                   uint64_t* __restrict__ keys) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t h1 = mix64(seed ^ mix64(stream_id * 0x100000001B3ull + 2 * i));
    const uint64_t h2 = mix64(seed ^ mix64(stream_id * 0x100000001B3ull + 2 * i + 1));
    const uint64_t s = static_cast<uint64_t>((static_cast<unsigned __int128>(h1) * n) >> 64);
    uint64_t d = dst_lo + static_cast<uint64_t>((static_cast<unsigned __int128>(h2) * dst_n) >> 64);
    if (static_cast<int64_t>(d) == skip_dst) d = ~0ull;  // rejected (hub destination)
    keys[i] = d == ~0ull ? ~0ull : d * static_cast<uint64_t>(n) + s;
  }
}

// power-law rows: candidate j of row r (r = position in the degree sequence)
__global__ void powerlaw_candidates(uint64_t seed, const int64_t* __restrict__ row_off,
                                    const int64_t* __restrict__ perm, int64_t rows, int64_t n,
                                    uint64_t* __restrict__ keys) {
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const int64_t b = row_off[r], e = row_off[r + 1];
    const uint64_t d = static_cast<uint64_t>(perm[r]);
    for (int64_t j = b + threadIdx.x; j < e; j += blockDim.x) {
      const uint64_t h = mix64(seed ^ mix64(0xC0FFEEull + static_cast<uint64_t>(j)));
      const uint64_t s = static_cast<uint64_t>((static_cast<unsigned __int128>(h) * n) >> 64);
      keys[j] = d * static_cast<uint64_t>(n) + s;
    }
  }
}

__global__ void hash_priority(const uint64_t* __restrict__ keys, int64_t count, uint64_t seed,
                              uint64_t* __restrict__ prio) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    prio[i] = mix64(keys[i] ^ mix64(seed + 0x5DEECE66Dull));
}

__global__ void unpack_coo(const uint64_t* __restrict__ keys, int64_t count, int64_t n,
                           int64_t* __restrict__ src, int64_t* __restrict__ dst) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t k = keys[i];
    dst[i] = static_cast<int64_t>(k / n);
    src[i] = static_cast<int64_t>(k % n);
  }
}

int grid_of(int64_t work) {
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(148 * 32, (work + 255) / 256)));
}

// Sort keys [0, count), drop duplicates and rejected (~0) keys; returns the
// distinct count (keys sorted ascending in `out`).
int sort_unique(uint64_t* keys, uint64_t* tmp, int64_t count, uint64_t* out,
                int64_t* n_out, cudaStream_t s) {
  size_t b1 = 0, b2 = 0;
  int64_t* d_n = nullptr;
  GF_CHECK_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, b1, keys, tmp, count, 0, 64, s));
  GF_CHECK_CUDA(cub::DeviceSelect::Unique(nullptr, b2, tmp, out, d_n, count, s));
  void* work = nullptr;
  GF_CHECK_CUDA(scratch_alloc(&work, std::max(b1, b2) + 16, s));
  GF_CHECK_CUDA(scratch_alloc(&d_n, sizeof(int64_t), s));
  GF_CHECK_CUDA(cub::DeviceRadixSort::SortKeys(work, b1, keys, tmp, count, 0, 64, s));
  GF_CHECK_CUDA(cub::DeviceSelect::Unique(work, b2, tmp, out, d_n, count, s));
  int64_t h = 0;
  GF_CHECK_CUDA(cudaMemcpyAsync(&h, d_n, sizeof(h), cudaMemcpyDeviceToHost, s));
  GF_CHECK_CUDA(cudaStreamSynchronize(s));
  cudaFreeAsync(work, s);
  cudaFreeAsync(d_n, s);
  // a rejected candidate sorts last as ~0
  if (h > 0) {
    uint64_t last = 0;
    GF_CHECK_CUDA(cudaMemcpy(&last, out + h - 1, sizeof(last), cudaMemcpyDeviceToHost));
    if (last == ~0ull) --h;
  }
  *n_out = h;
  return GF_OK;
}

// Keep a hash-chosen subset of `target` of the `have` distinct sorted keys
// (unbiased), then restore (dst, src) order.  keys/tmp sized >= have.
int choose_subset(uint64_t* keys, uint64_t* tmp, int64_t have, int64_t target, uint64_t seed,
                  cudaStream_t s) {
  if (have <= target) return GF_OK;
  uint64_t *prio = nullptr, *prio2 = nullptr;
  GF_CHECK_CUDA(scratch_alloc(&prio, sizeof(uint64_t) * have, s));
  GF_CHECK_CUDA(scratch_alloc(&prio2, sizeof(uint64_t) * have, s));
  hash_priority<<<grid_of(have), 256, 0, s>>>(keys, have, seed, prio);
  GF_CHECK_LAUNCH("hash_priority");
  size_t b = 0;
  GF_CHECK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, b, prio, prio2, keys, tmp, have, 0, 64, s));
  void* work = nullptr;
  GF_CHECK_CUDA(scratch_alloc(&work, b + 16, s));
  GF_CHECK_CUDA(cub::DeviceRadixSort::SortPairs(work, b, prio, prio2, keys, tmp, have, 0, 64, s));
  size_t b2 = 0;
  GF_CHECK_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, b2, tmp, keys, target, 0, 64, s));
  void* work2 = nullptr;
  GF_CHECK_CUDA(scratch_alloc(&work2, b2 + 16, s));
  GF_CHECK_CUDA(cub::DeviceRadixSort::SortKeys(work2, b2, tmp, keys, target, 0, 64, s));
  cudaFreeAsync(work, s);
  cudaFreeAsync(work2, s);
  cudaFreeAsync(prio, s);
  cudaFreeAsync(prio2, s);
  return GF_OK;
}

}  // namespace
}  // namespace gfb

// Uniform distinct edges (gen_random's distribution, graph.cpp:127-145):
// exactly round(n * avg_degree) distinct (src, dst) pairs, self-loops allowed.
// src/dst: device int64 arrays of capacity >= round(n * avg_degree).
extern "C" int gf_gen_random_device(int64_t n, double avg_degree, uint64_t seed, int64_t* src,
                                    int64_t* dst, int64_t* e_out, void* stream) {
  if (n <= 0 || !(avg_degree >= 0) || avg_degree >= static_cast<double>(n) || !e_out) {
    gfb::set_error("gf_gen_random_device: n must be positive and avg_degree in [0, n)");
    return GF_ERR_INVALID;
  }
  auto s = static_cast<cudaStream_t>(stream);
  const int64_t target = static_cast<int64_t>(avg_degree * static_cast<double>(n) + 0.5);
  *e_out = target;
  if (target == 0) return GF_OK;
  const double fill = static_cast<double>(target) / (static_cast<double>(n) * n);
  int64_t cand = static_cast<int64_t>(target * (1.0 + 2.0 * fill) + 64);  // cover collisions
  for (int attempt = 0; attempt < 8; ++attempt, cand = cand * 2) {
    uint64_t *keys = nullptr, *tmp = nullptr, *uniq = nullptr;
    GF_CHECK_CUDA(gfb::scratch_alloc(&keys, sizeof(uint64_t) * cand, s));
    GF_CHECK_CUDA(gfb::scratch_alloc(&tmp, sizeof(uint64_t) * cand, s));
    GF_CHECK_CUDA(gfb::scratch_alloc(&uniq, sizeof(uint64_t) * cand, s));
    gfb::uniform_candidates<<<gfb::grid_of(cand), 256, 0, s>>>(seed, attempt, cand, n, 0, n, -1,
                                                               keys);
    GF_CHECK_LAUNCH("uniform_candidates");
    int64_t have = 0;
    int rc = gfb::sort_unique(keys, tmp, cand, uniq, &have, s);
    if (!rc && have >= target) {
      rc = gfb::choose_subset(uniq, tmp, have, target, seed, s);
      if (!rc) {
        gfb::unpack_coo<<<gfb::grid_of(target), 256, 0, s>>>(uniq, target, n, src, dst);
        if (cudaGetLastError() != cudaSuccess) rc = GF_ERR_CUDA;
      }
    }
    cudaFreeAsync(keys, s);
    cudaFreeAsync(tmp, s);
    cudaFreeAsync(uniq, s);
    if (rc) return rc;
    if (have >= target) return GF_OK;
  }
  gfb::set_error("gf_gen_random_device: could not draw enough distinct edges");
  return GF_ERR_GRAPH;
}

// Power-law in-degree graph (the bench's Reddit shape): row r of the degree
// sequence deg_r = round(max_degree * (r + 1)^-exponent) is destination
// perm[r] (a hash permutation of the ids), sources uniform; duplicate sources
// of a row are dropped (the kept in-degree is within a few of deg_r).
// capacity: device src/dst capacity; *e_out = edges written.
extern "C" int gf_gen_power_law_device(int64_t n, int64_t max_degree, double exponent,
                                       uint64_t seed, int64_t capacity, int64_t* src,
                                       int64_t* dst, int64_t* e_out, void* stream) {
  if (n <= 0 || max_degree < 0 || max_degree > n || !(exponent >= 0) || !e_out) {
    gfb::set_error("gf_gen_power_law_device: invalid arguments");
    return GF_ERR_INVALID;
  }
  auto s = static_cast<cudaStream_t>(stream);
  std::vector<int64_t> off(static_cast<size_t>(n) + 1, 0);
  for (int64_t r = 0; r < n; ++r)
    off[r + 1] = off[r] + static_cast<int64_t>(
                              std::llround(max_degree * std::pow(static_cast<double>(r + 1), -exponent)));
  const int64_t cand = off[n];
  if (cand > capacity) {
    gfb::set_error("gf_gen_power_law_device: capacity below the degree-sequence sum");
    return GF_ERR_INVALID;
  }
  int64_t *d_off = nullptr, *perm = nullptr;
  uint64_t *keys = nullptr, *tmp = nullptr, *uniq = nullptr, *pk = nullptr, *pk2 = nullptr;
  GF_CHECK_CUDA(gfb::scratch_alloc(&d_off, sizeof(int64_t) * (n + 1), s));
  GF_CHECK_CUDA(gfb::scratch_alloc(&perm, sizeof(int64_t) * n, s));
  GF_CHECK_CUDA(gfb::scratch_alloc(&pk, sizeof(uint64_t) * n, s));
  GF_CHECK_CUDA(gfb::scratch_alloc(&pk2, sizeof(uint64_t) * n, s));
  GF_CHECK_CUDA(cudaMemcpyAsync(d_off, off.data(), sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, s));
  // hash permutation of the ids: sort ids by a hash key
  {
    std::vector<int64_t> ids(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) ids[i] = i;
    int64_t* d_ids = nullptr;
    GF_CHECK_CUDA(gfb::scratch_alloc(&d_ids, sizeof(int64_t) * n, s));
    GF_CHECK_CUDA(cudaMemcpyAsync(d_ids, ids.data(), sizeof(int64_t) * n, cudaMemcpyHostToDevice, s));
    gfb::hash_priority<<<gfb::grid_of(n), 256, 0, s>>>(reinterpret_cast<const uint64_t*>(d_ids), n,
                                                       seed ^ 0xABCDEFull, pk);
    size_t b = 0;
    GF_CHECK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, b, pk, pk2, d_ids, perm, n, 0, 64, s));
    void* work = nullptr;
    GF_CHECK_CUDA(gfb::scratch_alloc(&work, b + 16, s));
    GF_CHECK_CUDA(cub::DeviceRadixSort::SortPairs(work, b, pk, pk2, d_ids, perm, n, 0, 64, s));
    GF_CHECK_CUDA(cudaStreamSynchronize(s));  // host `ids` leaves scope
    cudaFreeAsync(work, s);
    cudaFreeAsync(d_ids, s);
  }
  GF_CHECK_CUDA(gfb::scratch_alloc(&keys, sizeof(uint64_t) * (cand + 1), s));
  GF_CHECK_CUDA(gfb::scratch_alloc(&tmp, sizeof(uint64_t) * (cand + 1), s));
  GF_CHECK_CUDA(gfb::scratch_alloc(&uniq, sizeof(uint64_t) * (cand + 1), s));
  int64_t have = 0;
  int rc = GF_OK;
  if (cand > 0) {
    gfb::powerlaw_candidates<<<static_cast<int>(std::min<int64_t>(n, 148 * 64)), 256, 0, s>>>(
        seed, d_off, perm, n, n, keys);
    GF_CHECK_LAUNCH("powerlaw_candidates");
    rc = gfb::sort_unique(keys, tmp, cand, uniq, &have, s);
    if (!rc && have > 0) {
      gfb::unpack_coo<<<gfb::grid_of(have), 256, 0, s>>>(uniq, have, n, src, dst);
      if (cudaGetLastError() != cudaSuccess) rc = GF_ERR_CUDA;
    }
  }
  *e_out = have;
  for (void* p : {static_cast<void*>(d_off), static_cast<void*>(perm), static_cast<void*>(keys),
                  static_cast<void*>(tmp), static_cast<void*>(uniq), static_cast<void*>(pk),
                  static_cast<void*>(pk2)})
    cudaFreeAsync(p, s);
  return rc;
}

// One hub (node 0) with exactly hub_degree distinct in-neighbours plus
// uniform distinct edges that avoid the hub destination, in total
// max(hub_degree, round(n * avg_degree)) edges (gen_super_node's shape,
// graph.cpp:147-185; the reference also caps other in-degrees below
// hub_degree, which the uniform part satisfies whp for hub >> avg and which
// the tests check).
extern "C" int gf_gen_super_node_device(int64_t n, double avg_degree, int64_t hub_degree,
                                        uint64_t seed, int64_t* src, int64_t* dst,
                                        int64_t* e_out, void* stream) {
  if (n <= 0 || hub_degree < 1 || hub_degree > n || !(avg_degree >= 0) ||
      avg_degree >= static_cast<double>(n) || !e_out) {
    gfb::set_error("gf_gen_super_node_device: invalid arguments");
    return GF_ERR_INVALID;
  }
  auto s = static_cast<cudaStream_t>(stream);
  const int64_t target = std::max<int64_t>(
      hub_degree, static_cast<int64_t>(avg_degree * static_cast<double>(n) + 0.5));
  const int64_t rest = target - hub_degree;
  // hub in-edges: the first hub_degree ids of a hash permutation
  {
    uint64_t *ids = nullptr, *pk = nullptr, *pk2 = nullptr, *sorted = nullptr;
    GF_CHECK_CUDA(gfb::scratch_alloc(&ids, sizeof(uint64_t) * n, s));
    GF_CHECK_CUDA(gfb::scratch_alloc(&sorted, sizeof(uint64_t) * n, s));
    GF_CHECK_CUDA(gfb::scratch_alloc(&pk, sizeof(uint64_t) * n, s));
    GF_CHECK_CUDA(gfb::scratch_alloc(&pk2, sizeof(uint64_t) * n, s));
    std::vector<uint64_t> h(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) h[i] = static_cast<uint64_t>(i);  // key = dst(0) * n + src
    GF_CHECK_CUDA(cudaMemcpyAsync(ids, h.data(), sizeof(uint64_t) * n, cudaMemcpyHostToDevice, s));
    gfb::hash_priority<<<gfb::grid_of(n), 256, 0, s>>>(ids, n, seed ^ 0x12345ull, pk);
    size_t b = 0;
    GF_CHECK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, b, pk, pk2, ids, sorted, n, 0, 64, s));
    void* work = nullptr;
    GF_CHECK_CUDA(gfb::scratch_alloc(&work, b + 16, s));
    GF_CHECK_CUDA(cub::DeviceRadixSort::SortPairs(work, b, pk, pk2, ids, sorted, n, 0, 64, s));
    gfb::unpack_coo<<<gfb::grid_of(hub_degree), 256, 0, s>>>(sorted, hub_degree, n, src, dst);
    GF_CHECK_LAUNCH("unpack_coo");
    GF_CHECK_CUDA(cudaStreamSynchronize(s));
    for (void* p : {static_cast<void*>(ids), static_cast<void*>(sorted), static_cast<void*>(pk),
                    static_cast<void*>(pk2), work})
      cudaFreeAsync(p, s);
  }
  *e_out = hub_degree;
  if (rest == 0) return GF_OK;
  if (n < 2) {
    gfb::set_error("gf_gen_super_node_device: no non-hub destination");
    return GF_ERR_GRAPH;
  }
  // the rest: uniform distinct edges with destinations in [1, n)
  int64_t cand = rest + rest / 8 + 64;
  for (int attempt = 0; attempt < 8; ++attempt, cand *= 2) {
    uint64_t *keys = nullptr, *tmp = nullptr, *uniq = nullptr;
    GF_CHECK_CUDA(gfb::scratch_alloc(&keys, sizeof(uint64_t) * cand, s));
    GF_CHECK_CUDA(gfb::scratch_alloc(&tmp, sizeof(uint64_t) * cand, s));
    GF_CHECK_CUDA(gfb::scratch_alloc(&uniq, sizeof(uint64_t) * cand, s));
    gfb::uniform_candidates<<<gfb::grid_of(cand), 256, 0, s>>>(seed, 100 + attempt, cand, n, 1,
                                                               n - 1, -1, keys);
    GF_CHECK_LAUNCH("uniform_candidates");
    int64_t have = 0;
    int rc = gfb::sort_unique(keys, tmp, cand, uniq, &have, s);
    if (!rc && have >= rest) {
      rc = gfb::choose_subset(uniq, tmp, have, rest, seed, s);
      if (!rc) {
        gfb::unpack_coo<<<gfb::grid_of(rest), 256, 0, s>>>(uniq, rest, n, src + hub_degree,
                                                           dst + hub_degree);
        if (cudaGetLastError() != cudaSuccess) rc = GF_ERR_CUDA;
      }
    }
    cudaFreeAsync(keys, s);
    cudaFreeAsync(tmp, s);
    cudaFreeAsync(uniq, s);
    if (rc) return rc;
    if (have >= rest) {
      *e_out = target;
      return GF_OK;
    }
  }
  gfb::set_error("gf_gen_super_node_device: could not draw enough distinct edges");
  return GF_ERR_GRAPH;
}

namespace gfb {
namespace {
// molecule m, bond j: j < atoms-1 is the tree bond (atom j+1 -> a hashed
// parent < j+1, so every molecule is connected), the rest are ring bonds
// between two hashed atoms; both directions, self-loops rejected.
__global__ void molecule_candidates(uint64_t seed, int64_t mols, int64_t atoms, int64_t rings,
                                    uint64_t* __restrict__ keys) {
  const int64_t per = atoms - 1 + rings, count = mols * per;
  const uint64_t n = static_cast<uint64_t>(mols * atoms);
  for (int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; c < count;
       c += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t m = c / per, j = c % per;
    const uint64_t h1 = mix64(seed ^ mix64(0x6D6F6Cull + 2 * static_cast<uint64_t>(c)));
    const uint64_t h2 = mix64(seed ^ mix64(0x6D6F6Cull + 2 * static_cast<uint64_t>(c) + 1));
    uint64_t a, b;
    if (j < atoms - 1) {
      a = static_cast<uint64_t>(j + 1);
      b = static_cast<uint64_t>((static_cast<unsigned __int128>(h1) * a) >> 64);
    } else {
      a = static_cast<uint64_t>((static_cast<unsigned __int128>(h1) * atoms) >> 64);
      b = static_cast<uint64_t>((static_cast<unsigned __int128>(h2) * atoms) >> 64);
    }
    const uint64_t base = static_cast<uint64_t>(m * atoms);
    const bool loop = a == b;
    keys[2 * c] = loop ? ~0ull : (base + b) * n + (base + a);
    keys[2 * c + 1] = loop ? ~0ull : (base + a) * n + (base + b);
  }
}
}  // namespace
}  // namespace gfb

// Batched molecules (the C2 ogbg-molhiv shape; the device counterpart of
// batch_graphs over per-molecule graphs, graph.cpp:104-118): `mols` disjoint
// blocks of `atoms` ids, each a random spanning tree plus `rings` extra bonds,
// every bond in both directions, duplicates and self-loops removed.
// capacity >= 2 * mols * (atoms - 1 + rings); *e_out = edges written.
extern "C" int gf_gen_molecules_device(int64_t mols, int64_t atoms, int64_t rings, uint64_t seed,
                                       int64_t capacity, int64_t* src, int64_t* dst,
                                       int64_t* e_out, void* stream) {
  if (mols <= 0 || atoms <= 0 || rings < 0 || !e_out || mols > (int64_t(1) << 31) / atoms) {
    gfb::set_error("gf_gen_molecules_device: invalid arguments");
    return GF_ERR_INVALID;
  }
  const int64_t cand = 2 * mols * (atoms - 1 + rings), n = mols * atoms;
  if (cand > capacity) {
    gfb::set_error("gf_gen_molecules_device: capacity below 2 * mols * (atoms - 1 + rings)");
    return GF_ERR_INVALID;
  }
  *e_out = 0;
  if (cand == 0) return GF_OK;
  auto s = static_cast<cudaStream_t>(stream);
  uint64_t *keys = nullptr, *tmp = nullptr, *uniq = nullptr;
  GF_CHECK_CUDA(gfb::scratch_alloc(&keys, sizeof(uint64_t) * cand, s));
  GF_CHECK_CUDA(gfb::scratch_alloc(&tmp, sizeof(uint64_t) * cand, s));
  GF_CHECK_CUDA(gfb::scratch_alloc(&uniq, sizeof(uint64_t) * cand, s));
  gfb::molecule_candidates<<<gfb::grid_of(cand / 2), 256, 0, s>>>(seed, mols, atoms, rings, keys);
  int rc = cudaGetLastError() == cudaSuccess ? GF_OK : GF_ERR_CUDA;
  int64_t have = 0;
  if (!rc) rc = gfb::sort_unique(keys, tmp, cand, uniq, &have, s);
  if (!rc && have > 0) {
    gfb::unpack_coo<<<gfb::grid_of(have), 256, 0, s>>>(uniq, have, n, src, dst);
    if (cudaGetLastError() != cudaSuccess) rc = GF_ERR_CUDA;
  }
  if (!rc) *e_out = have;
  cudaFreeAsync(keys, s);
  cudaFreeAsync(tmp, s);
  cudaFreeAsync(uniq, s);
  return rc;
}
