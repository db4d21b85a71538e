// Prints the 64-bit L2 policy words createpolicy produces on the device
// (checks the constant in csrc/gf_policy.h).  nvcc -arch=sm_100a policy_words.cu
#include <cstdint>
#include <cstdio>
__global__ void q(uint64_t* o, float f) {
  uint64_t a, b, c, d;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(a));
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(b));
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, %1;" : "=l"(c) : "f"(f));
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(d));
  o[0] = a, o[1] = b, o[2] = c, o[3] = d;
}
int main() {
  uint64_t* d;
  uint64_t h[4];
  cudaMalloc(&d, 32);
  q<<<1, 1>>>(d, 1.0f);
  cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
  printf("evict_last(1.0)=0x%016llx evict_first(1.0)=0x%016llx evict_last(runtime 1.0)=0x%016llx evict_normal(1.0)=0x%016llx\n",
         (unsigned long long)h[0], (unsigned long long)h[1], (unsigned long long)h[2], (unsigned long long)h[3]);
  return 0;
}
