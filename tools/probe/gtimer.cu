// Probe: %globaltimer resolution on this GPU (distinct increments seen by one thread).
#include <cstdio>
#include <cstdint>
__global__ void k(unsigned long long* out, int n) {
  unsigned long long prev, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(prev));
  int changes = 0;
  unsigned long long mind = ~0ull;
  for (int i = 0; i < n; ++i) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t != prev) { ++changes; if (t - prev < mind) mind = t - prev; prev = t; }
  }
  out[0] = changes; out[1] = mind;
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 16);
  k<<<1, 1>>>(d, 2000000);
  unsigned long long h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("globaltimer changes %llu min increment %llu ns\n", h[0], h[1]);
  return 0;
}
