#include <cub/cub.cuh>
#include <cstdio>
#include <vector>
int main() {
  const long long n = 1000;
  std::vector<unsigned long long> k(n); std::vector<long long> v(n);
  for (long long i = 0; i < n; ++i) { k[i] = (i * 7919) % 1000; v[i] = i; }
  unsigned long long *dk, *dk2; long long *dv, *dv2;
  cudaMalloc(&dk, n*8); cudaMalloc(&dk2, n*8); cudaMalloc(&dv, n*8); cudaMalloc(&dv2, n*8);
  cudaMemcpy(dk, k.data(), n*8, cudaMemcpyHostToDevice); cudaMemcpy(dv, v.data(), n*8, cudaMemcpyHostToDevice);
  size_t tb = 0; cub::DeviceRadixSort::SortPairs(nullptr, tb, dk, dk2, dv, dv2, n, 0, 42, 0);
  void* t; cudaMalloc(&t, tb);
  cudaError_t e = cub::DeviceRadixSort::SortPairs(t, tb, dk, dk2, dv, dv2, n, 0, 42, 0);
  std::vector<long long> o(n); cudaMemcpy(o.data(), dv2, n*8, cudaMemcpyDeviceToHost);
  std::vector<unsigned long long> ko(n); cudaMemcpy(ko.data(), dk2, n*8, cudaMemcpyDeviceToHost);
  int ok = 1; for (long long i = 1; i < n; ++i) if (ko[i-1] > ko[i]) ok = 0;
  printf("err=%d tb=%zu sorted=%d first=%lld,%lld keys %llu %llu\n", (int)e, tb, ok, o[0], o[1], ko[0], ko[1]);
  return 0;
}
