// CUB DeviceRadixSort::SortPairs on sm_100a: which parameters sort correctly?
#include <cub/cub.cuh>
#include <cstdio>
#include <vector>
#include <algorithm>
#include <random>
template <typename V, typename NI>
int check(long long n, int end_bit) {
  std::mt19937_64 rng(1);
  std::vector<unsigned long long> k(n); std::vector<V> v(n);
  for (long long i = 0; i < n; ++i) { k[i] = rng() & ((1ull << 42) - 1); v[i] = (V)i; }
  unsigned long long *dk, *dk2; V *dv, *dv2;
  cudaMalloc(&dk, n*8); cudaMalloc(&dk2, n*8); cudaMalloc(&dv, n*sizeof(V)); cudaMalloc(&dv2, n*sizeof(V));
  cudaMemcpy(dk, k.data(), n*8, cudaMemcpyHostToDevice); cudaMemcpy(dv, v.data(), n*sizeof(V), cudaMemcpyHostToDevice);
  size_t tb = 0; cub::DeviceRadixSort::SortPairs(nullptr, tb, dk, dk2, dv, dv2, (NI)n, 0, end_bit, 0);
  void* t; cudaMalloc(&t, tb);
  cub::DeviceRadixSort::SortPairs(t, tb, dk, dk2, dv, dv2, (NI)n, 0, end_bit, 0);
  cudaDeviceSynchronize();
  std::vector<V> o(n); cudaMemcpy(o.data(), dv2, n*sizeof(V), cudaMemcpyDeviceToHost);
  std::vector<long long> h(n); for (long long i = 0; i < n; ++i) h[i] = i;
  std::stable_sort(h.begin(), h.end(), [&](long long a, long long b) { return k[a] < k[b]; });
  int ok = 1; for (long long i = 0; i < n; ++i) if ((long long)o[i] != h[i]) { ok = 0; break; }
  cudaFree(dk); cudaFree(dk2); cudaFree(dv); cudaFree(dv2); cudaFree(t);
  return ok;
}
int main() {
  for (long long n : {1000LL, 20000LL, 1000000LL}) {
    printf("n=%lld  i64vals/i64n/42:%d  i64vals/int/42:%d  i64vals/i64n/64:%d  i32vals/int/42:%d  i32vals/int/64:%d\n", n,
           check<long long, long long>(n, 42), check<long long, int>(n, 42), check<long long, long long>(n, 64),
           check<int, int>(n, 42), check<int, int>(n, 64));
  }
}
