// standalone check of the plan-build renumbering kernels (morton keys + CUB sort + inversion)
#include "../../paper_2107_03632_b200/csrc/step_kernels.cuh"
#include <cub/cub.cuh>
#include <cstdio>
#include <vector>
#include <algorithm>
int main() {
  const long long N = 20000, Ni = 19000, B = N - Ni;
  std::vector<double> pos(2 * N);
  for (long long i = 0; i < N; ++i) { pos[2*i] = std::sin(0.37 * i) * 0.9; pos[2*i+1] = std::cos(0.91 * i) * 0.9; }
  std::vector<long long> interior(Ni); for (long long k = 0; k < Ni; ++k) interior[k] = B + k;
  double xmin = 1e300, xmax = -1e300, ymin = 1e300, ymax = -1e300;
  for (long long i = 0; i < N; ++i) { xmin = std::min(xmin, pos[2*i]); xmax = std::max(xmax, pos[2*i]); ymin = std::min(ymin, pos[2*i+1]); ymax = std::max(ymax, pos[2*i+1]); }
  const double sx = 2097151.0 / (xmax - xmin), sy = 2097151.0 / (ymax - ymin);
  double* dpos; long long *dint, *dval, *dord; unsigned long long *dkey, *dkey2;
  cudaMalloc(&dpos, 16*N); cudaMalloc(&dint, 8*Ni); cudaMalloc(&dval, 8*Ni); cudaMalloc(&dord, 8*Ni); cudaMalloc(&dkey, 8*Ni); cudaMalloc(&dkey2, 8*Ni);
  cudaMemcpy(dpos, pos.data(), 16*N, cudaMemcpyHostToDevice); cudaMemcpy(dint, interior.data(), 8*Ni, cudaMemcpyHostToDevice);
  rbf::morton_keys_kernel<<<64, 256>>>(dpos, dint, Ni, xmin, ymin, sx, sy, dkey, dval);
  size_t tb = 0; cub::DeviceRadixSort::SortPairs(nullptr, tb, dkey, dkey2, dval, dord, Ni, 0, 42, 0);
  void* t; cudaMalloc(&t, tb);
  cub::DeviceRadixSort::SortPairs(t, tb, dkey, dkey2, dval, dord, Ni, 0, 42, 0);
  std::vector<unsigned long long> key(Ni); cudaMemcpy(key.data(), dkey, 8*Ni, cudaMemcpyDeviceToHost);
  std::vector<long long> ord(Ni); cudaMemcpy(ord.data(), dord, 8*Ni, cudaMemcpyDeviceToHost);
  // host reference
  std::vector<unsigned long long> hk(Ni);
  for (long long k = 0; k < Ni; ++k) {
    long long v = interior[k];
    unsigned long long qx = (unsigned int)((pos[2*v] - xmin) * sx), qy = (unsigned int)((pos[2*v+1] - ymin) * sy);
    auto sp = [](unsigned long long v) { v &= 0x1fffffull; v = (v | (v << 32)) & 0x1f00000000ffffull; v = (v | (v << 16)) & 0x1f0000ff0000ffull; v = (v | (v << 8)) & 0x100f00f00f00f00full; v = (v | (v << 4)) & 0x10c30c30c30c30c3ull; v = (v | (v << 2)) & 0x1249249249249249ull; return v; };
    hk[k] = sp(qx) | (sp(qy) << 1);
  }
  int keys_ok = 1; for (long long k = 0; k < Ni; ++k) if (hk[k] != key[k]) { keys_ok = 0; printf("key %lld %llu vs %llu\n", k, key[k], hk[k]); break; }
  std::vector<long long> ho(Ni); for (long long k = 0; k < Ni; ++k) ho[k] = k;
  std::stable_sort(ho.begin(), ho.end(), [&](long long a, long long b) { return hk[a] < hk[b]; });
  int ord_ok = (ho == ord);
  std::vector<unsigned long long> ks(Ni); cudaMemcpy(ks.data(), dkey2, 8*Ni, cudaMemcpyDeviceToHost);
  int sorted = 1; for (long long i = 1; i < Ni; ++i) if (ks[i-1] > ks[i]) { sorted = 0; break; }
  int consistent = 1; for (long long i = 0; i < Ni; ++i) if (hk[ord[i]] != ks[i]) { consistent = 0; break; }
  long long ties = 0; for (long long i = 1; i < Ni; ++i) if (ks[i-1] == ks[i]) ++ties;
  long long first_diff = -1; for (long long i = 0; i < Ni; ++i) if (ho[i] != ord[i]) { first_diff = i; break; }
  printf("sorted=%d consistent=%d ties=%lld first_diff=%lld\n", sorted, consistent, ties, first_diff);
  // (a) the same keys uploaded from the host
  cudaMemcpy(dkey, hk.data(), 8*Ni, cudaMemcpyHostToDevice);
  cub::DeviceRadixSort::SortPairs(t, tb, dkey, dkey2, dval, dord, Ni, 0, 42, 0);
  cudaMemcpy(ks.data(), dkey2, 8*Ni, cudaMemcpyDeviceToHost);
  sorted = 1; for (long long i = 1; i < Ni; ++i) if (ks[i-1] > ks[i]) { sorted = 0; break; }
  printf("(a) host-uploaded keys: sorted=%d\n", sorted);
  // (b) end_bit 64
  size_t tb2 = 0; cub::DeviceRadixSort::SortPairs(nullptr, tb2, dkey, dkey2, dval, dord, Ni);
  void* t2p; cudaMalloc(&t2p, tb2);
  cub::DeviceRadixSort::SortPairs(t2p, tb2, dkey, dkey2, dval, dord, Ni);
  cudaMemcpy(ks.data(), dkey2, 8*Ni, cudaMemcpyDeviceToHost);
  sorted = 1; for (long long i = 1; i < Ni; ++i) if (ks[i-1] > ks[i]) { sorted = 0; break; }
  printf("(b) full 64 bits: sorted=%d\n", sorted);
  // (c) int num_items
  cub::DeviceRadixSort::SortPairs(t2p, tb2, dkey, dkey2, dval, dord, (int)Ni, 0, 64, 0);
  cudaMemcpy(ks.data(), dkey2, 8*Ni, cudaMemcpyDeviceToHost);
  sorted = 1; for (long long i = 1; i < Ni; ++i) if (ks[i-1] > ks[i]) { sorted = 0; break; }
  printf("(c) int n, 64 bits: sorted=%d  min key %llu max key %llu\n", sorted, *std::min_element(hk.begin(), hk.end()), *std::max_element(hk.begin(), hk.end()));
  printf("keys_ok=%d ord_ok=%d tb=%zu ord[0..3]=%lld %lld %lld host %lld %lld %lld err=%s\n", keys_ok, ord_ok, tb, ord[0], ord[1], ord[2], ho[0], ho[1], ho[2], cudaGetErrorString(cudaGetLastError()));
}
