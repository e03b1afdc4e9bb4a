// nodes.cpp -- the reference's advancing-front unit-disk node generator,
// natively (rbffd.geometry.generate_unit_disk_nodes,
// pkg/src/rbffd/geometry.py:105-198), bit-identical to the Python original.
//
// The algorithm is inherently sequential (ordered acceptance: each accepted
// node changes the test for every later candidate), so it stays on the host:
// a GPU version would have to change the node set.  What the Python original
// pays for is interpretation, not arithmetic -- ~10 min at N=1e7 -- so this
// restatement keeps every floating-point operation in the same order and the
// same libm calls, and replaces only the data structures:
//   * random.Random(seed) -> the same MT19937 stream (init_by_array over the
//     seed's 32-bit words, random() = (a*2^26 + b) / 2^53, CPython
//     Modules/_randommodule.c), one draw per candidate exactly as :172;
//   * the dict hash grid (:144-163) -> a dense padded int32 grid (0 = empty,
//     j+1 = node j) with the same last-writer-wins assignment;
//   * the front deque (:167-181) -> an index sweep: nodes enter the front in
//     acceptance order and leave it in the same order, so popleft() is i++.
// Candidate trigonometry does not depend on acceptance (the angle stream is
// fixed, the ring centre is an already accepted node), so it is computed in
// parallel blocks ahead of the sequential acceptance sweep.
//
// Built with -ffp-contract=off -fno-builtin (no FMA contraction, no sin/cos
// -> sincos fusion) so every expression rounds like CPython's float ops.
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <sys/mman.h>
#include <string>
#include <vector>

#include "../../include/rbffd_b200.h"

namespace rbf_detail {
int fail_c(int code, const char* msg);  // rbffd_b200.cu: sets rbf_last_error()
}

namespace {

// MT19937 as CPython seeds and draws it (_randommodule.c: init_genrand,
// init_by_array, genrand_uint32, random_random).
struct Mt19937 {
  uint32_t s[624];
  int idx = 625;

  void init_genrand(uint32_t seed) {
    s[0] = seed;
    for (int i = 1; i < 624; ++i) s[i] = 1812433253u * (s[i - 1] ^ (s[i - 1] >> 30)) + static_cast<uint32_t>(i);
    idx = 624;
  }
  void init_by_array(const uint32_t* key, int len) {
    init_genrand(19650218u);
    int i = 1, j = 0;
    for (int k = (624 > len ? 624 : len); k; --k) {
      s[i] = (s[i] ^ ((s[i - 1] ^ (s[i - 1] >> 30)) * 1664525u)) + key[j] + static_cast<uint32_t>(j);
      ++i;
      ++j;
      if (i >= 624) {
        s[0] = s[623];
        i = 1;
      }
      if (j >= len) j = 0;
    }
    for (int k = 623; k; --k) {
      s[i] = (s[i] ^ ((s[i - 1] ^ (s[i - 1] >> 30)) * 1566083941u)) - static_cast<uint32_t>(i);
      ++i;
      if (i >= 624) {
        s[0] = s[623];
        i = 1;
      }
    }
    s[0] = 0x80000000u;
  }
  uint32_t next() {
    if (idx >= 624) {
      int k = 0;
      for (; k < 624 - 397; ++k) {
        const uint32_t y = (s[k] & 0x80000000u) | (s[k + 1] & 0x7fffffffu);
        s[k] = s[k + 397] ^ (y >> 1) ^ ((y & 1u) ? 0x9908b0dfu : 0u);
      }
      for (; k < 623; ++k) {
        const uint32_t y = (s[k] & 0x80000000u) | (s[k + 1] & 0x7fffffffu);
        s[k] = s[k + (397 - 624)] ^ (y >> 1) ^ ((y & 1u) ? 0x9908b0dfu : 0u);
      }
      const uint32_t y = (s[623] & 0x80000000u) | (s[0] & 0x7fffffffu);
      s[623] = s[396] ^ (y >> 1) ^ ((y & 1u) ? 0x9908b0dfu : 0u);
      idx = 0;
    }
    uint32_t y = s[idx++];
    y ^= (y >> 11);
    y ^= (y << 7) & 0x9d2c5680u;
    y ^= (y << 15) & 0xefc60000u;
    y ^= (y >> 18);
    return y;
  }
  double random() {
    const uint32_t a = next() >> 5, b = next() >> 6;
    return (a * 67108864.0 + b) * (1.0 / 9007199254740992.0);
  }
};

constexpr double kAcceptFactor = 0.8;     // geometry.py:29
constexpr double kCandidateFactor = 0.95; // geometry.py:30
constexpr int kCandidates = 12;           // geometry.py:31
constexpr int kPad = 2;                   // the 5x5 block reaches 2 cells past the grid
constexpr int64_t kAhead = 6;             // candidates of grid prefetch look-ahead

struct Cell {
  double x, y;
};
constexpr double kEmpty = 8.0;            // >= 7 from any point of the disk: never "too close"
constexpr size_t kHuge = size_t(2) << 20;

}  // namespace

extern "C" int rbf_generate_unit_disk_nodes(double h, const uint32_t* seed_key, int32_t key_len,
                                            double** positions_out, int64_t* n_total,
                                            int64_t* n_boundary) {
  using rbf_detail::fail_c;
  if (!positions_out || !n_total || !n_boundary) return fail_c(RBF_ERR_PARAM, "NULL argument");
  *positions_out = nullptr;
  if (!(0.0 < h && h < 0.5)) return fail_c(RBF_ERR_PARAM, "spacing h outside the valid range (0, 0.5)");
  if (key_len < 1 || !seed_key) return fail_c(RBF_ERR_PARAM, "seed key must have at least one word");

  Mt19937 rng;
  rng.init_by_array(seed_key, key_len);

  // boundary ring, geometry.py:135-141
  const int64_t nb = static_cast<int64_t>(std::floor(2.0 * M_PI / h + 0.5));
  std::vector<double> xy;
  const double est = M_PI / (h * h) + 2.0 * M_PI / h;
  xy.reserve(static_cast<size_t>(2.0 * (est * 1.05 + 64.0)));
  for (int64_t k = 0; k < nb; ++k) {
    const double theta = 2.0 * M_PI * static_cast<double>(k) / static_cast<double>(nb);
    xy.push_back(std::cos(theta));
    xy.push_back(std::sin(theta));
  }

  const double accept = kAcceptFactor * h;
  const double accept2 = accept * accept;
  const double cell = accept / std::sqrt(2.0);
  // cells: int((x + 1) / cell) for x in [-1, 1]; padded by 2 on every side
  const double gmax = 2.0 / cell;
  if (!(gmax < 1.0e6)) return fail_c(RBF_ERR_PARAM, "spacing too small for the dense acceptance grid");
  const int64_t G = static_cast<int64_t>(gmax) + 1 + 2 * kPad;
  // each cell holds the coordinates of the node last assigned to it (the
  // dict's value, dereferenced), empty cells a far-away sentinel: the fits()
  // test is then 25 branch-free distance tests over 5 runs of contiguous
  // cells -- a sentinel is never within `accept`, so the verdict equals the
  // dict walk's.  2 MB-aligned + MADV_HUGEPAGE: the 5 runs lie G cells apart.
  const size_t cells = static_cast<size_t>(G * G);
  const size_t bytes = (cells * sizeof(Cell) + kHuge - 1) / kHuge * kHuge;
  Cell* grid = static_cast<Cell*>(std::aligned_alloc(kHuge, bytes));
  if (!grid) return fail_c(RBF_ERR_PARAM, "out of host memory for the acceptance grid");
  madvise(grid, bytes, MADV_HUGEPAGE);
#pragma omp parallel for schedule(static)
  for (int64_t c = 0; c < static_cast<int64_t>(cells); ++c) grid[c] = Cell{kEmpty, kEmpty};
  auto cell_index = [&](double x, double y) -> int64_t {
    const int64_t cx = static_cast<int64_t>((x + 1.0) / cell) + kPad;
    const int64_t cy = static_cast<int64_t>((y + 1.0) / cell) + kPad;
    return cx * G + cy;
  };
  for (int64_t i = 0; i < nb; ++i) grid[cell_index(xy[2 * i], xy[2 * i + 1])] = Cell{xy[2 * i], xy[2 * i + 1]};

  const double ring = kCandidateFactor * h;
  const double inside2 = std::pow(1.0 - 1e-9, 2.0);
  const double two_pi = 2.0 * M_PI;

  // candidate blocks: front nodes [b0, b1) -> (x, y) of their 12 candidates
  constexpr int64_t kBlock = 16384;
  std::vector<double> ang(static_cast<size_t>(kBlock * kCandidates));
  std::vector<double> cand(static_cast<size_t>(2 * kBlock * kCandidates));
  int64_t i = 0;
  int rc = RBF_OK;
  while (i < static_cast<int64_t>(xy.size() / 2)) {
    const int64_t b0 = i;
    const int64_t avail = static_cast<int64_t>(xy.size() / 2) - b0;
    const int64_t b1 = b0 + (avail < kBlock ? avail : kBlock);
    const int64_t nc = (b1 - b0) * kCandidates;
    for (int64_t c = 0; c < nc; ++c) ang[c] = two_pi * rng.random();  // geometry.py:172
    const double* pxy = xy.data();
#pragma omp parallel for schedule(static) if (nc >= 2048)
    for (int64_t c = 0; c < nc; ++c) {
      const int64_t f = b0 + c / kCandidates;
      const double a = ang[c];
      cand[2 * c] = pxy[2 * f] + ring * std::cos(a);      // :173
      cand[2 * c + 1] = pxy[2 * f + 1] + ring * std::sin(a);  // :174
    }
    for (int64_t c = 0; c < nc; ++c) {
      if (c + kAhead < nc) {  // the grid lines a later candidate will read
        const double px = cand[2 * (c + kAhead)], py = cand[2 * (c + kAhead) + 1];
        if (px > -1.0 && px < 1.0 && py > -1.0 && py < 1.0) {
          const int64_t qx = static_cast<int64_t>((px + 1.0) / cell) + kPad;
          const int64_t qy = static_cast<int64_t>((py + 1.0) / cell) + kPad;
          for (int64_t gx = qx - 2; gx <= qx + 2; ++gx) {
            __builtin_prefetch(grid + gx * G + qy - 2);
            __builtin_prefetch(grid + gx * G + qy + 2);
          }
        }
      }
      const double x = cand[2 * c], y = cand[2 * c + 1];
      if (x * x + y * y >= inside2) continue;  // :175-176
      // fits(x, y), :151-162: any accepted node in the 5x5 block closer than accept
      const int64_t cx = static_cast<int64_t>((x + 1.0) / cell) + kPad;
      const int64_t cy = static_cast<int64_t>((y + 1.0) / cell) + kPad;
      int hit = 0;
      for (int64_t gx = cx - 2; gx <= cx + 2; ++gx) {
        const Cell* col = grid + gx * G + (cy - 2);
        for (int k = 0; k < 5; ++k) {
          const double dx = x - col[k].x;
          const double dy = y - col[k].y;
          hit |= (dx * dx + dy * dy < accept2);
        }
      }
      const bool ok = !hit;
      if (!ok) continue;
      const int64_t j = static_cast<int64_t>(xy.size() / 2);
      if (j >= static_cast<int64_t>(INT32_MAX)) {
        rc = fail_c(RBF_ERR_PARAM, "node count exceeds 2^31-1");
        break;
      }
      xy.push_back(x);
      xy.push_back(y);
      grid[cx * G + cy] = Cell{x, y};
    }
    if (rc != RBF_OK) break;
    i = b1;
  }
  std::free(grid);
  if (rc != RBF_OK) return rc;

  const int64_t N = static_cast<int64_t>(xy.size() / 2);
  if (N - nb < 1 || nb < 3) {  // geometry.py:192-196
    return fail_c(RBF_ERR_PARAM, ("degenerate node set: " + std::to_string(N - nb) + " interior / " +
                                  std::to_string(nb) + " boundary nodes").c_str());
  }
  double* out = static_cast<double*>(std::malloc(sizeof(double) * 2 * static_cast<size_t>(N)));
  if (!out) return fail_c(RBF_ERR_PARAM, "out of host memory for the node set");
  std::memcpy(out, xy.data(), sizeof(double) * 2 * static_cast<size_t>(N));
  *positions_out = out;
  *n_total = N;
  *n_boundary = nb;
  return RBF_OK;
}

extern "C" void rbf_free_host(void* p) { std::free(p); }
