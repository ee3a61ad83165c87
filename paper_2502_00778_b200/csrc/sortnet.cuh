// sortnet.cuh -- register sorting networks and compile-time loops shared by
// K1 (edge_extract.cu: per-origin entry and item sorts) and the small-segment
// sort (primitives.cu).
#pragma once

#include <utility>

#include "dm_internal.cuh"

namespace dm {

// Batcher's odd-even merge sort on the first N slots of a 2^m network,
// expanded at compile time over registers.  Comparators touching a slot >= N
// are dropped: the padding slots hold kInf and a comparator never moves kInf
// to a lower slot, so they would be no-ops.
struct CmpNet {
  int n;
  unsigned short lo[1200], hi[1200];
};
constexpr CmpNet make_net(int N) {
  CmpNet r{};
  int N2 = 1;
  while (N2 < N) N2 <<= 1;
  for (int p = 1; p < N2; p <<= 1)
    for (int k = p; k >= 1; k >>= 1)
      for (int j = k % p; j + k < N2; j += 2 * k)
        for (int i = 0; i < k; ++i)
          if (i + j + k < N && (i + j) / (2 * p) == (i + j + k) / (2 * p)) {
            r.lo[r.n] = static_cast<unsigned short>(i + j);
            r.hi[r.n] = static_cast<unsigned short>(i + j + k);
            ++r.n;
          }
  return r;
}
template <int N>
struct NetOf {
  static constexpr CmpNet net = make_net(N);
};
template <int N, int I>
__device__ __forceinline__ void cmpx(u32 (&a)[N]) {
  constexpr int lo = NetOf<N>::net.lo[I], hi = NetOf<N>::net.hi[I];
  const u32 x = a[lo], y = a[hi];
  a[lo] = min(x, y);
  a[hi] = max(x, y);
}
template <int N, int... I>
__device__ __forceinline__ void run_net(u32 (&a)[N], std::integer_sequence<int, I...>) {
  (cmpx<N, I>(a), ...);
}
template <int N>
__device__ __forceinline__ void oem_sort(u32 (&a)[N]) {
  static_assert(N <= 128, "network size");
  run_net<N>(a, std::make_integer_sequence<int, NetOf<N>::net.n>{});
}

// Compile-time loop: f(std::integral_constant<int, B>) for B in [B0, B1)
// (nvcc stops fully unrolling large loop nests, which would leave register
// arrays dynamically indexed, i.e. in local memory).
template <int B0, int B1, typename Fn>
__device__ __forceinline__ void static_for(Fn&& f) {
  if constexpr (B0 < B1) {
    f(std::integral_constant<int, B0>{});
    static_for<B0 + 1, B1>(f);
  }
}

}  // namespace dm
