// ring_encode.cuh -- the per-edge ring walk encoding shared by the two plans
// of the GATHER path (rings.cu: Morton tiles, rowplan.cu: row tiles).
//
// For an interior edge (j,k) the incident tetrahedra form a closed ring
// {j, k, m_i, m_(i+1)}; for a boundary edge an open chain.  The dual-free
// term of element i is +-cross(m_i - x_k, m_(i+1) - x_k) (the face opposite j
// is {k, m_i, m_(i+1)}; the sign is the parity of (k, m_i, m_(i+1)) against
// the outward vertex order of the reference, mesh.cpp:15,103-110).
#pragma once

#include "dm_internal.cuh"

namespace dm {

// failure bits (also the plan's ring_fail bits)
constexpr int kRingTooLong = 4;     // more than kRingMax incidences
constexpr int kRingNonManifold = 8; // the walk does not consume every incident element
constexpr int kRingMixedSign = 16;  // inconsistently oriented fan
constexpr int kRingWideTile = 64;   // a slot beyond the 8-bit table of a tile over 256 nodes

// parity of the permutation taking (a0,a1,a2) to (b0,b1,b2): +1 even, -1 odd
__device__ __forceinline__ int perm_sign(int a0, int a1, int a2, int b0, int b1, int b2) {
  // rotate (a) so that a0 == b0, then compare the second entries
  const int x1 = a0 == b0 ? a1 : (a1 == b0 ? a2 : a0);
  (void)b2;
  return x1 == b1 ? 1 : -1;
}

struct RingWalk {
  int n = 0;         // incidences
  int start = -1;    // m_0
  int sign = 1;      // common orientation of the terms
  bool closed = false;
  int fail = 0;      // kRing* bits
};

// Walks the ring of edge (j,k) over its incident elements inc[pb .. pb+n)
// (ascending element ids, el = 4 ids per element).  emit(step, node) is
// called for m_0 (step 0) and then m_1 .. m_n (steps 1 .. n); a closed ring
// ends with m_n = m_0.  Deterministic: the start is the smallest node seen
// once (open chain), else the first element's first other node.
template <typename Emit>
__device__ RingWalk ring_walk_encode(int j, int k, int pb, int n, const int32_t* __restrict__ inc,
                                     const int32_t* __restrict__ el, Emit emit) {
  RingWalk r;
  r.n = n;
  if (n > kRingMax) {
    r.fail = kRingTooLong;
    return r;
  }
  int a[kRingMax], b[kRingMax], p0[kRingMax], p1[kRingMax], p2[kRingMax];
  for (int i = 0; i < n; ++i) {
    const int4 v = reinterpret_cast<const int4*>(el)[inc[pb + i]];
    const int vs[4] = {v.x, v.y, v.z, v.w};
    const int ij = vs[0] == j ? 0 : (vs[1] == j ? 1 : (vs[2] == j ? 2 : 3));
    const unsigned f = (kOppPacked >> (6 * ij)) & 63u;  // ref mesh.cpp:15
    p0[i] = vs[f & 3];
    p1[i] = vs[(f >> 2) & 3];
    p2[i] = vs[(f >> 4) & 3];
    int o[2], no = 0;
    for (int q = 0; q < 4; ++q)
      if (vs[q] != j && vs[q] != k && no < 2) o[no++] = vs[q];
    a[i] = o[0];
    b[i] = o[1];
  }
  // The walk from `start`: the next element is the first unused one holding
  // the current node.  Emits m_0 .. m_n; `end` is the last node.
  auto walk = [&](int start, int& end) -> int {
    emit(0, start);
    unsigned used = 0;
    int cur = start, sg0 = 0;
    for (int step = 0; step < n; ++step) {
      int pick = -1;
      for (int i = 0; i < n; ++i)
        if (!(used >> i & 1u) && (a[i] == cur || b[i] == cur)) {
          pick = i;
          break;
        }
      if (pick < 0) return kRingNonManifold;
      used |= 1u << pick;
      const int nxt = a[pick] == cur ? b[pick] : a[pick];
      const int sg = perm_sign(k, cur, nxt, p0[pick], p1[pick], p2[pick]);
      if (step == 0) sg0 = sg;
      else if (sg != sg0) return kRingMixedSign;
      emit(1 + step, nxt);
      cur = nxt;
    }
    r.sign = sg0 < 0 ? -1 : 1;
    end = cur;
    return 0;
  };
  // A closed ring (every node in exactly two elements: the interior edges)
  // starts at a[0].  The XOR of all nodes is 0 then; try that walk first and
  // keep it if it closes -- the same start and codes as the full search
  // below, without its n^2 node counts.
  int x = 0;
  for (int i = 0; i < n; ++i) x ^= a[i] ^ b[i];
  if (x == 0 && n >= 3) {
    int end = -1;
    if (walk(a[0], end) == 0 && end == a[0]) {
      r.start = a[0];
      r.closed = true;
      return r;
    }
  }
  // open chain (or not a fan): the start is the smallest node seen once
  int start = -1;
  for (int i = 0; i < n; ++i)
    for (int s = 0; s < 2; ++s) {
      const int v = s ? b[i] : a[i];
      int cnt = 0;
      for (int q = 0; q < n; ++q) cnt += (a[q] == v) + (b[q] == v);
      if (cnt == 1 && (start < 0 || v < start)) start = v;
    }
  const bool open = start >= 0;
  if (start < 0) start = a[0];
  r.start = start;
  int end = -1;
  r.fail = walk(start, end);
  if (r.fail) return r;
  r.closed = !open && end == start && n >= 3;
  return r;
}

}  // namespace dm
