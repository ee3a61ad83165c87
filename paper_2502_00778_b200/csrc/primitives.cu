// primitives.cu -- device scan and segmented sort used by edge extraction
// and by the derived CSR structures.  Hand-written; CUB's radix sort only
// for segments beyond one CTA's shared memory (> 4096 keys: a node with
// more than ~1300 incident tets), one call per such segment.
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "dm_internal.cuh"
#include "sortnet.cuh"

namespace dm {

namespace {

constexpr int kScanThreads = 256;
constexpr int kScanPerThread = 8;
constexpr int kScanBlock = kScanThreads * kScanPerThread;

// Block-local exclusive scan; writes the block total to bsum[blockIdx.x].
// T = u32 (bucket counts) or u64 (K1's packed (items << 32 | entries) counts:
// one scan gives both prefix sums while the low word cannot overflow).
template <typename T>
__global__ void __launch_bounds__(kScanThreads)
    k_scan_blocks(const T* in, T* out, T* bsum, i64 n) {
  __shared__ T wsum[kScanThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const i64 base = static_cast<i64>(blockIdx.x) * kScanBlock + threadIdx.x * kScanPerThread;
  T v[kScanPerThread];
  T tot = 0;
#pragma unroll
  for (int q = 0; q < kScanPerThread; ++q) {
    const i64 i = base + q;
    v[q] = i < n ? in[i] : T(0);
    tot += v[q];
  }
  T incl = tot;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    T w = lane < kScanThreads / 32 ? wsum[lane] : T(0);
    T wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      T t = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += t;
    }
    if (lane < kScanThreads / 32) wsum[lane] = wi - w;  // exclusive warp offsets
    if (lane == kScanThreads / 32 - 1) bsum[blockIdx.x] = wi;
  }
  __syncthreads();
  T run = incl - tot + wsum[warp];
#pragma unroll
  for (int q = 0; q < kScanPerThread; ++q) {
    const i64 i = base + q;
    if (i < n) out[i] = run;
    run += v[q];
  }
}

template <typename T>
__global__ void k_scan_add(T* out, const T* boff, i64 n) {
  const i64 i = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] += boff[i / kScanBlock];
}

template <typename T>
__global__ void k_copy_one(T* dst, const T* src) { *dst = *src; }

template <typename T>
int scan_rec(dm_ctx* c, const T* in, T* out, i64 n, T* tmp) {
  const i64 nb = (n + kScanBlock - 1) / kScanBlock;
  if (n == 0) {
    DM_CK(c, cudaMemsetAsync(out, 0, sizeof(T), c->stream));
    return DM_OK;
  }
  T* lvl = tmp;  // nb + 1 entries
  DM_LAUNCH(c, k_scan_blocks<T>, static_cast<unsigned>(nb), kScanThreads, 0, in, out, lvl, n);
  if (nb > 1) {
    int st = scan_rec<T>(c, lvl, lvl, nb, tmp + nb + 1);
    if (st) return st;
    DM_LAUNCH(c, k_scan_add<T>, grid_for(n, 256), 256, 0, out, lvl, n);
    DM_LAUNCH(c, k_copy_one<T>, 1, 1, 0, out + n, lvl + nb);
  } else {
    DM_LAUNCH(c, k_copy_one<T>, 1, 1, 0, out + n, lvl);
  }
  return DM_OK;
}

i64 scan_tmp_need(i64 n) {
  i64 need = 0, m = n;
  do {
    const i64 nb = (m + kScanBlock - 1) / kScanBlock;
    need += nb + 1;
    m = nb;
  } while (m > 1);
  return need + 4;
}

// ------------------------------------------------------------ segment sort
template <typename K>
__device__ __forceinline__ K key_max();
template <>
__device__ __forceinline__ u64 key_max<u64>() { return ~0ull; }
template <>
__device__ __forceinline__ u32 key_max<u32>() { return ~0u; }

template <typename K, bool kWarp>
__device__ void bitonic(K* buf, int P, int tid, int nthr) {
  for (int k = 2; k <= P; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = tid; i < P; i += nthr) {
        const int ixj = i ^ j;
        if (ixj > i) {
          K a = buf[i], b = buf[ixj];
          const bool up = (i & k) == 0;
          if ((a > b) == up) {
            buf[i] = b;
            buf[ixj] = a;
          }
        }
      }
      if (kWarp) __syncwarp();
      else __syncthreads();
    }
}

constexpr int kWarpSeg = 128;
constexpr int kBlockSeg = 4096;

// Warp per segment of <= kWarpSeg keys: rank sort.  The segment is staged in
// shared memory; each lane holds up to four keys and counts the keys below
// each of them with broadcast reads (one wavefront per read, no bitonic
// exchange traffic: 36 keys cost 36 broadcast loads instead of ~340
// conflict-free exchange wavefronts); ties broken by position unless the
// caller guarantees unique keys.  The sorted run is written back coalesced.
// With `ucnt` (u64 keys only) the warp also counts distinct high words
// (distinct k per origin bucket in K1) -- replacing a separate pass.
template <typename K, bool kUnique, int R>
__device__ __forceinline__ void rank_keys(const K* buf, int n, const K (&key)[4], int lane,
                                          int (&cnt)[4]) {
  for (int i = 0; i < n; i += 2) {  // buf[n] is padded with key_max
    const K v0 = buf[i], v1 = buf[i + 1];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (kUnique) {
        cnt[r] += (v0 < key[r]) + (v1 < key[r]);
      } else {
        const int me = lane + 32 * r;
        cnt[r] += ((v0 < key[r]) | ((v0 == key[r]) & (i < me))) +
                  ((v1 < key[r]) | ((v1 == key[r]) & (i + 1 < me)));
      }
    }
  }
}

template <typename K, bool kUnique>
__global__ void __launch_bounds__(256)
    k_segsort_warp(K* data, const u32* seg, i64 nseg, u32* big, int* nbig, u32* ucnt) {
  __shared__ __align__(16) K sbuf[8][kWarpSeg + 2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const i64 s = static_cast<i64>(blockIdx.x) * 8 + warp;
  if (s >= nseg) return;
  const u32 b = seg[s];
  const int n = static_cast<int>(seg[s + 1] - b);
  if (n <= 1) {
    if (ucnt && lane == 0) ucnt[s] = static_cast<u32>(n);
    return;
  }
  if (n > kWarpSeg) {
    if (lane == 0) big[atomicAdd(nbig, 1)] = static_cast<u32>(s);
    return;
  }
  K* buf = sbuf[warp];
  K key[4];
  int cnt[4] = {0, 0, 0, 0};
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int i = lane + 32 * r;
    key[r] = i < n ? data[b + i] : key_max<K>();
    if (i < kWarpSeg + 2) buf[i] = key[r];
  }
  if (lane < 2) buf[kWarpSeg + lane] = key_max<K>();
  __syncwarp();
  const int nr = (n + 31) >> 5;
  if (nr == 1) rank_keys<K, kUnique, 1>(buf, n, key, lane, cnt);
  else if (nr == 2) rank_keys<K, kUnique, 2>(buf, n, key, lane, cnt);
  else if (nr == 3) rank_keys<K, kUnique, 3>(buf, n, key, lane, cnt);
  else rank_keys<K, kUnique, 4>(buf, n, key, lane, cnt);
  __syncwarp();
#pragma unroll
  for (int r = 0; r < 4; ++r)
    if (lane + 32 * r < n) buf[cnt[r]] = key[r];
  __syncwarp();
  if constexpr (sizeof(K) == 8) {
    if (ucnt) {
      u32 heads = 0;
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int i = lane + 32 * r;
        const bool h = i < n && (i == 0 || (buf[i] >> 32) != (buf[i - 1] >> 32));
        heads += __popc(__ballot_sync(0xffffffffu, h));
      }
      if (lane == 0) ucnt[s] = heads;
    }
  }
  for (int i = lane; i < n; i += 32) data[b + i] = buf[i];
}

// ---- small segments of unique u32 keys (the incoming-edge and node-element
// CSRs: ~7 and ~24 keys per node): a lane sorts a whole segment in
// registers with a sorting network (sortnet.cuh) instead of a warp per
// segment.  A warp takes 32 consecutive segments; their contiguous key range
// is staged in shared memory when it fits.  Longer segments are listed for
// the warp rank sort (<= kWarpSeg keys) or the block sort.
constexpr int kSmallSeg = 32;
constexpr int kSmallStage = 1024;

template <int N>
__device__ __forceinline__ void lane_sort_segment(u32* p, int n) {  // p: shared or global
  u32 a[N];
#pragma unroll
  for (int i = 0; i < N; ++i) a[i] = i < n ? p[i] : 0xffffffffu;
  oem_sort<N>(a);
#pragma unroll
  for (int i = 0; i < N; ++i)
    if (i < n) p[i] = a[i];
}

__global__ void __launch_bounds__(256)
    k_segsort_small_u32(u32* data, const u32* seg, i64 nseg, u32* med, int* nmed, u32* big,
                        int* nbig) {
  constexpr unsigned F = 0xffffffffu;
  __shared__ u32 stage[8][kSmallStage];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const i64 s0 = (static_cast<i64>(blockIdx.x) * 8 + warp) * 32;
  if (s0 >= nseg) return;
  const i64 s = s0 + lane;
  const bool valid = s < nseg;
  const u32 b = valid ? seg[s] : 0u, e = valid ? seg[s + 1] : 0u;
  const int n = static_cast<int>(e - b);
  if (valid && n > kSmallSeg) {
    if (n > kWarpSeg) big[atomicAdd(nbig, 1)] = static_cast<u32>(s);
    else med[atomicAdd(nmed, 1)] = static_cast<u32>(s);
  }
  const int nl = valid && n <= kSmallSeg ? n : 0;
  const int nmax = __reduce_max_sync(F, static_cast<unsigned>(nl));
  if (nmax <= 1) return;
  const int last = 31 - __clz(__ballot_sync(F, valid));
  const u32 b0 = __shfl_sync(F, b, 0), bend = __shfl_sync(F, e, last);
  const bool staged = bend - b0 <= static_cast<u32>(kSmallStage);
  u32* buf = stage[warp];
  if (staged)
    for (u32 i = lane; i < bend - b0; i += 32) buf[i] = data[b0 + i];
  __syncwarp();
  u32* p = staged ? buf + (b - b0) : data + b;
  if (nmax <= 8) lane_sort_segment<8>(p, nl);
  else if (nmax <= 16) lane_sort_segment<16>(p, nl);
  else lane_sort_segment<32>(p, nl);
  __syncwarp();
  if (staged)
    for (u32 i = lane; i < bend - b0; i += 32) data[b0 + i] = buf[i];
}

// Warp rank sort of the listed segments (kSmallSeg < n <= kWarpSeg unique
// u32 keys), grid-stride over the list.
__global__ void __launch_bounds__(256)
    k_segsort_warp_list_u32(u32* data, const u32* seg, const u32* list, const int* nlist) {
  __shared__ __align__(16) u32 sbuf[8][kWarpSeg + 2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int cnt = *nlist;
  for (int q = blockIdx.x * 8 + warp; q < cnt; q += gridDim.x * 8) {
    const u32 s = list[q];
    const u32 b = seg[s];
    const int n = static_cast<int>(seg[s + 1] - b);
    u32* buf = sbuf[warp];
    u32 key[4];
    int rk[4] = {0, 0, 0, 0};
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int i = lane + 32 * r;
      key[r] = i < n ? data[b + i] : 0xffffffffu;
      buf[i] = key[r];
    }
    if (lane < 2) buf[kWarpSeg + lane] = 0xffffffffu;
    __syncwarp();
    const int nr = (n + 31) >> 5;
    if (nr == 2) rank_keys<u32, true, 2>(buf, n, key, lane, rk);
    else if (nr == 3) rank_keys<u32, true, 3>(buf, n, key, lane, rk);
    else rank_keys<u32, true, 4>(buf, n, key, lane, rk);
    __syncwarp();
#pragma unroll
    for (int r = 0; r < 4; ++r)
      if (lane + 32 * r < n) buf[rk[r]] = key[r];
    __syncwarp();
    for (int i = lane; i < n; i += 32) data[b + i] = buf[i];
    __syncwarp();
  }
}

// Unique u64 keys (K1's (k << 32 | e*L + l) items, the boundary-edge keys):
// warp per segment of <= kWarpSeg keys with compressed ranks.  The distinct
// high words are enumerated smallest first (a warp min-reduction per
// distinct value: ~7 rounds for a K1 origin bucket of ~36 items), giving
// every key its group g = rank of its high word among the distinct ones and
// the segment's distinct count (K1's edges per origin) on the way.  When the
// low words span < 2^24 and g < 127, g << 24 | (lo - lo_min) is an
// order-preserving 31-bit key, and a rank costs two integer ops per
// comparison (the sign bit of v - key accumulates "v < key") against four
// for the 64-bit compare-and-select; otherwise the 64-bit rank.  Keys are
// stored straight to their ranks (one segment spans a few sectors).
// Grid-stride over segments: most calls have ~nv short segments.
template <int R>
__device__ __forceinline__ void sort_unique_u64_segment(u64* data, u32 b, int n, int lane,
                                                        const u64 (&pre)[2], u32* b32, u64* b64,
                                                        u32* ucnt) {
  constexpr unsigned F = 0xffffffffu;
  u64 it[R];
  u32 lmin = ~0u, lmax = 0u;
  bool odd = false;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int i = lane + 32 * r;
    it[r] = R <= 2 ? pre[r] : (i < n ? data[b + i] : ~0ull);  // pre: ~0 past n
    if (i < n) {
      const u32 lo = static_cast<u32>(it[r]);
      lmin = min(lmin, lo);
      lmax = max(lmax, lo);
      odd |= (it[r] >> 32) == ~0u;  // a high word of ~0 reads as an empty slot below
    }
  }
  lmin = __reduce_min_sync(F, lmin);
  lmax = __reduce_max_sync(F, lmax);
  int cnt[R];
#pragma unroll
  for (int r = 0; r < R; ++r) cnt[r] = 0;
  u32 d = 0;
  bool ranked = false;
  if (lmax - lmin < (1u << 24) && !__any_sync(F, odd)) {
    u32 g[R], rem[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      g[r] = 0;
      rem[r] = static_cast<u32>(it[r] >> 32);
    }
    for (;;) {
      u32 m = rem[0];
#pragma unroll
      for (int r = 1; r < R; ++r) m = min(m, rem[r]);
      m = __reduce_min_sync(F, m);
      if (m == ~0u) break;
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (rem[r] == m) {
          g[r] = d;
          rem[r] = ~0u;
        }
      ++d;
    }
    if (d < 127) {
      u32 key[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        key[r] = lane + 32 * r < n ? (g[r] << 24 | (static_cast<u32>(it[r]) - lmin)) : 0x7fffffffu;
        b32[lane + 32 * r] = key[r];  // slots >= n hold 0x7fffffff: never below a key
      }
      __syncwarp();
      const uint4* q = reinterpret_cast<const uint4*>(b32);
      for (int i = 0, n4 = (n + 3) >> 2; i < n4; ++i) {
        const uint4 v = q[i];
#pragma unroll
        for (int r = 0; r < R; ++r)
          cnt[r] += static_cast<int>(((v.x - key[r]) >> 31) + ((v.y - key[r]) >> 31) +
                                     ((v.z - key[r]) >> 31) + ((v.w - key[r]) >> 31));
      }
      ranked = true;
    }
  }
  if (!ranked) {  // 64-bit rank; distinct high words counted on the sorted run
#pragma unroll
    for (int r = 0; r < R; ++r) b64[lane + 32 * r] = it[r];
    __syncwarp();
    for (int i = 0; i < n; i += 2) {  // b64[n] is an empty slot (~0) when n is odd
      const u64 v0 = b64[i], v1 = b64[i + 1];
#pragma unroll
      for (int r = 0; r < R; ++r) cnt[r] += (v0 < it[r]) + (v1 < it[r]);
    }
    __syncwarp();
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (lane + 32 * r < n) b64[cnt[r]] = it[r];
    __syncwarp();
    d = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = lane + 32 * r;
      if (i < n) data[b + i] = b64[i];  // coalesced
      const bool h = i < n && (i == 0 || (b64[i] >> 32) != (b64[i - 1] >> 32));
      d += __popc(__ballot_sync(F, h));
    }
  } else {
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (lane + 32 * r < n) data[b + cnt[r]] = it[r];
  }
  if (ucnt && lane == 0) *ucnt = d;
}

// Grid-stride over chunks of 32 consecutive segments per warp: the bounds
// of a chunk are read coalesced, empty and single-key segments are finished
// there (most boundary-edge buckets), and the next segment's (up to 64)
// keys are loaded before the current one is ranked, so the global-load
// latency overlaps the rank arithmetic.
__global__ void __launch_bounds__(256)
    k_segsort_u64u_warp(u64* data, const u32* seg, i64 nseg, u32* big, int* nbig, u32* ucnt) {
  constexpr unsigned F = 0xffffffffu;
  __shared__ __align__(16) u32 s32[8][kWarpSeg];
  __shared__ __align__(16) u64 s64[8][kWarpSeg + 2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const i64 stride = static_cast<i64>(gridDim.x) * 8 * 32;
  for (i64 s0 = (static_cast<i64>(blockIdx.x) * 8 + warp) * 32; s0 < nseg; s0 += stride) {
    const i64 s = s0 + lane;
    u32 sb = 0, sn = 0;
    if (s < nseg) {
      sb = seg[s];
      sn = seg[s + 1] - sb;
      if (ucnt && sn <= 1) ucnt[s] = sn;
      if (sn > static_cast<u32>(kWarpSeg)) big[atomicAdd(nbig, 1)] = static_cast<u32>(s);
    }
    unsigned work = __ballot_sync(F, s < nseg && sn > 1 && sn <= static_cast<u32>(kWarpSeg));
    if (!work) continue;
    auto fetch = [&](int t, u32& b, int& n, u64 (&pre)[2]) {
      b = __shfl_sync(F, sb, t);
      n = static_cast<int>(__shfl_sync(F, sn, t));
      pre[0] = lane < n ? data[b + lane] : ~0ull;
      pre[1] = n <= 64 && lane + 32 < n ? data[b + lane + 32] : ~0ull;
    };
    int t = __ffs(work) - 1;
    work &= work - 1;
    u32 b;
    int n;
    u64 pre[2];
    fetch(t, b, n, pre);
    for (;;) {
      const int tn = work ? __ffs(work) - 1 : -1;
      u32 nb = 0;
      int nn = 0;
      u64 npre[2] = {~0ull, ~0ull};
      if (tn >= 0) {
        work &= work - 1;
        fetch(tn, nb, nn, npre);
      }
      u32* uc = ucnt ? ucnt + s0 + t : nullptr;
      if (n <= 32) {
        sort_unique_u64_segment<1>(data, b, n, lane, pre, s32[warp], s64[warp], uc);
      } else if (n <= 64) {
        sort_unique_u64_segment<2>(data, b, n, lane, pre, s32[warp], s64[warp], uc);
      } else {
        sort_unique_u64_segment<4>(data, b, n, lane, pre, s32[warp], s64[warp], uc);
      }
      __syncwarp();
      if (tn < 0) break;
      t = tn;
      b = nb;
      n = nn;
      pre[0] = npre[0];
      pre[1] = npre[1];
    }
  }
}

template <typename K>
__global__ void __launch_bounds__(512)
    k_segsort_block(K* data, const u32* seg, const u32* big, const int* nbig, int* flag,
                    u32* ucnt) {
  extern __shared__ unsigned char smem_raw[];
  K* buf = reinterpret_cast<K*>(smem_raw);
  const int count = *nbig;
  for (int q = blockIdx.x; q < count; q += gridDim.x) {
    const u32 s = big[q];
    const u32 b = seg[s];
    const int n = static_cast<int>(seg[s + 1] - b);
    if (n > kBlockSeg) {  // left to the host loop of segment_sort
      if (threadIdx.x == 0) atomicExch(flag, 1);
      continue;
    }
    int P = 2;
    while (P < n) P <<= 1;
    for (int i = threadIdx.x; i < P; i += blockDim.x) buf[i] = i < n ? data[b + i] : key_max<K>();
    __syncthreads();
    bitonic<K, false>(buf, P, threadIdx.x, blockDim.x);
    for (int i = threadIdx.x; i < n; i += blockDim.x) data[b + i] = buf[i];
    if constexpr (sizeof(K) == 8) {
      if (ucnt) {
        int heads = 0;
        for (int i0 = 0; i0 < n; i0 += blockDim.x) {
          const int i = i0 + threadIdx.x;
          heads += __syncthreads_count(i < n && (i == 0 || (buf[i] >> 32) != (buf[i - 1] >> 32)));
        }
        if (threadIdx.x == 0) ucnt[s] = static_cast<u32>(heads);
      }
    }
    __syncthreads();
  }
}

// (segment id, start, length) of the queued segments, for the host loop.
__global__ void k_big_lengths(const u32* seg, const u32* big, const int* nbig, uint4* out) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= *nbig) return;
  const u32 s = big[q];
  out[q] = make_uint4(s, seg[s], seg[s + 1] - seg[s], 0u);
}

// Distinct high words of one sorted segment (one CTA).
__global__ void __launch_bounds__(1024) k_count_heads(const u64* data, u32 n, u32* out) {
  int heads = 0;
  for (u32 i0 = 0; i0 < n; i0 += blockDim.x) {
    const u32 i = i0 + threadIdx.x;
    heads += __syncthreads_count(i < n && (i == 0 || (data[i] >> 32) != (data[i - 1] >> 32)));
  }
  if (threadIdx.x == 0) *out = static_cast<u32>(heads);
}

// Segments longer than kBlockSeg: one device radix sort each.
template <typename K>
int sort_huge_segments(dm_ctx* c, K* data, const u32* seg, u32* ucnt) {
  int nb = 0;
  DM_CK(c, cudaMemcpyAsync(&nb, c->flag.p + 1, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  DM_CK(c, cudaStreamSynchronize(c->stream));
  DevBuf<uint4> info;
  DM_CK(c, info.ensure(static_cast<size_t>(nb)));
  DM_LAUNCH(c, k_big_lengths, grid_for(nb, 256), 256, 0, seg, c->seg_big.p, c->flag.p + 1, info.p);
  std::vector<uint4> h(static_cast<size_t>(nb));
  DM_CK(c, cudaMemcpyAsync(h.data(), info.p, sizeof(uint4) * nb, cudaMemcpyDeviceToHost,
                           c->stream));
  DM_CK(c, cudaStreamSynchronize(c->stream));
  DevBuf<K> alt;
  DevBuf<unsigned char> tmp;
  for (const uint4& q : h) {
    if (q.z <= static_cast<u32>(kBlockSeg)) continue;
    DM_CK(c, alt.ensure(q.z));
    size_t tb = 0;
    DM_CK(c, cub::DeviceRadixSort::SortKeys(nullptr, tb, data + q.y, alt.p, static_cast<int>(q.z),
                                            0, static_cast<int>(8 * sizeof(K)), c->stream));
    DM_CK(c, tmp.ensure(tb));
    DM_CK(c, cub::DeviceRadixSort::SortKeys(tmp.p, tb, data + q.y, alt.p, static_cast<int>(q.z),
                                            0, static_cast<int>(8 * sizeof(K)), c->stream));
    DM_CK(c, cudaMemcpyAsync(data + q.y, alt.p, sizeof(K) * q.z, cudaMemcpyDeviceToDevice,
                             c->stream));
    if constexpr (sizeof(K) == 8) {
      if (ucnt) DM_LAUNCH(c, k_count_heads, 1, 1024, 0, data + q.y, q.z, ucnt + q.x);
    }
  }
  DM_CK(c, cudaStreamSynchronize(c->stream));  // scratch dies here
  return DM_OK;
}

template <typename K, bool kUnique>
int segment_sort(dm_ctx* c, K* data, const u32* seg, i64 nseg, u32* ucnt) {
  if (nseg <= 0) return DM_OK;
  DevBuf<u32>& big = c->seg_big;  // persistent scratch (no free/malloc stalls)
  DM_CK(c, big.ensure(static_cast<size_t>(nseg)));
  DM_CK(c, c->flag.ensure(4));
  DM_CK(c, cudaMemsetAsync(c->flag.p, 0, 4 * sizeof(int), c->stream));
  int* nbig = c->flag.p + 1;
  if constexpr (sizeof(K) == 8 && kUnique) {
    const unsigned grid = static_cast<unsigned>(std::min<i64>(grid_for(nseg, 256), 148 * 8));
    DM_LAUNCH(c, k_segsort_u64u_warp, grid, 256, 0, data, seg, nseg, big.p, nbig, ucnt);
  } else if constexpr (sizeof(K) == 4 && kUnique) {
    DevBuf<u32>& med = c->seg_med;
    DM_CK(c, med.ensure(static_cast<size_t>(nseg)));
    int* nmed = c->flag.p + 2;
    DM_LAUNCH(c, k_segsort_small_u32, grid_for(nseg, 256), 256, 0, data, seg, nseg, med.p, nmed,
              big.p, nbig);
    DM_LAUNCH(c, k_segsort_warp_list_u32, 148 * 8, 256, 0, data, seg, med.p, nmed);
  } else {
    DM_LAUNCH(c, (k_segsort_warp<K, kUnique>), grid_for(nseg, 8), 256, 0, data, seg, nseg, big.p,
              nbig, ucnt);
  }
  const size_t smem = kBlockSeg * sizeof(K);
  DM_CK(c, cudaFuncSetAttribute(k_segsort_block<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(smem)));
  DM_LAUNCH(c, k_segsort_block<K>, 296, 512, smem, data, seg, big.p, nbig, c->flag.p, ucnt);
  int f = 0;
  int st = read_flag(c, &f);
  if (st) return st;
  return f ? sort_huge_segments<K>(c, data, seg, ucnt) : DM_OK;
}

// ---- key/value variant: sorts (key, value) pairs lexicographically
template <bool kWarp>
__device__ void bitonic_kv(u64* k, u32* v, int P, int tid, int nthr) {
  for (int kk = 2; kk <= P; kk <<= 1)
    for (int j = kk >> 1; j > 0; j >>= 1) {
      for (int i = tid; i < P; i += nthr) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const u64 a = k[i], b = k[ixj];
          const u32 va = v[i], vb = v[ixj];
          const bool gt = a > b || (a == b && va > vb);
          if (gt == ((i & kk) == 0)) {
            k[i] = b;
            k[ixj] = a;
            v[i] = vb;
            v[ixj] = va;
          }
        }
      }
      if (kWarp) __syncwarp();
      else __syncthreads();
    }
}

__global__ void __launch_bounds__(256)
    k_segsort_kv_warp(u64* keys, u32* vals, const u32* seg, i64 nseg, u32* big, int* nbig) {
  __shared__ u64 sk[8][kWarpSeg];
  __shared__ u32 sv[8][kWarpSeg];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const i64 s = static_cast<i64>(blockIdx.x) * 8 + warp;
  if (s >= nseg) return;
  const u32 b = seg[s];
  const int n = static_cast<int>(seg[s + 1] - b);
  if (n <= 1) return;
  if (n > kWarpSeg) {
    if (lane == 0) big[atomicAdd(nbig, 1)] = static_cast<u32>(s);
    return;
  }
  int P = 2;
  while (P < n) P <<= 1;
  for (int i = lane; i < P; i += 32) {
    sk[warp][i] = i < n ? keys[b + i] : ~0ull;
    sv[warp][i] = i < n ? vals[b + i] : ~0u;
  }
  __syncwarp();
  bitonic_kv<true>(sk[warp], sv[warp], P, lane, 32);
  for (int i = lane; i < n; i += 32) {
    keys[b + i] = sk[warp][i];
    vals[b + i] = sv[warp][i];
  }
}

__global__ void __launch_bounds__(512)
    k_segsort_kv_block(u64* keys, u32* vals, const u32* seg, const u32* big, const int* nbig,
                       int* flag) {
  extern __shared__ unsigned char smem_raw[];
  u64* sk = reinterpret_cast<u64*>(smem_raw);
  u32* sv = reinterpret_cast<u32*>(sk + kBlockSeg);
  const int count = *nbig;
  for (int q = blockIdx.x; q < count; q += gridDim.x) {
    const u32 s = big[q];
    const u32 b = seg[s];
    const int n = static_cast<int>(seg[s + 1] - b);
    if (n > kBlockSeg) {  // left to sort_huge_segments_kv
      if (threadIdx.x == 0) atomicExch(flag, 1);
      continue;
    }
    int P = 2;
    while (P < n) P <<= 1;
    for (int i = threadIdx.x; i < P; i += blockDim.x) {
      sk[i] = i < n ? keys[b + i] : ~0ull;
      sv[i] = i < n ? vals[b + i] : ~0u;
    }
    __syncthreads();
    bitonic_kv<false>(sk, sv, P, threadIdx.x, blockDim.x);
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      keys[b + i] = sk[i];
      vals[b + i] = sv[i];
    }
    __syncthreads();
  }
}

}  // namespace

// (key, value) segments longer than kBlockSeg: two stable radix passes each
// (by value, then by key) give the lexicographic order.
int sort_huge_segments_kv(dm_ctx* c, u64* keys, u32* vals, const u32* seg) {
  int nb = 0;
  DM_CK(c, cudaMemcpyAsync(&nb, c->flag.p + 1, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  DM_CK(c, cudaStreamSynchronize(c->stream));
  DevBuf<uint4> info;
  DM_CK(c, info.ensure(static_cast<size_t>(nb)));
  DM_LAUNCH(c, k_big_lengths, grid_for(nb, 256), 256, 0, seg, c->seg_big.p, c->flag.p + 1, info.p);
  std::vector<uint4> h(static_cast<size_t>(nb));
  DM_CK(c, cudaMemcpyAsync(h.data(), info.p, sizeof(uint4) * nb, cudaMemcpyDeviceToHost,
                           c->stream));
  DM_CK(c, cudaStreamSynchronize(c->stream));
  DevBuf<u64> k2;
  DevBuf<u32> v2;
  DevBuf<unsigned char> tmp;
  for (const uint4& q : h) {
    if (q.z <= static_cast<u32>(kBlockSeg)) continue;
    const int n = static_cast<int>(q.z);
    u64* k = keys + q.y;
    u32* v = vals + q.y;
    DM_CK(c, k2.ensure(q.z));
    DM_CK(c, v2.ensure(q.z));
    size_t t1 = 0, t2 = 0;
    DM_CK(c, cub::DeviceRadixSort::SortPairs(nullptr, t1, v, v2.p, k, k2.p, n, 0, 32, c->stream));
    DM_CK(c, cub::DeviceRadixSort::SortPairs(nullptr, t2, k2.p, k, v2.p, v, n, 0, 64, c->stream));
    DM_CK(c, tmp.ensure(std::max(t1, t2)));
    DM_CK(c, cub::DeviceRadixSort::SortPairs(tmp.p, t1, v, v2.p, k, k2.p, n, 0, 32, c->stream));
    DM_CK(c, cub::DeviceRadixSort::SortPairs(tmp.p, t2, k2.p, k, v2.p, v, n, 0, 64, c->stream));
  }
  DM_CK(c, cudaStreamSynchronize(c->stream));  // scratch dies here
  return DM_OK;
}

int segment_sort_kv(dm_ctx* c, u64* keys, u32* vals, const u32* seg, i64 nseg) {
  if (nseg <= 0) return DM_OK;
  DevBuf<u32>& big = c->seg_big;  // persistent scratch (no free/malloc stalls)
  DM_CK(c, big.ensure(static_cast<size_t>(nseg)));
  DM_CK(c, c->flag.ensure(4));
  DM_CK(c, cudaMemsetAsync(c->flag.p, 0, 4 * sizeof(int), c->stream));
  int* nbig = c->flag.p + 1;
  DM_LAUNCH(c, k_segsort_kv_warp, grid_for(nseg, 8), 256, 0, keys, vals, seg, nseg, big.p, nbig);
  const size_t smem = kBlockSeg * (sizeof(u64) + sizeof(u32));
  DM_CK(c, cudaFuncSetAttribute(k_segsort_kv_block, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(smem)));
  DM_LAUNCH(c, k_segsort_kv_block, 296, 512, smem, keys, vals, seg, big.p, nbig, c->flag.p);
  int f = 0;
  int st = read_flag(c, &f);
  if (st) return st;
  return f ? sort_huge_segments_kv(c, keys, vals, seg) : DM_OK;
}

// ---- global sort of u64 keys (with optional u32 values): buckets on the
// top 16 significant key bits (count, scan, atomic placement), then the
// segmented sort orders each bucket -- (key, value) lexicographically, which
// is a stable sort's order when the values enter in ascending order.  The
// Morton orders of the ring plan (rings.cu) and its boundary lists use it.
namespace {
__global__ void k_umax64(const u64* __restrict__ k, i64 n, unsigned long long* out) {
  unsigned long long m = 0;
  for (i64 i = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<i64>(gridDim.x) * blockDim.x)
    m = max(m, static_cast<unsigned long long>(k[i]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}
__global__ void k_bkt_count(const u64* __restrict__ k, i64 n, int shift, u32* __restrict__ cnt) {
  const i64 i = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) atomicAdd(cnt + (k[i] >> shift), 1u);
}
__global__ void k_bkt_place(const u64* __restrict__ k, const u32* __restrict__ v, i64 n,
                            int shift, const u32* __restrict__ start, u32* __restrict__ fill,
                            u64* __restrict__ ko, u32* __restrict__ vo) {
  const i64 i = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const u64 key = k[i];
  const u64 b = key >> shift;
  const u32 pos = start[b] + atomicAdd(fill + b, 1u);
  ko[pos] = key;
  if (vo) vo[pos] = v[i];
}
}  // namespace

int sort_u64(dm_ctx* c, const u64* keys, const u32* vals, i64 n, u64* keys_out, u32* vals_out) {
  if (n <= 0) return DM_OK;
  DevBuf<unsigned long long> mx;
  DM_CK(c, mx.ensure(1));
  DM_CK(c, cudaMemsetAsync(mx.p, 0, sizeof(unsigned long long), c->stream));
  DM_LAUNCH(c, k_umax64, static_cast<unsigned>(std::min<i64>(grid_for(n, 256), 1184)), 256, 0,
            keys, n, mx.p);
  unsigned long long hmax = 0;
  DM_CK(c, cudaMemcpyAsync(&hmax, mx.p, sizeof(hmax), cudaMemcpyDeviceToHost, c->stream));
  DM_CK(c, cudaStreamSynchronize(c->stream));
  const int bits = hmax ? 64 - __builtin_clzll(hmax) : 1;
  const int shift = bits > 16 ? bits - 16 : 0;
  const i64 nb = static_cast<i64>(hmax >> shift) + 1;
  DevBuf<u32> start, fill;
  DM_CK(c, start.ensure(static_cast<size_t>(nb + 1)));
  DM_CK(c, fill.ensure(static_cast<size_t>(nb + 1)));
  DM_CK(c, cudaMemsetAsync(start.p, 0, (nb + 1) * sizeof(u32), c->stream));
  DM_CK(c, cudaMemsetAsync(fill.p, 0, (nb + 1) * sizeof(u32), c->stream));
  DM_LAUNCH(c, k_bkt_count, grid_for(n, 256), 256, 0, keys, n, shift, start.p);
  int st = scan_exclusive(c, start.p, start.p, nb);
  if (st) return st;
  DM_LAUNCH(c, k_bkt_place, grid_for(n, 256), 256, 0, keys, vals, n, shift, start.p, fill.p,
            keys_out, vals_out);
  st = vals_out ? segment_sort_kv(c, keys_out, vals_out, start.p, nb)
                : segment_sort_unique_u64(c, keys_out, start.p, nb, nullptr);
  if (st) return st;
  DM_CK(c, cudaStreamSynchronize(c->stream));  // the bucket scratch dies here
  return DM_OK;
}

int scan_exclusive(dm_ctx* c, const u32* in, u32* out, i64 n) {
  DM_CK(c, c->scan_tmp.ensure(static_cast<size_t>(scan_tmp_need(n))));
  return scan_rec<u32>(c, in, out, n, c->scan_tmp.p);
}

int scan_exclusive_u64(dm_ctx* c, const u64* in, u64* out, i64 n) {
  DM_CK(c, c->scan_tmp64.ensure(static_cast<size_t>(scan_tmp_need(n))));
  return scan_rec<u64>(c, in, out, n, c->scan_tmp64.p);
}

int segment_sort_u64(dm_ctx* c, u64* data, const u32* seg, i64 nseg) {
  return segment_sort<u64, false>(c, data, seg, nseg, nullptr);
}
int segment_sort_unique_u64(dm_ctx* c, u64* data, const u32* seg, i64 nseg, u32* ucnt) {
  return segment_sort<u64, true>(c, data, seg, nseg, ucnt);
}
int segment_sort_u32(dm_ctx* c, u32* data, const u32* seg, i64 nseg) {
  return segment_sort<u32, true>(c, data, seg, nseg, nullptr);
}

int read_flag(dm_ctx* c, int* value) {
  DM_CK(c, cudaMemcpyAsync(value, c->flag.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  DM_CK(c, cudaStreamSynchronize(c->stream));
  return DM_OK;
}

}  // namespace dm
