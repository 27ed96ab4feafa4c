// lp_sort.cu -- K2: tiling and global sort (rows a4-a7).
//
// The method orders every tile's list by (depth key, primitive id) (readings 8, 10, 11).
// Instead of one 64-bit (tile|depth) radix sort over all E entries we
//   1. sort the N primitives by depth key (stable LSD radix, 4 x 8-bit passes over N, ties by id),
//   2. exclusive-scan tiles_touched in that order,
//   3. emit (tile, id) entries in depth order (warp-cooperative),
//   4. stable LSD radix sort of the entries by tile id only (ceil(log2 T / 8) passes over E),
//   5. per-tile [start, end) ranges.
// The output equals the full (tile|depth, id) sort bit for bit (stable sorts compose), but the
// E-sized work drops from ~6 passes to 1-2.
//
// Radix pass = histogram kernel + per-digit scan kernel + scatter kernel.  The scatter ranks keys
// stably inside a 4096-key block with warp match_any (order = element index), stages the block in
// shared memory in sorted order and writes it out digit-run by digit-run (coalesced).
#include <cuda_runtime.h>
#include <stdint.h>

#include "lp_kernels.h"

namespace lp {

constexpr int RADIX = 256;
constexpr int RADIX_FUSE_BLOCKS = 128;   // up to this many scatter blocks the per-digit scan is fused in
constexpr int WARPS = SORT_THREADS / 32;

// lanes of the warp holding the same 8-bit digit d as this lane (valid lanes only): eight ballots, one
// per digit bit, instead of MATCH.ANY (whose latency grows with the number of distinct values -- up
// to 32 for the random low bytes of depth keys; measured in the k_radix_scatter stall profile)
__device__ __forceinline__ unsigned digit_peers(uint32_t d, bool valid) {
#ifdef LP_SORT_MATCH_ANY
  return __match_any_sync(0xffffffffu, valid ? d : 0x100u + (threadIdx.x & 31));
#else
  unsigned peers = __ballot_sync(0xffffffffu, valid);
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    const unsigned m = __ballot_sync(0xffffffffu, (d >> b) & 1u);
    peers &= ((d >> b) & 1u) ? m : ~m;
  }
  return valid ? peers : (1u << (threadIdx.x & 31));
#endif
}

__device__ __forceinline__ int64_t item_count(const uint32_t *n_dev, int64_t n_host) {
  if (!n_dev) return n_host;
  const int64_t n = (int64_t)*n_dev;
  return n < n_host ? n : n_host;   // n_host is the capacity when n_dev is given
}

// ---------------------------------------------------------------------------------------------
// DROP: keys equal to RADIX_DROP_KEY are not counted (and not written by the scatter)
template <bool DROP>
__global__ void __launch_bounds__(SORT_THREADS) k_radix_hist(const uint32_t *__restrict__ keys, const uint32_t *n_dev,
                                                             int64_t n_host, int shift, uint32_t *__restrict__ hist,
                                                             int nblk) {
  __shared__ uint32_t s_h[WARPS][RADIX];
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int d = tid; d < WARPS * RADIX; d += SORT_THREADS) (&s_h[0][0])[d] = 0;
  __syncthreads();
  const int64_t n = item_count(n_dev, n_host);
  const int64_t start = (int64_t)blockIdx.x * SORT_TILE;
  if (start < n) {
    const int64_t end = start + SORT_TILE < n ? start + SORT_TILE : n;
    for (int64_t e = start + tid; e < end; e += SORT_THREADS) {
      const uint32_t k = keys[e];
      if (!DROP || k != RADIX_DROP_KEY) atomicAdd(&s_h[warp][(k >> shift) & 0xFF], 1u);
    }
  }
  __syncthreads();
  uint32_t s = 0;
#pragma unroll
  for (int w = 0; w < WARPS; ++w) s += s_h[w][tid];
  hist[(size_t)tid * nblk + blockIdx.x] = s;
}

// block-wide exclusive scan of one value per thread (blockDim multiple of 32, <= 1024)
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t *s_warp, uint32_t &total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < nw ? s_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < nw) s_warp[lane] = w;
  }
  __syncthreads();
  const uint32_t wbase = warp ? s_warp[warp - 1] : 0;
  total = s_warp[nw - 1];
  __syncthreads();
  return wbase + x - v;
}

// one block per digit: exclusive scan over the blocks of hist[d][*]; digit total -> tot[d].  256
// threads, each owning SCAN_PER consecutive blocks per round (a 1024-thread block per digit spent its
// time in the 32-warp block scan with most threads idle at these block counts)
constexpr int SCAN_THREADS = 256, SCAN_PER = 4;
__global__ void __launch_bounds__(SCAN_THREADS) k_radix_scan(uint32_t *__restrict__ hist, int nblk,
                                                             uint32_t *__restrict__ tot) {
  __shared__ uint32_t s_warp[32];
  uint32_t *row = hist + (size_t)blockIdx.x * nblk;
  uint32_t carry = 0;
  for (int base = 0; base < nblk; base += SCAN_THREADS * SCAN_PER) {
    const int i0 = base + threadIdx.x * SCAN_PER;
    uint32_t v[SCAN_PER], s = 0;
#pragma unroll
    for (int k = 0; k < SCAN_PER; ++k) {
      v[k] = i0 + k < nblk ? row[i0 + k] : 0u;
      s += v[k];
    }
    uint32_t total;
    uint32_t run = carry + block_exclusive_scan(s, s_warp, total);
#pragma unroll
    for (int k = 0; k < SCAN_PER; ++k) {
      if (i0 + k < nblk) row[i0 + k] = run;
      run += v[k];
    }
    carry += total;
  }
  if (threadIdx.x == 0) tot[blockIdx.x] = carry;
}

// FUSED (few blocks): hist holds the raw per-block digit counts (no k_radix_scan launch); each
// block sums its own prefix and the digit totals from them (<= RADIX_FUSE_BLOCKS loads per digit).
// DROP: keys equal to RADIX_DROP_KEY are dropped (the output holds the kept pairs in order, their
// number -> *kept by block 0)
template <bool FUSED, bool DROP>
__global__ void __launch_bounds__(SORT_THREADS) k_radix_scatter(const uint32_t *__restrict__ keys_in,
                                                                const uint32_t *__restrict__ vals_in,
                                                                uint32_t *__restrict__ keys_out,
                                                                uint32_t *__restrict__ vals_out, const uint32_t *n_dev,
                                                                int64_t n_host, int shift,
                                                                const uint32_t *__restrict__ hist,
                                                                const uint32_t *__restrict__ tot, int nblk,
                                                                uint32_t *__restrict__ kept) {
  __shared__ uint32_t s_keys[SORT_TILE];
  __shared__ uint32_t s_vals[SORT_TILE];
  __shared__ uint32_t s_wcnt[WARPS][RADIX];
  __shared__ uint32_t s_base[RADIX];    // global position of this block's first key of digit d
  __shared__ uint32_t s_local[RADIX];   // start of digit d inside the block's sorted tile
  __shared__ uint32_t s_warp[32];
  const int64_t n = item_count(n_dev, n_host);
  const int64_t start = (int64_t)blockIdx.x * SORT_TILE;
  if (start >= n) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cnt = (int)(n - start < SORT_TILE ? n - start : SORT_TILE);

  for (int d = lane; d < RADIX; d += 32) s_wcnt[warp][d] = 0;
  __syncwarp();
  // ---- stable rank within (warp, digit): element index = start + warp*32*ITEMS + r*32 + lane
  uint32_t key[SORT_ITEMS], val[SORT_ITEMS], rank[SORT_ITEMS];
  unsigned vmask = 0u;   // bit r: key r is kept
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int r = 0; r < SORT_ITEMS; ++r) {
    const int li = warp * 32 * SORT_ITEMS + r * 32 + lane;
    bool valid = li < cnt;
    key[r] = valid ? keys_in[start + li] : 0u;
    val[r] = valid ? vals_in[start + li] : 0u;
    if (DROP) valid = valid && key[r] != RADIX_DROP_KEY;
    vmask |= valid ? 1u << r : 0u;
    const uint32_t d = (key[r] >> shift) & 0xFF;
    const unsigned peers = digit_peers(d, valid);
    const int leader = __ffs(peers) - 1;
    uint32_t b = 0;
    if (valid && lane == leader) {
      b = s_wcnt[warp][d];
      s_wcnt[warp][d] = b + __popc(peers);
    }
    b = __shfl_sync(0xffffffffu, b, leader);
    rank[r] = b + __popc(peers & lt);
    __syncwarp();
  }
  __syncthreads();
  // ---- per digit: exclusive prefix over warps; block digit counts -> local digit starts
  uint32_t bkept;   // keys of this block kept (all valid ones unless DROP)
  {
    const int d = tid;   // SORT_THREADS == RADIX
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) {
      const uint32_t c = s_wcnt[w][d];
      s_wcnt[w][d] = run;
      run += c;
    }
    const uint32_t ex = block_exclusive_scan(run, s_warp, bkept);
    s_local[d] = ex;
    // global start of digit d = (keys of smaller digits, all blocks) + (digit d, earlier blocks)
    uint32_t tsum, pre;
    if (FUSED) {
      tsum = 0;
      pre = 0;
      const uint32_t *row = hist + (size_t)d * nblk;
      for (int b2 = 0; b2 < nblk; ++b2) {
        const uint32_t c = row[b2];
        tsum += c;
        pre += b2 < (int)blockIdx.x ? c : 0u;
      }
    } else {
      tsum = tot[d];
      pre = hist[(size_t)d * nblk + blockIdx.x];
    }
    uint32_t gtotal;
    const uint32_t gex = block_exclusive_scan(tsum, s_warp, gtotal);
    s_base[d] = gex + pre;
    if (DROP && blockIdx.x == 0 && d == 0) *kept = gtotal;
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < SORT_ITEMS; ++r) {
    if ((vmask >> r) & 1u) {
      const uint32_t d = (key[r] >> shift) & 0xFF;
      const uint32_t lp = s_local[d] + s_wcnt[warp][d] + rank[r];
      s_keys[lp] = key[r];
      s_vals[lp] = val[r];
    }
  }
  __syncthreads();
  for (int i = tid; i < (int)bkept; i += SORT_THREADS) {
    const uint32_t k = s_keys[i];
    const uint32_t d = (k >> shift) & 0xFF;
    const uint32_t g = s_base[d] + (uint32_t)i - s_local[d];
    keys_out[g] = k;
    vals_out[g] = s_vals[i];
  }
}

size_t radix_hist_words(int64_t max_items) {
  const int64_t nblk = (max_items + SORT_TILE - 1) / SORT_TILE;
  return (size_t)(nblk > 0 ? nblk : 1) * RADIX + RADIX;
}

template <bool DROP>
static void radix_pass(uint32_t *ki, uint32_t *vi, uint32_t *ko, uint32_t *vo, int64_t n_max, const uint32_t *n_dev,
                       int shift, uint32_t *hist, int nblk, uint32_t *kept, cudaStream_t st, bool hist_ready = false) {
  uint32_t *tot = hist + (size_t)nblk * RADIX;
  if (!hist_ready) k_radix_hist<DROP><<<nblk, SORT_THREADS, 0, st>>>(ki, n_dev, n_max, shift, hist, nblk);
  if (nblk <= RADIX_FUSE_BLOCKS) {   // small sorts: two launches per pass instead of three
    k_radix_scatter<true, DROP><<<nblk, SORT_THREADS, 0, st>>>(ki, vi, ko, vo, n_dev, n_max, shift, hist, tot, nblk,
                                                               kept);
  } else {
    k_radix_scan<<<RADIX, SCAN_THREADS, 0, st>>>(hist, nblk, tot);
    k_radix_scatter<false, DROP><<<nblk, SORT_THREADS, 0, st>>>(ki, vi, ko, vo, n_dev, n_max, shift, hist, tot, nblk,
                                                                kept);
  }
}

int radix_sort_pairs(uint32_t *keys, uint32_t *keys_alt, uint32_t *vals, uint32_t *vals_alt, int64_t n_max,
                     const uint32_t *n_dev, int bits, uint32_t *hist, cudaStream_t st, uint32_t *kept, bool hist0_ready) {
  if (kept && n_max <= 0) cudaMemsetAsync(kept, 0, sizeof(uint32_t), st);
  if (n_max <= 0 || bits <= 0) return 0;
  const int nblk = (int)((n_max + SORT_TILE - 1) / SORT_TILE);
  int flip = 0;
  for (int shift = 0; shift < bits; shift += 8) {
    uint32_t *ki = flip ? keys_alt : keys, *vi = flip ? vals_alt : vals;
    uint32_t *ko = flip ? keys : keys_alt, *vo = flip ? vals : vals_alt;
    if (kept && shift == 0) radix_pass<true>(ki, vi, ko, vo, n_max, n_dev, shift, hist, nblk, kept, st);
    else radix_pass<false>(ki, vi, ko, vo, n_max, kept ? kept : n_dev, shift, hist, nblk, nullptr, st,
                           hist0_ready && shift == 0);
    flip ^= 1;
  }
  return flip;
}

// ---------------------------------------------------------------------------------------------
// exclusive scan of tiles_touched in depth order (a4)
// ---------------------------------------------------------------------------------------------
size_t scan_tmp_words(int64_t max_items) { return (size_t)((max_items + SCAN_TILE - 1) / SCAN_TILE) + 32; }

__global__ void __launch_bounds__(256) k_scan_reduce(const uint32_t *__restrict__ order, const uint32_t *__restrict__ tt,
                                                     int n_host, const uint32_t *n_dev, uint32_t *__restrict__ part) {
  __shared__ uint32_t s_warp[32];
  const int n = (int)item_count(n_dev, n_host);
  const int base = blockIdx.x * SCAN_TILE;
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < SCAN_TILE / 256; ++k) {
    const int j = base + k * 256 + threadIdx.x;
    if (j < n) s += tt[order[j]];
  }
  uint32_t total;
  block_exclusive_scan(s, s_warp, total);
  if (threadIdx.x == 0) part[blockIdx.x] = total;
}

__global__ void __launch_bounds__(1024) k_scan_top(uint32_t *__restrict__ part, int nb, uint32_t *__restrict__ offsets,
                                                   int n_host, const uint32_t *n_dev, uint32_t *__restrict__ counters,
                                                   int64_t capacity) {
  __shared__ uint32_t s_warp[32];
  const int n = (int)item_count(n_dev, n_host);
  uint32_t carry = 0;
  for (int base = 0; base < nb; base += 1024) {
    const int i = base + threadIdx.x;
    const uint32_t v = i < nb ? part[i] : 0;
    uint32_t total;
    const uint32_t ex = block_exclusive_scan(v, s_warp, total);
    if (i < nb) part[i] = carry + ex;
    carry += total;
  }
  if (threadIdx.x == 0) {
    offsets[n] = carry;
    counters[LP_CNT_ENTRIES] = carry;
    counters[LP_CNT_OVERFLOW] = (int64_t)carry > capacity ? 1u : 0u;
  }
}

// prim_emit (deterministic frames, else null): first emitted entry of every primitive
__global__ void __launch_bounds__(256) k_scan_down(const uint32_t *__restrict__ order, const uint32_t *__restrict__ tt,
                                                   int n_host, const uint32_t *n_dev, const uint32_t *__restrict__ part,
                                                   uint32_t *__restrict__ offsets, uint32_t *__restrict__ prim_emit) {
  __shared__ uint32_t s_warp[32];
  const int n = (int)item_count(n_dev, n_host);
  const int base = blockIdx.x * SCAN_TILE;
  if (base >= n) return;
  // thread t owns 8 consecutive elements: base + 8t .. 8t+7
  uint32_t v[SCAN_TILE / 256];
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < SCAN_TILE / 256; ++k) {
    const int j = base + threadIdx.x * (SCAN_TILE / 256) + k;
    v[k] = j < n ? tt[order[j]] : 0;
    s += v[k];
  }
  uint32_t total;
  uint32_t run = part[blockIdx.x] + block_exclusive_scan(s, s_warp, total);
#pragma unroll
  for (int k = 0; k < SCAN_TILE / 256; ++k) {
    const int j = base + threadIdx.x * (SCAN_TILE / 256) + k;
    if (j < n) {
      offsets[j] = run;
      if (prim_emit) prim_emit[order[j]] = run;
    }
    run += v[k];
  }
}

void launch_scan_tiles(const lp_frame &F, int n, const uint32_t *n_dev, cudaStream_t st) {
  const int nb = (n + SCAN_TILE - 1) / SCAN_TILE;
  if (n > 0) k_scan_reduce<<<nb, 256, 0, st>>>(F.prim_order, F.tiles_touched, n, n_dev, F.scan_tmp);
  k_scan_top<<<1, 1024, 0, st>>>(F.scan_tmp, nb, F.offsets, n, n_dev, F.counters, F.capacity);
  if (n > 0)
    k_scan_down<<<nb, 256, 0, st>>>(F.prim_order, F.tiles_touched, n, n_dev, F.scan_tmp, F.offsets, F.prim_emit);
}

// ---------------------------------------------------------------------------------------------
// emission (a5): entries of sorted primitive j at [offsets[j], offsets[j] + tiles_touched)
//
// Load-balanced over OUTPUT entries: a CTA owns EMIT_TILE consecutive entries, finds the
// depth-sorted primitives that produce them (binary search in the scan), stages their offsets,
// ids and rects in shared memory and writes its entries coalesced.  (A thread or warp per
// primitive is badly imbalanced: the nearest primitives -- adjacent in depth order -- are the
// largest and cover thousands of tiles each.)
// ---------------------------------------------------------------------------------------------
constexpr int EMIT_TILE = 2048;

// max j: a[j] <= x for a non-decreasing a with a[0] <= x, by one warp: 32 probes per round narrow
// the interval 32-fold, so ~4 dependent global loads instead of ~20 (the search is the latency
// chain at the head of every k_emit block)
__device__ __forceinline__ int warp_last_leq(const uint32_t *__restrict__ a, int n, uint32_t x) {
  const int lane = threadIdx.x & 31;
  int lo = 0, hi = n - 1;
  while (hi - lo >= 32) {
    const int step = (hi - lo + 31) / 32;
    const int probe = min(lo + (lane + 1) * step, hi);
    const unsigned m = __ballot_sync(0xffffffffu, a[probe] <= x);
    if (m == 0u) {
      hi = lo + step - 1;
    } else {
      const int last = 31 - __clz(m);
      const int nlo = min(lo + (last + 1) * step, hi);
      if (last < 31) hi = min(hi, nlo + step - 1);
      lo = nlo;
    }
  }
  const int probe = lo + lane;
  const unsigned m = __ballot_sync(0xffffffffu, probe <= hi && a[probe] <= x);
  return lo + 31 - __clz(m);
}

__global__ void __launch_bounds__(256) k_emit(const uint32_t *__restrict__ order, const uint32_t *__restrict__ offsets,
                                              const ushort4 *__restrict__ rect, int n_host, const uint32_t *n_dev,
                                              int tiles_x, int64_t capacity,
                                              const uint32_t *__restrict__ E_dev, uint32_t *__restrict__ tile_key,
                                              uint32_t *__restrict__ entry_val, uint32_t *__restrict__ emit_prim,
                                              uint32_t *__restrict__ hist0, int nblk) {
  __shared__ uint32_t s_off[EMIT_TILE];
  __shared__ uint32_t s_id[EMIT_TILE];
  __shared__ ushort4 s_rect[EMIT_TILE];
  __shared__ int s_own[EMIT_TILE];
  __shared__ int s_wmax[8];
  __shared__ int s_j0, s_cnt;
  __shared__ uint32_t s_h0[RADIX];   // hist0: this block's low-byte tile-id histogram
  const int64_t E = item_count(E_dev, capacity);
  const int64_t e0 = (int64_t)blockIdx.x * EMIT_TILE;
  if (hist0) s_h0[threadIdx.x] = 0u;   // blockDim == RADIX
  if (e0 >= E) {
    if (hist0) hist0[(size_t)threadIdx.x * nblk + blockIdx.x] = 0u;
    return;
  }
  const int64_t e1 = e0 + EMIT_TILE < E ? e0 + EMIT_TILE : E;
  const int n = (int)item_count(n_dev, n_host);
  if (threadIdx.x < 64) {   // warp 0 finds the first primitive of the range, warp 1 the last
    const int j = warp_last_leq(offsets, n, (uint32_t)(threadIdx.x < 32 ? e0 : e1 - 1));
    if (threadIdx.x == 0) s_j0 = j;
    if (threadIdx.x == 32) s_cnt = j;
  }
  __syncthreads();
  if (threadIdx.x == 0) s_cnt = s_cnt - s_j0 + 1;   // every primitive in the range owns >= 1 entry: <= EMIT_TILE
  __syncthreads();
  const int j0 = s_j0, cnt = s_cnt;
  const int len = (int)(e1 - e0);
  // owner of every output slot: heads (each primitive's first entry) then a block-wide prefix max
  // (the primitives' offsets increase with their index, so the owner of slot e is the last head <= e)
  for (int k = threadIdx.x; k < EMIT_TILE; k += blockDim.x) s_own[k] = 0;
  __syncthreads();
  for (int q = threadIdx.x; q < cnt; q += blockDim.x) {
    const uint32_t i = order[j0 + q];
    const uint32_t off = offsets[j0 + q];
    s_off[q] = off;
    s_id[q] = i;
    s_rect[q] = rect[i];
    const int64_t pos = (int64_t)off - e0;
    if (pos > 0 && pos < len) atomicMax(&s_own[pos], q);   // slot 0 belongs to q = 0 (its head may precede e0)
  }
  __syncthreads();
  {
    constexpr int PER = EMIT_TILE / 256;   // 8 consecutive slots per thread
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    int v[PER], run = 0;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      run = max(run, s_own[t * PER + k]);
      v[k] = run;
    }
    int incl = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl = max(incl, y);
    }
    if (lane == 31) s_wmax[w] = incl;
    int excl = __shfl_up_sync(0xffffffffu, incl, 1);
    if (lane == 0) excl = 0;
    __syncthreads();
    int wpre = 0;
    for (int k = 0; k < w; ++k) wpre = max(wpre, s_wmax[k]);
    const int pre = max(excl, wpre);
#pragma unroll
    for (int k = 0; k < PER; ++k) s_own[t * PER + k] = max(v[k], pre);
  }
  __syncthreads();
  for (int64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
    const int lo = s_own[e - e0];
    const uint32_t k = (uint32_t)e - s_off[lo];
    const ushort4 r = s_rect[lo];
    const uint32_t rw = (uint32_t)r.z - r.x + 1;
    const uint32_t ty = r.y + k / rw, tx = r.x + k % rw;
    LP_CHECK(tx <= r.z && ty <= r.w && (int64_t)e < capacity);
    const uint32_t tk = ty * (uint32_t)tiles_x + tx;
    tile_key[e] = tk;
    if (hist0) atomicAdd(&s_h0[tk & 0xFFu], 1u);
    if (emit_prim) {            // deterministic frames: the sort carries the emission index
      entry_val[e] = (uint32_t)e;
      emit_prim[e] = s_id[lo];
    } else {
      entry_val[e] = s_id[lo];
    }
  }
  if (hist0) {   // the first tile-sort pass's histogram column of this block (k_radix_hist not launched)
    __syncthreads();
    hist0[(size_t)threadIdx.x * nblk + blockIdx.x] = s_h0[threadIdx.x];
  }
}

// deterministic frames, after the stable tile sort: emit_pos[k] = sorted position of emitted entry k,
// and the sorted values back to primitive ids (the raster kernels see the usual list)
__global__ void __launch_bounds__(256) k_det_fixup(uint32_t *__restrict__ sorted_val, const uint32_t *__restrict__ emit_prim,
                                                   uint32_t *__restrict__ emit_pos, const uint32_t *E_dev, int64_t capacity) {
  const int64_t E = item_count(E_dev, capacity);
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t k = sorted_val[e];
    LP_CHECK((int64_t)k < capacity);
    emit_pos[k] = (uint32_t)e;
    sorted_val[e] = emit_prim[k];
  }
}

void launch_det_fixup(const lp_frame &F, uint32_t *sorted_val, cudaStream_t st) {
  if (F.capacity <= 0) return;
  k_det_fixup<<<148 * 8, 256, 0, st>>>(sorted_val, F.emit_prim, F.emit_pos, F.counters + LP_CNT_ENTRIES, F.capacity);
}

bool launch_emit(const lp_frame &F, int n, const uint32_t *n_dev, int64_t max_entries, bool hist0, cudaStream_t st) {
  static_assert(EMIT_TILE == SORT_TILE && RADIX == 256, "an emission block is a radix block");
  if (n == 0 || max_entries <= 0) return false;
  const int64_t grid = (max_entries + EMIT_TILE - 1) / EMIT_TILE;
  k_emit<<<(unsigned)grid, 256, 0, st>>>(F.prim_order, F.offsets, reinterpret_cast<const ushort4 *>(F.rect), n, n_dev,
                                         F.tiles_x, F.capacity, F.counters + LP_CNT_ENTRIES, F.tile_key, F.entry_val,
                                         F.deterministic ? F.emit_prim : nullptr, hist0 ? F.sort_hist : nullptr,
                                         (int)grid);
  return hist0;
}

// ---------------------------------------------------------------------------------------------
// per-tile ranges (a7)
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_ranges(const uint32_t *__restrict__ tile, const uint32_t *n_dev,
                                                int64_t capacity, uint32_t *__restrict__ ranges) {
  const int64_t E = item_count(n_dev, capacity);
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  const uint32_t t = tile[e];
  LP_CHECK(e == 0 || tile[e - 1] <= t);
  if (e == 0 || tile[e - 1] != t) ranges[2 * (size_t)t] = (uint32_t)e;
  if (e == E - 1 || tile[e + 1] != t) ranges[2 * (size_t)t + 1] = (uint32_t)(e + 1);
}

void launch_ranges(const lp_frame &F, const uint32_t *sorted_tile, int tiles, cudaStream_t st) {
  cudaMemsetAsync(F.ranges, 0, sizeof(uint32_t) * 2 * (size_t)tiles, st);
  if (F.capacity <= 0) return;
  const int64_t grid = (F.capacity + 255) / 256;
  k_ranges<<<(unsigned)grid, 256, 0, st>>>(sorted_tile, F.counters + LP_CNT_ENTRIES, F.capacity, F.ranges);
}

// ---------------------------------------------------------------------------------------------
// Small problems (C1-sized frames): launch latency, not bandwidth, bounds the ~23-launch pipeline
// above, so one 1024-thread CTA does the depth sort + scan in shared memory (k_small_depth_scan)
// and another the tile sort + ranges (k_small_tile_sort): lp_bin_sort becomes 3 launches (with
// k_emit).  Same stable LSD passes as the multi-block path (match_any ranks in element order),
// hence the same order bit for bit.
// ---------------------------------------------------------------------------------------------
constexpr int SMALL_THREADS = 1024, SMALL_WARPS = SMALL_THREADS / 32;

// one stable 8-bit LSD pass of (key, val) over n <= 32 * 32 * ITEMS elements in shared memory
template <int ITEMS>
__device__ void small_radix_pass(const uint32_t *ki, const uint32_t *vi, uint32_t *ko, uint32_t *vo, int n, int shift,
                                 uint32_t (*s_wcnt)[RADIX], uint32_t *s_local, uint32_t *s_tmp) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int d = lane; d < RADIX; d += 32) s_wcnt[warp][d] = 0;
  __syncwarp();
  uint32_t key[ITEMS], val[ITEMS], rank[ITEMS];
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int r = 0; r < ITEMS; ++r) {
    const int li = warp * 32 * ITEMS + r * 32 + lane;
    const bool valid = li < n;
    key[r] = valid ? ki[li] : 0u;
    val[r] = valid ? vi[li] : 0u;
    const uint32_t d = (key[r] >> shift) & 0xFF;
    const unsigned peers = digit_peers(d, valid);
    const int leader = __ffs(peers) - 1;
    uint32_t b = 0;
    if (valid && lane == leader) {
      b = s_wcnt[warp][d];
      s_wcnt[warp][d] = b + __popc(peers);
    }
    b = __shfl_sync(0xffffffffu, b, leader);
    rank[r] = b + __popc(peers & lt);
    __syncwarp();
  }
  __syncthreads();
  // per digit (threads 0..255): exclusive prefix over the warps, then over the digits
  uint32_t run = 0;
  if (tid < RADIX) {
#pragma unroll 4
    for (int w = 0; w < SMALL_WARPS; ++w) {
      const uint32_t c = s_wcnt[w][tid];
      s_wcnt[w][tid] = run;
      run += c;
    }
    uint32_t x = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_tmp[warp] = x;
    s_local[tid] = x - run;   // exclusive within the warp
  }
  __syncthreads();
  if (tid < RADIX) {
    uint32_t base = 0;
    for (int w = 0; w < warp; ++w) base += s_tmp[w];
    s_local[tid] += base;
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < ITEMS; ++r) {
    const int li = warp * 32 * ITEMS + r * 32 + lane;
    if (li < n) {
      const uint32_t d = (key[r] >> shift) & 0xFF;
      const uint32_t pos = s_local[d] + s_wcnt[warp][d] + rank[r];
      ko[pos] = key[r];
      vo[pos] = val[r];
    }
  }
  __syncthreads();
}

constexpr int SMALL_DEPTH_ITEMS = 4;                                   // n <= 4096 primitives
constexpr int SMALL_TILE_ITEMS = 8;                                    // E <= 8192 entries
constexpr int SMALL_N = SMALL_THREADS * SMALL_DEPTH_ITEMS;
constexpr int SMALL_E = SMALL_THREADS * SMALL_TILE_ITEMS;

// depth sort of the n primitives (keys prim_key: invisible ones 0xFFFFFFFF sort last) + exclusive
// scan of tiles_touched in that order -> prim_order, offsets[0..n], E, overflow (and prim_emit)
__global__ void __launch_bounds__(SMALL_THREADS) k_small_depth_scan(lp_frame F, int n) {
  extern __shared__ __align__(16) uint32_t s_dyn[];
  uint32_t *kA = s_dyn, *vA = kA + SMALL_N, *kB = vA + SMALL_N, *vB = kB + SMALL_N;
  __shared__ uint32_t s_wcnt[SMALL_WARPS][RADIX];
  __shared__ uint32_t s_local[RADIX], s_tmp[SMALL_WARPS];
  const int tid = threadIdx.x;
  for (int i = tid; i < n; i += SMALL_THREADS) {
    kA[i] = F.prim_key[i];
    vA[i] = (uint32_t)i;
  }
  __syncthreads();
  small_radix_pass<SMALL_DEPTH_ITEMS>(kA, vA, kB, vB, n, 0, s_wcnt, s_local, s_tmp);
  small_radix_pass<SMALL_DEPTH_ITEMS>(kB, vB, kA, vA, n, 8, s_wcnt, s_local, s_tmp);
  small_radix_pass<SMALL_DEPTH_ITEMS>(kA, vA, kB, vB, n, 16, s_wcnt, s_local, s_tmp);
  small_radix_pass<SMALL_DEPTH_ITEMS>(kB, vB, kA, vA, n, 24, s_wcnt, s_local, s_tmp);
  // exclusive scan of tiles_touched in depth order: thread t owns elements 4t .. 4t+3
  uint32_t v[SMALL_DEPTH_ITEMS], sum = 0;
#pragma unroll
  for (int k = 0; k < SMALL_DEPTH_ITEMS; ++k) {
    const int j = tid * SMALL_DEPTH_ITEMS + k;
    v[k] = j < n ? F.tiles_touched[vA[j]] : 0u;
    sum += v[k];
  }
  uint32_t total;
  uint32_t run = block_exclusive_scan(sum, s_tmp, total);
#pragma unroll
  for (int k = 0; k < SMALL_DEPTH_ITEMS; ++k) {
    const int j = tid * SMALL_DEPTH_ITEMS + k;
    if (j < n) {
      F.prim_order[j] = vA[j];
      F.prim_key[j] = kA[j];
      F.offsets[j] = run;
      if (F.prim_emit) F.prim_emit[vA[j]] = run;
    }
    run += v[k];
  }
  if (tid == 0) {
    F.offsets[n] = total;
    F.counters[LP_CNT_ENTRIES] = total;
    F.counters[LP_CNT_OVERFLOW] = (int64_t)total > F.capacity ? 1u : 0u;
  }
}

// stable sort of the E <= capacity <= 8192 emitted (tile, value) pairs by tile (in place in
// tile_key / entry_val) and the per-tile ranges
__global__ void __launch_bounds__(SMALL_THREADS) k_small_tile_sort(lp_frame F, int bits, int tiles) {
  extern __shared__ __align__(16) uint32_t s_dyn[];
  uint32_t *kA = s_dyn, *vA = kA + SMALL_E, *kB = vA + SMALL_E, *vB = kB + SMALL_E;
  __shared__ uint32_t s_wcnt[SMALL_WARPS][RADIX];
  __shared__ uint32_t s_local[RADIX], s_tmp[SMALL_WARPS];
  const int tid = threadIdx.x;
  const int E = (int)min((int64_t)F.counters[LP_CNT_ENTRIES], F.capacity);
  for (int i = tid; i < E; i += SMALL_THREADS) {
    kA[i] = F.tile_key[i];
    vA[i] = F.entry_val[i];
  }
  for (int t = tid; t < 2 * tiles; t += SMALL_THREADS) F.ranges[t] = 0u;
  __syncthreads();
  uint32_t *ki = kA, *vi = vA, *ko = kB, *vo = vB;
  for (int shift = 0; shift < bits; shift += 8) {
    small_radix_pass<SMALL_TILE_ITEMS>(ki, vi, ko, vo, E, shift, s_wcnt, s_local, s_tmp);
    uint32_t *t0 = ki, *t1 = vi;
    ki = ko;
    vi = vo;
    ko = t0;
    vo = t1;
  }
  for (int e = tid; e < E; e += SMALL_THREADS) {
    const uint32_t t = ki[e];
    F.tile_key[e] = t;
    F.entry_val[e] = vi[e];
    if (e == 0 || ki[e - 1] != t) F.ranges[2 * (size_t)t] = (uint32_t)e;
    if (e == E - 1 || ki[e + 1] != t) F.ranges[2 * (size_t)t + 1] = (uint32_t)(e + 1);
  }
}

bool small_bin_ok(const lp_frame &F) {
  return F.n <= SMALL_N && F.capacity <= SMALL_E && F.capacity > 0;
}

void launch_small_depth_scan(const lp_frame &F, cudaStream_t st) {
  static bool init = false;
  const int smem = 4 * SMALL_N * 4;
  if (!init) {
    cudaFuncSetAttribute(k_small_depth_scan, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    init = true;
  }
  k_small_depth_scan<<<1, SMALL_THREADS, smem, st>>>(F, F.n);
}

void launch_small_tile_sort(const lp_frame &F, int bits, int tiles, cudaStream_t st) {
  static bool init = false;
  const int smem = 4 * SMALL_E * 4;
  if (!init) {
    cudaFuncSetAttribute(k_small_tile_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    init = true;
  }
  k_small_tile_sort<<<1, SMALL_THREADS, smem, st>>>(F, bits, tiles);
}

}  // namespace lp

// =============================================================================================
// LP_SORT_BUCKET: (tile, depth, id) order without a global sort.
//   K1 adds each visible primitive's tile rect to a 2-D difference grid (4 atomics);
//   k_tile_counts: 2-D prefix -> per-tile counts -> exclusive scan -> ranges, cursors, E;
//   k_bucket: every primitive appends (depth key, id) to the buckets of its tiles (cursor atomics;
//             order inside a bucket is arbitrary);
//   k_tile_sort: one CTA per tile sorts its bucket by the 64-bit (depth key << 32 | id) in shared
//             memory (bitonic network, ascending-only variant so +inf padding never moves), or in
//             place in global memory for a bucket larger than the shared-memory capacity.
// The result is the same total order as the radix path and the oracle.
// =============================================================================================
namespace lp {

constexpr int TS_THREADS = 256;
constexpr int TS_CAP = 4096;      // entries sorted in shared memory (32 KB of u64)

__global__ void __launch_bounds__(1024) k_tile_counts(int32_t *__restrict__ diff, int gx, int gy,
                                                      uint32_t *__restrict__ ranges, uint32_t *__restrict__ cursor,
                                                      uint32_t *__restrict__ counters, int64_t capacity) {
  extern __shared__ int32_t s_grid[];   // (gy+1) x (gx+1)
  __shared__ uint32_t s_warp[32];
  const int cols = gx + 1, rows = gy + 1, cells = cols * rows;
  for (int c = threadIdx.x; c < cells; c += blockDim.x) s_grid[c] = diff[c];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  // inclusive prefix along x, one warp per row (32-wide chunks with carry)
  for (int r = warp; r < rows; r += nw) {
    int carry = 0;
    for (int c0 = 0; c0 < cols; c0 += 32) {
      const int c = c0 + lane;
      int v = c < cols ? s_grid[r * cols + c] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
      }
      if (c < cols) s_grid[r * cols + c] = v + carry;
      carry += __shfl_sync(0xffffffffu, v, 31);
    }
  }
  __syncthreads();
  // inclusive prefix along y, one warp per column
  for (int c = warp; c < cols; c += nw) {
    int carry = 0;
    for (int r0 = 0; r0 < rows; r0 += 32) {
      const int r = r0 + lane;
      int v = r < rows ? s_grid[r * cols + c] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
      }
      if (r < rows) s_grid[r * cols + c] = v + carry;
      carry += __shfl_sync(0xffffffffu, v, 31);
    }
  }
  __syncthreads();
  // exclusive scan of the per-tile counts in row-major tile order
  const int tiles = gx * gy;
  uint32_t base = 0;
  for (int t0 = 0; t0 < tiles; t0 += blockDim.x) {
    const int t = t0 + threadIdx.x;
    const uint32_t cnt = t < tiles ? (uint32_t)s_grid[(t / gx) * cols + (t % gx)] : 0u;
    uint32_t total;
    const uint32_t ex = block_exclusive_scan(cnt, s_warp, total);
    if (t < tiles) {
      const uint32_t off = base + ex;
      ranges[2 * (size_t)t] = off;
      ranges[2 * (size_t)t + 1] = off + cnt;
      cursor[t] = off;
    }
    base += total;
  }
  if (threadIdx.x == 0) {
    counters[LP_CNT_ENTRIES] = base;
    counters[LP_CNT_OVERFLOW] = (int64_t)base > capacity ? 1u : 0u;
  }
}

__global__ void __launch_bounds__(256) k_bucket(const uint32_t *__restrict__ tt, const ushort4 *__restrict__ rect,
                                                const uint32_t *__restrict__ depth_key, int n, int tiles_x,
                                                int64_t capacity, uint32_t *__restrict__ cursor,
                                                uint32_t *__restrict__ bkey, uint32_t *__restrict__ bval) {
  const int lane = threadIdx.x & 31;
  const int i0 = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t my_tt = 0, my_key = 0;
  ushort4 my_r = make_ushort4(0, 0, 0, 0);
  if (i0 < n) {
    my_tt = tt[i0];
    if (my_tt) {
      my_r = rect[i0];
      my_key = depth_key[i0];
    }
  }
  unsigned todo = __ballot_sync(0xffffffffu, my_tt != 0);
  while (todo) {
    const int src = __ffs(todo) - 1;
    todo &= todo - 1;
    const uint32_t i = (uint32_t)((i0 & ~31) + src);
    const uint32_t cnt = __shfl_sync(0xffffffffu, my_tt, src);
    const uint32_t key = __shfl_sync(0xffffffffu, my_key, src);
    const uint32_t tx0 = __shfl_sync(0xffffffffu, (uint32_t)my_r.x, src);
    const uint32_t ty0 = __shfl_sync(0xffffffffu, (uint32_t)my_r.y, src);
    const uint32_t tx1 = __shfl_sync(0xffffffffu, (uint32_t)my_r.z, src);
    const uint32_t rw = tx1 - tx0 + 1;
    for (uint32_t k = lane; k < cnt; k += 32) {
      const uint32_t t = (ty0 + k / rw) * (uint32_t)tiles_x + tx0 + k % rw;
      const uint32_t pos = atomicAdd(cursor + t, 1u);
      if ((int64_t)pos < capacity) {
        bkey[pos] = key;
        bval[pos] = i;
      }
    }
  }
}

__device__ __forceinline__ unsigned long long composite(uint32_t key, uint32_t id) {
  return ((unsigned long long)key << 32) | id;
}

__global__ void __launch_bounds__(TS_THREADS) k_tile_sort(const uint32_t *__restrict__ ranges, int64_t capacity,
                                                          uint32_t *__restrict__ bkey, uint32_t *__restrict__ bval,
                                                          uint32_t *__restrict__ out_tile,
                                                          uint32_t *__restrict__ out_val) {
  __shared__ unsigned long long s_k[TS_CAP];
  const int t = blockIdx.x;
  int64_t off = ranges[2 * (size_t)t], end = ranges[2 * (size_t)t + 1];
  if (end > capacity) end = capacity;
  if (off >= end) return;
  const int L = (int)(end - off);
  int P = 1;
  while (P < L) P <<= 1;
  if (P <= TS_CAP) {
    for (int i = threadIdx.x; i < P; i += TS_THREADS)
      s_k[i] = i < L ? composite(bkey[off + i], bval[off + i]) : ~0ull;
    __syncthreads();
    for (int k = 2; k <= P; k <<= 1) {
      for (int j = k - 1; j > 0; j = (j == k - 1) ? (k >> 2) : (j >> 1)) {
        for (int i = threadIdx.x; i < P; i += TS_THREADS) {
          const int p = i ^ j;
          if (p > i) {
            const unsigned long long a = s_k[i], b = s_k[p];
            if (a > b) { s_k[i] = b; s_k[p] = a; }
          }
        }
        __syncthreads();
        if (k == 2) break;
      }
    }
    for (int i = threadIdx.x; i < L; i += TS_THREADS) {
      out_val[off + i] = (uint32_t)s_k[i];
      out_tile[off + i] = (uint32_t)t;
    }
    return;
  }
  // oversize bucket: the same network in place in global memory; partners beyond L are +inf
  uint32_t *K = bkey + off, *V = bval + off;
  for (int k = 2; k <= P; k <<= 1) {
    for (int j = k - 1; j > 0; j = (j == k - 1) ? (k >> 2) : (j >> 1)) {
      for (int i = threadIdx.x; i < L; i += TS_THREADS) {
        const int p = i ^ j;
        if (p > i && p < L) {
          const unsigned long long a = composite(K[i], V[i]), b = composite(K[p], V[p]);
          if (a > b) {
            K[i] = (uint32_t)(b >> 32); V[i] = (uint32_t)b;
            K[p] = (uint32_t)(a >> 32); V[p] = (uint32_t)a;
          }
        }
      }
      __syncthreads();
      if (k == 2) break;
    }
  }
  for (int i = threadIdx.x; i < L; i += TS_THREADS) {
    out_val[off + i] = V[i];
    out_tile[off + i] = (uint32_t)t;
  }
}

void launch_tile_counts(const lp_frame &F, cudaStream_t st) {
  const size_t smem = 4 * (size_t)(F.tiles_x + 1) * (F.tiles_y + 1);
  if (smem > 48 * 1024) {   // grids above ~12k tiles (e.g. > 4K x 3K pixels) need the opt-in carve-out
    if (cudaFuncSetAttribute(k_tile_counts, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return;   // the launch below is skipped; lp_bin_sort reports the recorded CUDA error
  }
  k_tile_counts<<<1, 1024, smem, st>>>(F.tile_diff, F.tiles_x, F.tiles_y, F.ranges, F.tile_cursor, F.counters,
                                       F.capacity);
}

void launch_bucket(const lp_frame &F, cudaStream_t st) {
  if (F.n == 0) return;
  k_bucket<<<(F.n + 255) / 256, 256, 0, st>>>(F.tiles_touched, reinterpret_cast<const ushort4 *>(F.rect), F.depth_key,
                                              F.n, F.tiles_x, F.capacity, F.tile_cursor, F.tile_key_alt,
                                              F.entry_val_alt);
}

void launch_tile_sort(const lp_frame &F, cudaStream_t st) {
  const int tiles = F.tiles_x * F.tiles_y;
  if (tiles == 0) return;
  k_tile_sort<<<tiles, TS_THREADS, 0, st>>>(F.ranges, F.capacity, F.tile_key_alt, F.entry_val_alt, F.tile_key,
                                            F.entry_val);
}

}  // namespace lp
