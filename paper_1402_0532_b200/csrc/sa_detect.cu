// sa_detect.cu -- detection on the device-resident map:
// detection.find_peaks (detection.py:85-108) and the two maxima behind
// detection.sidelobe_floor_db (detection.py:148-171).
//
// Magnitude: numpy's complex absolute value on this host is the SIMD loop
//   L = max(|re|,|im|), S = min(|re|,|im|), r = S/L (0 when L == 0),
//   |v| = sqrt(fma(r, r, 1)) * L
// (verified bit-exact against np.abs on 2e5 random complex128 / complex64
// values, tests/golden/make_golden.py); IEEE division / sqrt and an explicit
// fma reproduce it here, so strict comparisons and ties match the reference.
//
// Peaks: a cell qualifies when strictly greater than its 8 neighbours (cells
// beyond the edge are -inf and never block, detection.py:96-104); the k
// strongest are returned strongest first, equal magnitudes in row-major order
// (the stable argsort of detection.py:106).
//   k_peaks_strip (complex64, k <= 32, the default for those maps): one warp per
//     30-column x 64-row strip, rows walked in registers, each |v| computed once,
//     a running warp top k of integer keys; k_peaks_select_key merges the strip
//     lists (integer keys, refill loads prefetched one advance ahead);
//   k_peaks_tile: one CTA per 32x64 tile, magnitudes + halo in smem, strict
//     maxima; for k <= 32 each warp first extracts its own top k from registers
//     (k rounds of a warp argmax); a candidate's rank in the tile is the number
//     of better candidates, and the top k land sorted in the tile's list;
//   k_peaks_select: one CTA, k rounds of a block-wide argmax over the heads of
//     the tile lists (heads cached in registers, only the winner advances).
//     Maps up to 8192 tiles (16.7M cells) -- C5 is 4096.
// Floor: one grid-stride pass gives max |v| overall, max |v| outside every
// guard box (|l - l0| <= g0 and circular |p - p0| <= g1) and the number of
// outside cells; the dB arithmetic stays on the host as in the reference.
#include <algorithm>
#include <climits>

#include "sa_common.cuh"
#include "sa_internal.h"

namespace {

template <typename T> using C2 = typename SaVec<T>::c2;

struct Cand {
  double mag;
  long long idx;
};
constexpr int TILE = 32;    // tile rows
constexpr int TILE_W = 64;  // tile columns
constexpr int TILE_THREADS = 256;
constexpr int MAX_CAND = TILE * TILE_W / 4;  // strict maxima are never 8-adjacent: <= 1 per 2x2
constexpr int WARP_K = 32;  // k <= WARP_K: per-warp selection before the tile rank
constexpr int MERGE_THREADS = 512;
static_assert(TILE_W * 4 == 256 && (8 * WARP_K + 8 * 64) * 8 <= MAX_CAND * 16,
              "complex64 path: a warp's cells are 4 tile rows; key lists fit in cand");

SA_HD Cand sentinel() { return {-1.0, LLONG_MAX}; }
// strongest first; equal magnitudes in row-major order
SA_HD bool better(const Cand &a, const Cand &b) { return a.mag > b.mag || (a.mag == b.mag && a.idx < b.idx); }


template <typename T>
__global__ void __launch_bounds__(TILE_THREADS) k_peaks_tile(const C2<T> *__restrict__ map, int64_t rows,
                                                             int64_t cols, int k, Cand *__restrict__ out) {
  __shared__ T mag[TILE + 2][TILE_W + 3];
  __shared__ Cand cand[MAX_CAND];
  __shared__ int cnt;
  const int64_t r0 = (int64_t)blockIdx.y * TILE, c0 = (int64_t)blockIdx.x * TILE_W;
  if (threadIdx.x == 0) cnt = 0;
  auto fill = [&](int lr, int lc) {
    const int64_t r = r0 - 1 + lr, c = c0 - 1 + lc;
    T v = T(-INFINITY);
    if (r >= 0 && r < rows && c >= 0 && c < cols) {
      const C2<T> z = map[r * cols + c];
      v = np_cabs<T>(z.x, z.y);
    }
    mag[lr][lc] = v;
  };
  if constexpr (sizeof(T) == 4) {
    // the 64 tile columns of the TILE + 2 rows (shifts, no division), then the two
    // halo columns; all of a thread's loads are issued before the first magnitude
    constexpr int NL = ((TILE + 2) * TILE_W + 2 * (TILE + 2) + TILE_THREADS - 1) / TILE_THREADS;
    C2<T> z[NL];
    int lrc[NL];
#pragma unroll
    for (int i = 0; i < NL; ++i) {
      const int e = threadIdx.x + TILE_THREADS * i;
      int lr = -1, lc = 0;
      if (e < (TILE + 2) * TILE_W) lr = e / TILE_W, lc = e % TILE_W + 1;
      else if (e < (TILE + 2) * (TILE_W + 2)) lr = (e - (TILE + 2) * TILE_W) >> 1, lc = (e & 1) ? TILE_W + 1 : 0;
      const int64_t r = r0 - 1 + lr, c = c0 - 1 + lc;
      const bool in = lr >= 0 && r >= 0 && r < rows && c >= 0 && c < cols;
      lrc[i] = lr < 0 ? -1 : (lr << 8) | lc | (in ? 1 << 16 : 0);
      if (in) z[i] = __ldg(&map[r * cols + c]);
    }
#pragma unroll
    for (int i = 0; i < NL; ++i)
      if (lrc[i] >= 0)
        mag[(lrc[i] >> 8) & 255][lrc[i] & 255] = (lrc[i] >> 16) ? np_cabs<T>(z[i].x, z[i].y) : T(-INFINITY);
  } else {
    for (int e = threadIdx.x; e < (TILE + 2) * (TILE_W + 2); e += blockDim.x) fill(e / (TILE_W + 2), e % (TILE_W + 2));
  }
  __syncthreads();
  Cand *o = out + ((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * k;
  auto strict_at = [&](int e, Cand &cd) {  // tile cell e -> is it a strict maximum?
    const int lr = e / TILE_W + 1, lc = e % TILE_W + 1;
    const int64_t r = r0 + lr - 1, c = c0 + lc - 1;
    if (r >= rows || c >= cols) return false;
    const T m = mag[lr][lc];
    bool strict = true;
#pragma unroll
    for (int dl = -1; dl <= 1; ++dl)
#pragma unroll
      for (int dp = -1; dp <= 1; ++dp)
        if (dl != 0 || dp != 0) strict &= m > mag[lr + dl][lc + dp];
    cd = {(double)m, (long long)(r * cols + c)};
    return strict;
  };
  if (sizeof(T) == 4 && k <= WARP_K) {
    // complex64 maps, small k: integer keys (float magnitude bits << 32 | ~tile
    // index) -- larger key = stronger, ties to the earlier cell -- so each warp
    // argmax round is two redux.sync max (high word, then low word among the
    // lanes holding the high maximum) instead of five 128-bit shuffle rounds.
    using u64 = unsigned long long;
    constexpr int PER_LANE = TILE * TILE_W / TILE_THREADS;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // The warp's 256 cells are 4 tile rows: strict maxima are never 8-adjacent, so
    // at most 64 of them; they are compacted (ballot + prefix popcount) into a
    // per-warp list, at most two per lane, before the selection rounds.
    constexpr int NW = TILE_THREADS / 32;
    u64 *keys = reinterpret_cast<u64 *>(cand);  // 8 warps x WARP_K sorted winners
    u64 *wl = keys + warp * WARP_K;
    u64 *cl = keys + NW * WARP_K + warp * 64;   // this warp's strict maxima (cand holds 1024 u64)
    const unsigned lt = (1u << lane) - 1u;
    int nc = 0;
#pragma unroll
    for (int j = 0; j < PER_LANE; ++j) {
      const int e = warp * 32 * PER_LANE + lane + 32 * j;
      Cand cd;
      const bool st = strict_at(e, cd);
      const unsigned bal = __ballot_sync(0xffffffffu, st);
      if (st) cl[nc + __popc(bal & lt)] = ((u64)__float_as_uint((float)cd.mag) << 32) | (0xFFFFFFFFu - (unsigned)e);
      nc += __popc(bal);
    }
    __syncwarp();
    constexpr int SL = 2;
    u64 mine[SL];
#pragma unroll
    for (int j = 0; j < SL; ++j) mine[j] = lane + 32 * j < nc ? cl[lane + 32 * j] : 0ull;
    auto warp_max = [&](u64 b) {
      const unsigned mh = __reduce_max_sync(0xffffffffu, (unsigned)(b >> 32));
      const unsigned ml = __reduce_max_sync(0xffffffffu, (unsigned)(b >> 32) == mh ? (unsigned)b : 0u);
      return ((u64)mh << 32) | ml;
    };
    int got = 0;
    for (int rd = 0; rd < k && rd < nc; ++rd) {
      u64 b = 0;
#pragma unroll
      for (int j = 0; j < SL; ++j) b = mine[j] > b ? mine[j] : b;
      const u64 w = warp_max(b);
      if (lane == 0) wl[rd] = w;
      ++got;
#pragma unroll
      for (int j = 0; j < SL; ++j)
        if (mine[j] == w) mine[j] = 0;
    }
    for (int rd = got + lane; rd < k; rd += 32) wl[rd] = 0;
    __syncthreads();
    if (warp == 0) {  // k-way merge of the 8 sorted warp lists: lane w holds list w's head
      int pos = 0;
      u64 h = lane < NW ? keys[lane * WARP_K] : 0ull;
      int rd = 0;
      for (; rd < k; ++rd) {
        const u64 w = warp_max(h);
        if (w == 0) break;
        if (lane == 0) {
          const int e = (int)(0xFFFFFFFFu - (unsigned)w);
          o[rd] = {(double)__uint_as_float((unsigned)(w >> 32)),
                   (long long)((r0 + e / TILE_W) * cols + c0 + e % TILE_W)};
        }
        if (lane < NW && h == w) {
          ++pos;
          h = pos < k ? keys[lane * WARP_K + pos] : 0ull;
        }
      }
      for (int e = rd + lane; e < k; e += 32) o[e] = sentinel();
    }
    return;
  }
  if (k <= WARP_K) {
    // Small k: each warp keeps the strict maxima of its 256 cells in registers
    // (8 per lane), extracts its own top k by k rounds of a warp argmax, and the
    // tile ranks only those <= 8k warp winners.
    constexpr int PER_LANE = TILE * TILE_W / TILE_THREADS;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    Cand mine[PER_LANE];
#pragma unroll
    for (int j = 0; j < PER_LANE; ++j) {
      Cand cd;
      if (!strict_at(warp * 32 * PER_LANE + lane + 32 * j, cd)) cd = sentinel();
      mine[j] = cd;
    }
    Cand *wl = cand + warp * WARP_K;  // this warp's winners, best first
    int got = 0;
    for (int rd = 0; rd < k; ++rd) {
      Cand b = sentinel();
#pragma unroll
      for (int j = 0; j < PER_LANE; ++j)
        if (better(mine[j], b)) b = mine[j];
      for (int sh = 16; sh > 0; sh >>= 1) {
        Cand x;
        x.mag = __shfl_xor_sync(0xffffffffu, b.mag, sh);
        x.idx = __shfl_xor_sync(0xffffffffu, b.idx, sh);
        if (better(x, b)) b = x;
      }
      if (b.mag < 0.0) break;  // warp exhausted (uniform)
      if (lane == 0) wl[rd] = b;
      ++got;
#pragma unroll
      for (int j = 0; j < PER_LANE; ++j)
        if (mine[j].idx == b.idx) mine[j] = sentinel();
    }
    for (int rd = got + lane; rd < k; rd += 32) wl[rd] = sentinel();
    __syncthreads();
    if (warp == 0) {  // k-way merge of the 8 sorted warp lists: lane w holds list w's head
      constexpr int NW = TILE_THREADS / 32;
      int pos = 0;
      Cand h = lane < NW ? cand[lane * WARP_K] : sentinel();
      int rd = 0;
      for (; rd < k; ++rd) {
        Cand b = h;
        for (int sh = 16; sh > 0; sh >>= 1) {
          Cand x;
          x.mag = __shfl_xor_sync(0xffffffffu, b.mag, sh);
          x.idx = __shfl_xor_sync(0xffffffffu, b.idx, sh);
          if (better(x, b)) b = x;
        }
        if (b.mag < 0.0) break;
        if (lane == 0) o[rd] = b;
        if (lane < NW && h.idx == b.idx && h.mag >= 0.0) {
          ++pos;
          h = pos < k ? cand[lane * WARP_K + pos] : sentinel();
        }
      }
      for (int e = rd + lane; e < k; e += 32) o[e] = sentinel();
    }
    return;
  }
  for (int e = threadIdx.x; e < TILE * TILE_W; e += blockDim.x) {
    Cand cd;
    if (strict_at(e, cd)) cand[atomicAdd(&cnt, 1)] = cd;
  }
  __syncthreads();
  // the tile's top k by rank counting: a candidate's rank = number of better
  // candidates (a total order, so ranks are distinct); slot rank holds it
  const int n = cnt;
  for (int e = threadIdx.x; e < n; e += blockDim.x) {
    const Cand me = cand[e];
    int rank = 0;
    // branchless count, stopping once the candidate is out of the top k
    for (int j0 = 0; j0 < n && rank < k; j0 += 8) {
#pragma unroll
      for (int j = j0; j < j0 + 8; ++j)
        if (j < n) {
          const Cand c = cand[j];
          rank += (int)(c.mag > me.mag) | ((int)(c.mag == me.mag) & (int)(c.idx < me.idx));
        }
    }
    if (rank < k) o[rank] = me;
  }
  for (int e = n + threadIdx.x; e < k; e += blockDim.x) o[e] = sentinel();
}

// complex64 maps, k <= 32 (< 2^32 cells): one WARP per strip of 30 columns x
// SROWS rows, no shared memory.  Lane l holds column 30 s + l - 1 (lanes 0 and 31
// are the strip's halo columns), the warp walks down the rows keeping |v| of rows
// r - 1, r, r + 1 and their left / right neighbours (shuffles) in registers, with
// the loads of the next SPF rows in flight; each |v| is computed once.  Strict
// maxima become integer keys (float magnitude bits << 32 | ~index: larger =
// stronger, ties to the earlier cell) and enter the warp's running top k, a
// sorted list held one key per lane (lane i = i-th best) -- only keys above the
// current k-th best are inserted.  The list is the strip's sorted candidate list.
#ifndef SA_DET_SPF
#define SA_DET_SPF 4
#endif
#ifndef SA_DET_SROWS
#define SA_DET_SROWS 64
#endif
constexpr int SROWS = SA_DET_SROWS, SCOLS = 30, SPF = SA_DET_SPF, STRIP_THREADS = 128;
int64_t strip_lists(int64_t rows, int64_t cols) { return ((cols + SCOLS - 1) / SCOLS) * ((rows + SROWS - 1) / SROWS); }

__global__ void __launch_bounds__(STRIP_THREADS, 8) k_peaks_strip(const float2 *__restrict__ map, int64_t rows,
                                                               int64_t cols, int k,
                                                               unsigned long long *__restrict__ out) {
  using u64 = unsigned long long;
  const int lane = threadIdx.x & 31;
  const int64_t wid = ((int64_t)blockIdx.x * STRIP_THREADS + threadIdx.x) >> 5;
  const int64_t nstrips = (cols + SCOLS - 1) / SCOLS;
  if (wid >= nstrips * ((rows + SROWS - 1) / SROWS)) return;  // (warp-uniform)
  const int64_t seg = wid / nstrips, strip = wid % nstrips;
  const int64_t c = strip * SCOLS + lane - 1, rs = seg * SROWS, re = min(rs + SROWS, rows);
  const bool col_in = c >= 0 && c < cols;
  const bool own = lane >= 1 && lane <= SCOLS && col_in;
  const float2 *colp = map + (col_in ? c : 0);  // this lane's column
  auto load = [&](int64_t r) {  // row r of this lane's column (-inf magnitude outside the map)
    return (col_in && r >= 0 && r < rows) ? __ldg(colp + r * cols) : make_float2(NAN, NAN);
  };
  auto mag_of = [&](int64_t r, float2 z) {
    return (col_in && r >= 0 && r < rows) ? np_cabs<float>(z.x, z.y) : -INFINITY;
  };
  float2 pf[SPF];  // raw rows r + 2 .. r + 1 + SPF
#pragma unroll
  for (int i = 0; i < SPF; ++i) pf[i] = load(rs + 1 + i);
  float pm = mag_of(rs - 1, load(rs - 1));
  float cm = mag_of(rs, load(rs));
  float pl = __shfl_up_sync(~0u, pm, 1), pr = __shfl_down_sync(~0u, pm, 1);
  float cl = __shfl_up_sync(~0u, cm, 1), cr = __shfl_down_sync(~0u, cm, 1);
  u64 list = 0, thr = 0;  // lane i < k: the i-th best key so far; thr = the k-th best (0 until k found)
  for (int64_t r0 = rs; r0 < re; r0 += SPF) {
#pragma unroll
    for (int i = 0; i < SPF; ++i) {
      const int64_t r = r0 + i;
      if (r < re) {  // (warp-uniform)
        const float2 z = pf[i];
        pf[i] = load(r + 1 + SPF);
        const float nm = mag_of(r + 1, z);
        const float nl = __shfl_up_sync(~0u, nm, 1), nr = __shfl_down_sync(~0u, nm, 1);
        const bool st = own && cm > pl && cm > pm && cm > pr && cm > cl && cm > cr && cm > nl && cm > nm && cm > nr;
        const u64 key = ((u64)__float_as_uint(cm) << 32) | (0xFFFFFFFFu - (unsigned)(r * cols + c));
        unsigned bal = __ballot_sync(~0u, st && key > thr);
        while (bal) {  // insert the candidates above the k-th best, one at a time
          const int src = __ffs(bal) - 1;
          bal &= bal - 1;
          const u64 kk = __shfl_sync(~0u, key, src);
          if (kk <= thr) continue;  // (uniform) overtaken by an earlier insertion
          const int pos = __popc(__ballot_sync(~0u, lane < k && list > kk));
          const u64 up = __shfl_up_sync(~0u, list, 1);
          if (lane < k) list = lane < pos ? list : (lane == pos ? kk : up);
          thr = __shfl_sync(~0u, list, k - 1);
        }
        pm = cm, pl = cl, pr = cr;
        cm = nm, cl = nl, cr = nr;
      }
    }
  }
  if (lane < k) out[wid * k + lane] = list;  // the strip's sorted key list (0 past its last candidate)
}

// Global top k from the per-tile sorted lists (ntiles x k): k rounds of a
// block-wide argmax over the list heads.  Each thread caches the heads of its
// tiles (t = tid + j*MERGE_THREADS, j < HEADS) in registers; only the winner's
// owner advances.  Writes idx/mag (-1 / 0 past the last peak) and the count.
constexpr int HEADS = 16;

SA_HD Cand warp_best(Cand c) {
  for (int o = 16; o > 0; o >>= 1) {
    Cand x;
    x.mag = __shfl_xor_sync(0xffffffffu, c.mag, o);
    x.idx = __shfl_xor_sync(0xffffffffu, c.idx, o);
    if (better(x, c)) c = x;
  }
  return c;
}

__global__ void __launch_bounds__(MERGE_THREADS) k_peaks_select(const Cand *__restrict__ lists, int64_t ntiles,
                                                                int k, long long *idx, double *mag, int *count) {
  __shared__ Cand wbest[MERGE_THREADS / 32];
  __shared__ int wtile[MERGE_THREADS / 32];
  __shared__ Cand win;
  __shared__ int win_tile;
  Cand head[HEADS];
  int pos[HEADS];
#pragma unroll
  for (int j = 0; j < HEADS; ++j) {
    const int64_t t = threadIdx.x + (int64_t)j * MERGE_THREADS;
    pos[j] = 0;
    head[j] = t < ntiles ? lists[t * k] : sentinel();
  }
  int found = 0;
  for (int r = 0; r < k; ++r) {
    Cand best = sentinel();
    int bt = -1;
#pragma unroll
    for (int j = 0; j < HEADS; ++j)
      if (better(head[j], best)) {
        best = head[j];
        bt = j;
      }
    const Cand wb = warp_best(best);
    const unsigned owner = __ballot_sync(0xffffffffu, best.mag == wb.mag && best.idx == wb.idx && bt >= 0);
    if ((threadIdx.x & 31) == 0) {
      wbest[threadIdx.x >> 5] = wb;
      wtile[threadIdx.x >> 5] = owner ? (int)((threadIdx.x & ~31u) + __ffs(owner) - 1) : -1;
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      Cand c = threadIdx.x < MERGE_THREADS / 32 ? wbest[threadIdx.x] : sentinel();
      const Cand g = warp_best(c);
      const unsigned w = __ballot_sync(0xffffffffu, c.mag == g.mag && c.idx == g.idx && threadIdx.x < MERGE_THREADS / 32);
      if (threadIdx.x == 0) {
        win = g;
        win_tile = w ? wtile[__ffs(w) - 1] : -1;  // the owning thread
      }
    }
    __syncthreads();
    const Cand g = win;
    if (g.mag < 0.0) break;  // all lists exhausted
    if (threadIdx.x == 0) {
      idx[r] = g.idx;
      mag[r] = g.mag;
    }
    ++found;
    if ((int)threadIdx.x == win_tile) {  // advance the winning list
#pragma unroll
      for (int j = 0; j < HEADS; ++j)
        if (j == bt) {
          const int64_t t = threadIdx.x + (int64_t)j * MERGE_THREADS;
          ++pos[j];
          head[j] = pos[j] < k ? lists[t * k + pos[j]] : sentinel();
        }
    }
    __syncthreads();
  }
  for (int r = found + threadIdx.x; r < k; r += blockDim.x) {
    idx[r] = -1;
    mag[r] = 0.0;
  }
  if (threadIdx.x == 0) *count = found;
}

// complex64 maps (< 2^32 cells): the same selection on integer keys -- float
// magnitude bits << 32 | ~index (larger = stronger, ties to the earlier cell) --
// so a round is two redux.sync per warp and two block barriers.
constexpr int KSEL_THREADS = 1024, KHEADS = 8;
SA_HD unsigned long long cand_key(const Cand &c) {
  return c.mag < 0.0 ? 0ull
                     : ((unsigned long long)__float_as_uint((float)c.mag) << 32) | (0xFFFFFFFFu - (unsigned)c.idx);
}
SA_HD unsigned long long warp_max_key(unsigned long long b) {
  const unsigned mh = __reduce_max_sync(0xffffffffu, (unsigned)(b >> 32));
  const unsigned ml = __reduce_max_sync(0xffffffffu, (unsigned)(b >> 32) == mh ? (unsigned)b : 0u);
  return ((unsigned long long)mh << 32) | ml;
}
SA_HD unsigned long long cand_key(unsigned long long key) { return key; }
template <typename E> SA_HD E empty_of();
template <> SA_HD Cand empty_of<Cand>() { return sentinel(); }
template <> SA_HD unsigned long long empty_of<unsigned long long>() { return 0ull; }
template <typename E>
__global__ void __launch_bounds__(KSEL_THREADS) k_peaks_select_key(const E *__restrict__ lists, int64_t ntiles,
                                                                   int k, long long *idx, double *mag, int *count) {
  using u64 = unsigned long long;
  __shared__ u64 wk[KSEL_THREADS / 32];
  __shared__ u64 win;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // each list's head and the element after it, prefetched raw: a refill load is
  // only waited on when that list wins again (a dependent load per round would put
  // the L2 latency on every round's critical path)
  u64 head[KHEADS];
  E nxt[KHEADS];
  int pos[KHEADS];
#pragma unroll
  for (int j = 0; j < KHEADS; ++j) {
    const int64_t t = threadIdx.x + (int64_t)j * KSEL_THREADS;
    pos[j] = 0;
    head[j] = t < ntiles ? cand_key(lists[t * k]) : 0ull;
    nxt[j] = t < ntiles && k > 1 ? lists[t * k + 1] : empty_of<E>();
  }
  auto best_of = [&]() {
    u64 b = 0;
#pragma unroll
    for (int j = 0; j < KHEADS; ++j) b = head[j] > b ? head[j] : b;
    return b;
  };
  u64 best = best_of();  // only the owner of a round's winner changes its best
  int found = 0;
  for (int r = 0; r < k; ++r) {
    const u64 wb = warp_max_key(best);
    if (lane == 0) wk[warp] = wb;
    __syncthreads();
    if (warp == 0) {
      const u64 g = warp_max_key(lane < KSEL_THREADS / 32 ? wk[lane] : 0ull);
      if (lane == 0) win = g;
    }
    __syncthreads();
    const u64 g = win;
    if (g == 0) break;  // all lists exhausted
    if (threadIdx.x == 0) {
      idx[r] = (long long)(0xFFFFFFFFu - (unsigned)g);
      mag[r] = (double)__uint_as_float((unsigned)(g >> 32));
    }
    ++found;
    if (best == g) {  // the owner (keys are unique) advances the winning list
#pragma unroll
      for (int j = 0; j < KHEADS; ++j)
        if (head[j] == g) {
          const int64_t t = threadIdx.x + (int64_t)j * KSEL_THREADS;
          ++pos[j];
          head[j] = cand_key(nxt[j]);  // the refill load was issued when this list last advanced
          nxt[j] = pos[j] + 1 < k ? lists[t * k + pos[j] + 1] : empty_of<E>();
        }
      best = best_of();
    }
  }
  for (int r = found + threadIdx.x; r < k; r += blockDim.x) {
    idx[r] = -1;
    mag[r] = 0.0;
  }
  if (threadIdx.x == 0) *count = found;
}

SA_HD unsigned long long dbits(double v) { return (unsigned long long)__double_as_longlong(v); }

template <typename T>
__global__ void __launch_bounds__(256) k_map_floor(const C2<T> *__restrict__ map, int64_t rows, int64_t cols,
                                                   const int *__restrict__ centers, int ncent, int g0, int g1,
                                                   unsigned long long *out) {
  double all = 0.0, outside = 0.0;
  unsigned long long n_out = 0;
  const int64_t total = rows * cols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const C2<T> z = map[e];
    const double m = (double)np_cabs<T>(z.x, z.y);
    const int64_t l = e / cols, p = e % cols;
    bool in = false;
    for (int b = 0; b < ncent && !in; ++b) {
      const int64_t dl = l - centers[2 * b];
      int64_t d = (p - centers[2 * b + 1]) % cols;
      if (d < 0) d += cols;
      const int64_t dp = d < cols - d ? d : cols - d;
      in = (dl <= g0 && dl >= -g0 && dp <= g1);
    }
    all = fmax(all, m);
    if (!in) {
      outside = fmax(outside, m);
      ++n_out;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    all = fmax(all, __shfl_xor_sync(0xffffffffu, all, o));
    outside = fmax(outside, __shfl_xor_sync(0xffffffffu, outside, o));
    n_out += __shfl_xor_sync(0xffffffffu, n_out, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(&out[0], dbits(all));  // non-negative doubles order as their bit patterns
    atomicMax(&out[1], dbits(outside));
    atomicAdd(&out[2], n_out);
  }
}

int64_t n_tiles(int64_t rows, int64_t cols) { return ((rows + TILE - 1) / TILE) * ((cols + TILE_W - 1) / TILE_W); }

}  // namespace

int64_t sa_peaks_ws_bytes(int64_t rows, int64_t cols, int k) {
  return std::max(n_tiles(rows, cols), strip_lists(rows, cols)) * k * (int64_t)sizeof(Cand);
}

int sa_launch_map_peaks(int dtype, const void *map, int64_t rows, int64_t cols, int k, long long *idx, double *mag,
                        int *count, void *ws, cudaStream_t s) {
  const int64_t nt = n_tiles(rows, cols);
  if (nt > (int64_t)HEADS * MERGE_THREADS) {
    sa_set_error("find_peaks: map of %lld tiles exceeds %d", (long long)nt, HEADS * MERGE_THREADS);
    return SA_ERR_UNSUPPORTED;
  }
  Cand *lists = (Cand *)ws;
  const int64_t ns = strip_lists(rows, cols);
  if (dtype == SA_C64 && k <= WARP_K && rows * cols < 0xFFFFFFFFLL && ns <= (int64_t)KHEADS * KSEL_THREADS) {
    k_peaks_strip<<<(unsigned)((ns * 32 + STRIP_THREADS - 1) / STRIP_THREADS), STRIP_THREADS, 0, s>>>(
        (const float2 *)map, rows, cols, k, (unsigned long long *)ws);
    SA_LAUNCH_CHECK();
    k_peaks_select_key<<<1, KSEL_THREADS, 0, s>>>((const unsigned long long *)ws, ns, k, idx, mag, count);
    SA_LAUNCH_CHECK();
    return SA_OK;
  }
  dim3 grid((unsigned)((cols + TILE_W - 1) / TILE_W), (unsigned)((rows + TILE - 1) / TILE));
  if (dtype == SA_C64)
    k_peaks_tile<float><<<grid, TILE_THREADS, 0, s>>>((const float2 *)map, rows, cols, k, lists);
  else
    k_peaks_tile<double><<<grid, TILE_THREADS, 0, s>>>((const double2 *)map, rows, cols, k, lists);
  SA_LAUNCH_CHECK();
  if (dtype == SA_C64 && rows * cols <= 0xFFFFFFFFLL && nt <= (int64_t)KHEADS * KSEL_THREADS)
    k_peaks_select_key<<<1, KSEL_THREADS, 0, s>>>(lists, nt, k, idx, mag, count);
  else
    k_peaks_select<<<1, MERGE_THREADS, 0, s>>>(lists, nt, k, idx, mag, count);
  SA_LAUNCH_CHECK();
  return SA_OK;
}

int sa_launch_map_floor(int dtype, const void *map, int64_t rows, int64_t cols, const int *centers, int ncent,
                        int g0, int g1, unsigned long long *out, cudaStream_t s) {
  SA_CUDA_TRY(cudaMemsetAsync(out, 0, 3 * sizeof(unsigned long long), s));
  const int64_t total = rows * cols;
  const unsigned g = (unsigned)std::min<int64_t>((total + 255) / 256, 148 * 16);
  if (dtype == SA_C64)
    k_map_floor<float><<<g, 256, 0, s>>>((const float2 *)map, rows, cols, centers, ncent, g0, g1, out);
  else
    k_map_floor<double><<<g, 256, 0, s>>>((const double2 *)map, rows, cols, centers, ncent, g0, g1, out);
  SA_LAUNCH_CHECK();
  return SA_OK;
}
