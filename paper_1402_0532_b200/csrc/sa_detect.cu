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
  for (int e = threadIdx.x; e < (TILE + 2) * (TILE_W + 2); e += blockDim.x) {
    const int lr = e / (TILE_W + 2), lc = e % (TILE_W + 2);
    const int64_t r = r0 - 1 + lr, c = c0 - 1 + lc;
    T v = T(-INFINITY);
    if (r >= 0 && r < rows && c >= 0 && c < cols) {
      const C2<T> z = map[r * cols + c];
      v = np_cabs<T>(z.x, z.y);
    }
    mag[lr][lc] = v;
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
    u64 mine[PER_LANE];
#pragma unroll
    for (int j = 0; j < PER_LANE; ++j) {
      const int e = warp * 32 * PER_LANE + lane + 32 * j;
      Cand cd;
      mine[j] = strict_at(e, cd) ? ((u64)__float_as_uint((float)cd.mag) << 32) | (0xFFFFFFFFu - (unsigned)e) : 0ull;
    }
    u64 *keys = reinterpret_cast<u64 *>(cand);  // 8 warps x WARP_K sorted winners
    u64 *wl = keys + warp * WARP_K;
    auto warp_max = [&](u64 b) {
      const unsigned mh = __reduce_max_sync(0xffffffffu, (unsigned)(b >> 32));
      const unsigned ml = __reduce_max_sync(0xffffffffu, (unsigned)(b >> 32) == mh ? (unsigned)b : 0u);
      return ((u64)mh << 32) | ml;
    };
    int got = 0;
    for (int rd = 0; rd < k; ++rd) {
      u64 b = 0;
#pragma unroll
      for (int j = 0; j < PER_LANE; ++j) b = mine[j] > b ? mine[j] : b;
      const u64 w = warp_max(b);
      if (w == 0) break;  // warp exhausted (uniform)
      if (lane == 0) wl[rd] = w;
      ++got;
#pragma unroll
      for (int j = 0; j < PER_LANE; ++j)
        if (mine[j] == w) mine[j] = 0;
    }
    for (int rd = got + lane; rd < k; rd += 32) wl[rd] = 0;
    __syncthreads();
    if (warp == 0) {  // k-way merge of the 8 sorted warp lists: lane w holds list w's head
      constexpr int NW = TILE_THREADS / 32;
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

int64_t sa_peaks_ws_bytes(int64_t rows, int64_t cols, int k) { return n_tiles(rows, cols) * k * (int64_t)sizeof(Cand); }

int sa_launch_map_peaks(int dtype, const void *map, int64_t rows, int64_t cols, int k, long long *idx, double *mag,
                        int *count, void *ws, cudaStream_t s) {
  const int64_t nt = n_tiles(rows, cols);
  if (nt > (int64_t)HEADS * MERGE_THREADS) {
    sa_set_error("find_peaks: map of %lld tiles exceeds %d", (long long)nt, HEADS * MERGE_THREADS);
    return SA_ERR_UNSUPPORTED;
  }
  Cand *lists = (Cand *)ws;
  dim3 grid((unsigned)((cols + TILE_W - 1) / TILE_W), (unsigned)((rows + TILE - 1) / TILE));
  if (dtype == SA_C64)
    k_peaks_tile<float><<<grid, TILE_THREADS, 0, s>>>((const float2 *)map, rows, cols, k, lists);
  else
    k_peaks_tile<double><<<grid, TILE_THREADS, 0, s>>>((const double2 *)map, rows, cols, k, lists);
  SA_LAUNCH_CHECK();
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
