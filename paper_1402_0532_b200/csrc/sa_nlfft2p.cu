// sa_nlfft2p.cu -- persistent work-queue NL-FFT for N = 2^16 (BASELINE config C3).
//
// N = 256 x 256 two-pass DIT (value-identical to transforms.py:254-298), built
// so that many independent tiles are in flight per SM and no CTA ever waits for
// a fixed partner:
//   A-item (signal s, column tile c0): TMA-load X[i][c0..c0+TC) (x[256 i + c]),
//     global stages 1..8 in two register radix-16 rounds (stage 1 = 2-point
//     NDFT bottom), store node rows R = rev8(c) into an L2-resident ring slot.
//   B-item (signal s, column tile q0): once all 16 A-items of s are done
//     (per-signal counter, release/acquire), TMA-load node columns q0.. of s,
//     stages 9..16 along R (twiddle j = (R mod 2^(t-1))*256 + q), store y.
// Items are handed out by one atomic ticket counter in the order
//   A(0) | A(1) B(0) | A(2) B(1) | ... | B(C-1)     (chunks of S signals)
// so a B-item's producers were dequeued one chunk earlier, and a ring slot is
// reused (A of chunk c waits for all B of chunk c-RING) only after its readers
// were dequeued: every wait targets items already held by running CTAs, so the
// persistent grid cannot deadlock.  The next item's tile is prefetched with TMA
// while the current one computes whenever its dependency is already satisfied.
// HBM traffic: x once, y once; the intermediate stays in L2 (ring of RING*S
// signals, re-written before it is evicted).
#include <algorithm>
#include <cudaTypedefs.h>

#include "sa_internal.h"
#include "sa_regs.cuh"

namespace {

constexpr int NN = 1 << 16;
constexpr int S_CHUNK = 16;  // signals per chunk
constexpr int LOOK = 2;      // A-items run LOOK chunks ahead of B-items
constexpr int RING = LOOK + 2;  // ring slots (chunks) for the intermediate
constexpr int TILES = 16;   // column tiles per signal per pass (TC = 16 / 8 -> 16 / 32)

template <typename T> struct Q;
template <> struct Q<float> {
  static constexpr int TC = 16;
  static constexpr int MINB = 2;  // CTAs per SM
};
template <> struct Q<double> {
  static constexpr int TC = 8;
  static constexpr int MINB = 2;
};

template <typename T> struct QP {
  static constexpr int TC = Q<T>::TC;
  static constexpr int THREADS = 16 * TC;
  static constexpr int NT = 256 / TC;  // tiles per pass per signal
  using C2 = typename Ar<T>::C2;
  using C4 = typename Ar<T>::C4;
  static constexpr size_t TILE = sizeof(C2) * 256 * TC;
  static constexpr size_t TWA = sizeof(C4) * 255;
  static constexpr size_t SMEM = 2 * TILE + TWA + 64;
  static constexpr int EW = sizeof(C2) / 8;
};

SA_HD int rev4(int v) { return (int)(__brev((unsigned)v) >> 28); }
SA_HD int rev8(int v) { return (int)(__brev((unsigned)v) >> 24); }
constexpr int crev4(int v) { return ((v & 1) << 3) | ((v & 2) << 1) | ((v & 4) >> 1) | ((v & 8) >> 3); }

struct Item {
  int kind;  // 0 = A, 1 = B, -1 = none
  int chunk;
  int64_t sig;
  int tile;
};

// ticket -> item.  Sequence: A(0..LOOK-1), then for p = LOOK .. C-1+LOOK:
// [A(p) if p < C] followed by [B(p-LOOK)].  itemsA = itemsB = NT * S per chunk.
SA_HD Item decode(int64_t t, int64_t nchunks, int nt) {
  const int64_t per = (int64_t)nt * S_CHUNK;
  Item it{-1, 0, 0, 0};
  const int64_t pre = (nchunks < LOOK ? nchunks : LOOK) * per;
  int64_t r, chunk;
  if (t < pre) {
    it.kind = 0;
    chunk = t / per;
    r = t % per;
  } else {
    int64_t tp = t - pre;
    int64_t nA = nchunks > LOOK ? nchunks - LOOK : 0;  // phases that still carry an A block
    if (tp < nA * 2 * per) {
      int64_t p = tp / (2 * per);
      r = tp % (2 * per);
      if (r < per) {
        it.kind = 0;
        chunk = p + LOOK;
      } else {
        it.kind = 1;
        chunk = p;
        r -= per;
      }
    } else {
      tp -= nA * 2 * per;
      chunk = nA + tp / per;
      r = tp % per;
      if (chunk >= nchunks) return it;  // past the end
      it.kind = 1;
    }
  }
  it.chunk = (int)chunk;
  it.sig = chunk * S_CHUNK + r / nt;
  it.tile = (int)(r % nt);
  return it;
}

SA_HD int ld_acquire(const int *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
SA_HD void red_release_add(int *p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
SA_HD void fence_proxy_async_all() { asm volatile("fence.proxy.async;" ::: "memory"); }

template <typename T>
__global__ void __launch_bounds__(QP<T>::THREADS, Q<T>::MINB)
    k_nlfft2p_dit(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmr,
                  typename Ar<T>::C2 *__restrict__ ring, typename Ar<T>::C2 *__restrict__ y,
                  int64_t batch, const typename Ar<T>::C4 *__restrict__ stage,
                  const typename Ar<T>::C2 *__restrict__ stage2, T gain, int use_gain,
                  int *__restrict__ ctr /* [ticket, cntA[batch], cntB[nchunks]] */) {
  using P = QP<T>;
  using A = Ar<T>;
  using V = typename A::V;
  using C2 = typename P::C2;
  using C4 = typename P::C4;
  constexpr int TC = P::TC, NT = P::NT;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  C2 *buf0 = reinterpret_cast<C2 *>(smem_raw);
  C4 *twA = reinterpret_cast<C4 *>(smem_raw + 2 * P::TILE);
  uint64_t *mbar = reinterpret_cast<uint64_t *>(smem_raw + 2 * P::TILE + P::TWA);
  volatile long long *s_next = reinterpret_cast<volatile long long *>(mbar + 2);  // [ticket, prefetched]

  const int64_t nchunks = (batch + S_CHUNK - 1) / S_CHUNK;
  int *ticket = ctr;
  int *cntA = ctr + 1;
  int *cntB = ctr + 1 + batch;
  const int tid = threadIdx.x;
  const int m1_cc = tid % TC, m1_g = tid / TC;
  const int m2_g = tid & 15, m2_cc = tid >> 4;

  for (int e = tid; e < 255; e += P::THREADS) twA[e] = stage[e];  // global stages 1..8
  if (tid == 0) {
    sa_mbar_init(&mbar[0], 1);
    sa_mbar_init(&mbar[1], 1);
    sa_fence_mbar_init();
  }
  __syncthreads();

  auto chunk_sigs = [&](int chunk) -> int {
    const int64_t left = batch - (int64_t)chunk * S_CHUNK;
    return (int)(left < S_CHUNK ? left : S_CHUNK);
  };
  // dependency of an item: B needs cntA[sig] == NT ; A (chunk >= RING) needs
  // cntB[chunk - RING] == NT * sigs(chunk - RING)
  auto dep_ready = [&](const Item &it) -> bool {
    if (it.kind == 1) return ld_acquire(&cntA[it.sig]) >= NT;
    if (it.chunk >= RING) return ld_acquire(&cntB[it.chunk - RING]) >= NT * chunk_sigs(it.chunk - RING);
    return true;
  };
  auto issue = [&](const Item &it, int b) {  // thread 0 only
    fence_proxy_async_all();
    sa_mbar_expect_tx(&mbar[b], (uint32_t)P::TILE);
    C2 *dst = buf0 + b * 256 * TC;
    if (it.kind == 0)
      sa_tma_load_2d(dst, &tmx, it.tile * TC * P::EW, (int)(it.sig * 256), &mbar[b]);
    else
      sa_tma_load_2d(dst, &tmr, it.tile * TC * P::EW,
                     (int)((((int64_t)(it.chunk % RING) * S_CHUNK) + (it.sig % S_CHUNK)) * 256), &mbar[b]);
  };
  auto valid = [&](const Item &it) { return it.kind >= 0 && it.sig < batch; };

  // prologue: first item (blocking dependency wait is safe: nothing is held)
  if (tid == 0) {
    int64_t t = atomicAdd(ticket, 1);
    Item it = decode(t, nchunks, NT);
    while (it.kind >= 0 && !valid(it)) {  // items of a partial last chunk: skip
      t = atomicAdd(ticket, 1);
      it = decode(t, nchunks, NT);
    }
    if (it.kind >= 0) {
      while (!dep_ready(it)) __nanosleep(64);
      issue(it, 0);
    }
    s_next[0] = t;
  }
  __syncthreads();
  int64_t t = s_next[0];
  int b = 0;
  uint32_t ph[2] = {0, 0};

  for (;;) {
    Item it = decode(t, nchunks, NT);
    if (it.kind < 0) break;
    // grab the next item now; prefetch its tile if its dependency already holds
    if (tid == 0) {
      int64_t tn = atomicAdd(ticket, 1);
      Item nx = decode(tn, nchunks, NT);
      while (nx.kind >= 0 && !valid(nx)) {
        tn = atomicAdd(ticket, 1);
        nx = decode(tn, nchunks, NT);
      }
      long long pre = 0;
      if (nx.kind >= 0 && dep_ready(nx)) {
        issue(nx, b ^ 1);
        pre = 1;
      }
      s_next[0] = tn;
      s_next[1] = pre;
    }
    sa_mbar_wait(&mbar[b], ph[b]);
    ph[b] ^= 1;
    C2 *wk = buf0 + b * 256 * TC;
    V v[16];
    if (it.kind == 0) {
      // ---------------- A-item: stages 1..8 on sub-transforms c = 16*tile + cc
      const int rg = rev4(m1_g);
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        V x = A::from(wk[(crev4(k) * 16 + rg) * TC + m1_cc]);
        v[k] = use_gain ? A::scale(x, gain) : x;
      }
#pragma unroll
      for (int k = 0; k < 16; k += 2) r_two_point<T>(v[k], v[k + 1]);  // stage 1
#pragma unroll
      for (int k = 0; k < 16; ++k)  // stage 2
        if (!(k & 2)) {
          if (k & 1) r_dit_mj<T>(v[k], v[k + 2]);
          else r_dit_one<T>(v[k], v[k + 2]);
        }
#pragma unroll
      for (int k = 0; k < 16; ++k)  // stage 3
        if (!(k & 4)) {
          const int j = k & 3;
          if (j == 0) r_dit_one<T>(v[k], v[k + 4]);
          else if (j == 2) r_dit_mj<T>(v[k], v[k + 4]);
          else r_dit<T>(v[k], v[k + 4], twA[3 + j]);
        }
#pragma unroll
      for (int k = 0; k < 8; ++k) {  // stage 4
        if (k == 0) r_dit_one<T>(v[k], v[k + 8]);
        else if (k == 4) r_dit_mj<T>(v[k], v[k + 8]);
        else r_dit<T>(v[k], v[k + 8], twA[7 + k]);
      }
      __syncthreads();
#pragma unroll
      for (int k = 0; k < 16; ++k) wk[(m1_g * 16 + k) * TC + (m1_cc ^ (k & (TC - 1)))] = A::to(v[k]);
      __syncthreads();
#pragma unroll
      for (int k = 0; k < 16; ++k) v[k] = A::from(wk[(m2_g + 16 * k) * TC + (m2_cc ^ (m2_g & (TC - 1)))]);
#pragma unroll
      for (int tt = 5; tt <= 8; ++tt) {
        const int hr = 1 << (tt - 5), h = 1 << (tt - 1);
#pragma unroll
        for (int k = 0; k < 16; ++k)
          if (!(k & hr)) r_dit<T>(v[k], v[k + hr], twA[(h - 1) + m2_g + 16 * (k & (hr - 1))]);
      }
      C2 *node = ring + (((int64_t)(it.chunk % RING) * S_CHUNK) + (it.sig % S_CHUNK)) * NN;
      const int R = rev8(it.tile * TC + m2_cc);
#pragma unroll
      for (int k = 0; k < 16; ++k) node[R * 256 + m2_g + 16 * k] = A::to(v[k]);
    } else {
      // ---------------- B-item: stages 9..16 on node columns q = TC*tile + qq
      const int q = it.tile * TC + m1_cc;
      const bool gen = __any_sync(0xffffffffu, q == 0 || q == 128);
#pragma unroll
      for (int k = 0; k < 16; ++k) v[k] = A::from(wk[(m1_g * 16 + k) * TC + m1_cc]);
      if (gen) {
#pragma unroll
        for (int tt = 1; tt <= 4; ++tt) {
          const int h = 1 << (tt - 1);
          C4 w[8];
#pragma unroll
          for (int a = 0; a < h; ++a) w[a] = sa_ldg(&stage[(1 << (7 + tt)) - 1 + a * 256 + q]);
#pragma unroll
          for (int k = 0; k < 16; ++k)
            if (!(k & h)) r_dit<T>(v[k], v[k + h], w[k & (h - 1)]);
        }
      } else {
#pragma unroll
        for (int tt = 1; tt <= 4; ++tt) {
          const int h = 1 << (tt - 1);
          C2 w[8];
#pragma unroll
          for (int a = 0; a < h; ++a) w[a] = sa_ldg(&stage2[(1 << (7 + tt)) - 1 + a * 256 + q]);
#pragma unroll
          for (int k = 0; k < 16; ++k)
            if (!(k & h)) r_dit_fast<T>(v[k], v[k + h], w[k & (h - 1)]);
        }
      }
#pragma unroll
      for (int k = 0; k < 16; ++k) wk[(m1_g * 16 + k) * TC + m1_cc] = A::to(v[k]);
      __syncthreads();
#pragma unroll
      for (int k = 0; k < 16; ++k) v[k] = A::from(wk[(m1_g + 16 * k) * TC + m1_cc]);
      if (gen) {
#pragma unroll
        for (int tt = 5; tt <= 8; ++tt) {
          const int hr = 1 << (tt - 5);
          C4 w[8];
#pragma unroll
          for (int a = 0; a < hr; ++a)
            w[a] = sa_ldg(&stage[(1 << (7 + tt)) - 1 + (m1_g + 16 * a) * 256 + q]);
#pragma unroll
          for (int k = 0; k < 16; ++k)
            if (!(k & hr)) r_dit<T>(v[k], v[k + hr], w[k & (hr - 1)]);
        }
      } else {
#pragma unroll
        for (int tt = 5; tt <= 8; ++tt) {
          const int hr = 1 << (tt - 5);
          C2 w[8];
#pragma unroll
          for (int a = 0; a < hr; ++a)
            w[a] = sa_ldg(&stage2[(1 << (7 + tt)) - 1 + (m1_g + 16 * a) * 256 + q]);
#pragma unroll
          for (int k = 0; k < 16; ++k)
            if (!(k & hr)) r_dit_fast<T>(v[k], v[k + hr], w[k & (hr - 1)]);
        }
      }
      C2 *ys = y + it.sig * NN;
#pragma unroll
      for (int k = 0; k < 16; ++k) __stcs(&ys[(m1_g + 16 * k) * 256 + q], A::to(v[k]));
    }
    __syncthreads();  // all stores of this item issued; tile buffer b free
    if (tid == 0) {
      if (it.kind == 0) {
        __threadfence();
        red_release_add(&cntA[it.sig], 1);  // node rows of this tile published
      } else {
        atomicAdd(&cntB[it.chunk], 1);  // ring slot reads of this tile done
      }
      if (!s_next[1]) {  // next item was not prefetched: wait for its dependency now
        Item nx = decode(s_next[0], nchunks, NT);
        if (nx.kind >= 0) {
          while (!dep_ready(nx)) __nanosleep(64);
          issue(nx, b ^ 1);
        }
      }
    }
    __syncthreads();
    t = s_next[0];
    b ^= 1;
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  }
  return fn;
}

template <typename T>
int make_map(CUtensorMap *map, const void *base, int64_t rows) {
  using P = QP<T>;
  auto enc = encode_fn();
  if (!enc) {
    sa_set_error("cuTensorMapEncodeTiled unavailable");
    return SA_ERR_CUDA;
  }
  cuuint64_t dims[2] = {(cuuint64_t)(256 * P::EW), (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(256 * sizeof(typename P::C2))};
  cuuint32_t box[2] = {(cuuint32_t)(P::TC * P::EW), 256};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, const_cast<void *>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    sa_set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
    return SA_ERR_CUDA;
  }
  return SA_OK;
}

template <typename T>
int launch2p(const void *x, void *y, int64_t batch, const SaTwiddles *tw, double gain,
             cudaStream_t s) {
  using P = QP<T>;
  const int64_t nchunks = (batch + S_CHUNK - 1) / S_CHUNK;
  const size_t ring_bytes = sizeof(typename P::C2) * (size_t)RING * S_CHUNK * NN;
  const size_t ctr_bytes = sizeof(int) * (size_t)(1 + batch + nchunks);
  void *ws = nullptr;
  {
    const int rc_ = sa_scratch_alloc((void **)&ws, ring_bytes + ctr_bytes, s);
    if (rc_) return rc_;
  }
  int *ctr = reinterpret_cast<int *>((char *)ws + ring_bytes);
  SA_CUDA_TRY(cudaMemsetAsync(ctr, 0, ctr_bytes, s));
  CUtensorMap mx, mr;
  int rc = make_map<T>(&mx, x, batch * 256);
  if (!rc) rc = make_map<T>(&mr, ws, (int64_t)RING * S_CHUNK * 256);
  if (rc) {
    cudaFreeAsync(ws, s);
    return rc;
  }
  auto kern = k_nlfft2p_dit<T>;
  SA_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P::SMEM));
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  SA_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, P::THREADS, P::SMEM));
  if (per_sm < 1) per_sm = 1;
  int64_t items = 2 * nchunks * (int64_t)P::NT * S_CHUNK;
  int grid = (int)std::min<int64_t>((int64_t)sms * per_sm, items);
  kern<<<grid, P::THREADS, P::SMEM, s>>>(mx, mr, (typename P::C2 *)ws, (typename P::C2 *)y, batch,
                                         (const typename P::C4 *)tw->stage,
                                         (const typename P::C2 *)tw->stage2, (T)gain,
                                         (int)(gain != 1.0), ctr);
  SA_LAUNCH_CHECK();
  SA_CUDA_TRY(cudaFreeAsync(ws, s));
  return SA_OK;
}

}  // namespace

int sa_launch_nlfft2p(int dtype, int variant, const void *x, void *y, int64_t batch, int64_t n,
                      const SaTwiddles *tw, double gain, cudaStream_t s) {
  if (n != NN || variant != SA_DIT || batch < 1 || x == y) return SA_ERR_UNSUPPORTED;
  if (((uintptr_t)x & 15) != 0) return SA_ERR_UNSUPPORTED;
  if (dtype == SA_C64) return launch2p<float>(x, y, batch, tw, gain, s);
  return launch2p<double>(x, y, batch, tw, gain, s);
}
