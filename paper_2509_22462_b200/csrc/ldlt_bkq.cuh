// Blocked Bunch-Kaufman LDL^T with the panel factored by ONE 8-CTA CLUSTER
// (round 2; the IPM's KKT sizes up to n = 16384).  Same contract, pivot rule,
// zero-pivot rules and output format as ldlt_bkp.cuh (reference
// proj/src/linalg.cpp:101-287: LAPACK dlasyf lower order, alpha =
// (1 + sqrt 17) / 8, ties to the smaller index, |d| <= eps -> zero L column,
// negligible column -> exact zero pivot).
//
// ldlt_bkp.cuh factors each panel in ONE CTA (n <= 2048) and stages the whole
// n x nb W panel in every CTA for the trailing update; the grid kernel
// ldlt_bk.cuh takes every larger n with several grid barriers per pivot.
// Here the panel's rows are spread over the 8 CTAs of cluster 0 (storage
// row P lives in CTA P % 8 at local index P / 8, up to 4 rows per thread),
// so one SM's shared memory holds 1/8 of the panel:
//   1. zs = D^{-1} W(q, :) -- jj remote (DSMEM) loads from q's owner CTA;
//   2. each CTA: its rows' entries of the updated column from its W slice,
//      a CTA maximum (key = |v| with 65535 - logical index in the low 16
//      bits, the signed value, the storage row), the diagonal by its owner;
//   3. one cluster barrier; lanes 0-7 of every warp read the 8 records in
//      ONE DSMEM round trip and every thread takes the SAME pivot decision;
//   4. column r (when the pivot test needs it) the same way into the scratch
//      slot of column jj + 1; a 1x1 pivot at r swaps the two slots' roles
//      (slot offsets, no data moves), a 2x2 block uses them as they are.
// Inside a panel interchanges only relabel: loc (logical -> storage row) is
// the identity but for <= nb displaced positions, a table in every cluster
// CTA's shared memory; each thread keeps the logical index and the active
// flag of its own rows in registers.  After the panel the whole grid applies
// the rank-nb update AND the panel's permutation in one pass over the
// trailing block, from one n x n buffer into the other:
//     A'(i, j) = A(loc i, loc j) - sum_c L(loc i, c) W(loc j, c),  i, j >= k0'
// (64 x 64 tiles on the FP64 tensor pipe, double-buffered cp.async gathers), so every panel starts from a
// compact trailing matrix in logical order: no retired rows inside the
// updated block, and shared memory never holds n x nb.  L columns are
// stored by ORIGINAL row (orig maps storage rows to original rows).
// Cooperative launch with __cluster_dims__(8): grid barriers and DSMEM.
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace gbb {
namespace bkq {

namespace cg = cooperative_groups;

constexpr int kC = 8;    // CTAs in the panel cluster (up to n = 9500) ...
constexpr int kC16 = 16;  // ... or 16 (non-portable cluster size; larger n: twice the slice room)
constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kR = 4;                        // panel rows per thread
constexpr int kMaxN = kC16 * kThreads * kR;  // 32768 (the key's 16-bit logical index allows 65535)
constexpr int kMaxNb = 32;
constexpr int kT = 64;                       // trailing-update tile (kT x kT)
constexpr int kLdA = kT + 1;                 // its A block's row stride (doubles; odd: column reads)
constexpr int kLdi = kT + 4;                 // L / W staging row stride (doubles)
constexpr double kAlpha = 0.64038820320220756872;  // (1 + sqrt(17)) / 8

struct Params {
  double* a;      // [n][n] full symmetric (equilibrated) matrix: panel 0's storage
  double* a2;     // [n][n] the other storage buffer (panels alternate)
  double* lcols;  // [n][n] L by logical column, ORIGINAL row (scratch)
  double* l;      // [n][ldl] output: unit lower L, logical order (strict lower part)
  int ldl;
  double* d;      // [n]
  double* e;      // [n]
  int* piv;       // [n]
  int* perm;      // [n] output: logical -> original row
  int* orig_a;    // [n] storage -> original row of buffer a ...
  int* orig_b;    // [n] ... and of a2
  int* locg;      // [n] the panel's loc, published for the update
  double* pan_w;  // [kMaxNb][n]: the panel's W columns (storage rows)
  double* pan_l;  // [kMaxNb][n]: the panel's L columns (storage rows)
  int* ctl;       // [4]: panel width
  int n;
  int nb;
  double eps;
  long long* trace;  // diagnostics (GBOPT_LDLT_TIMING): CTA 0's clocks per phase [10], or null
};

// shared-memory bytes of the panel kernel for (n, nb): the W slice
__host__ __device__ inline int64_t smem_bytes(int n, int nb, int ctas) {
  const int64_t lr = (n + ctas - 1) / ctas;
  return 8 * static_cast<int64_t>(nb + 2) * lr + 64;
}
// ... and of the update kernel: the A block, L and W staging, loc
constexpr int kUpdThreads = 256;
constexpr int kUpdSmem = 8 * (kT * kLdA + 2 * kMaxNb * kLdi) + 4 * 2 * kT;

// loc[i] from the displaced-position table (dpos[e] holds dval[e]; every
// other position is the identity): one warp-wide probe, uniform i
__device__ __forceinline__ int loc_of(int i, const int* dpos, const int* dval, int nd) {
  const int lane = threadIdx.x & 31;
  int v = i;
  for (int e0 = 0; e0 < nd; e0 += 32) {
    const int e = e0 + lane;
    const unsigned hit = __ballot_sync(0xffffffffu, e < nd && dpos[e] == i);
    if (hit) v = dval[e0 + __ffs(hit) - 1];
  }
  return v;
}

// index of position i in the displaced-position table (nd: not there), one
// warp-wide probe like loc_of
__device__ __forceinline__ int loc_slot(int i, const int* dpos, int nd) {
  const int lane = threadIdx.x & 31;
  for (int e0 = 0; e0 < nd; e0 += 32) {
    const unsigned hit = __ballot_sync(0xffffffffu, e0 + lane < nd && dpos[e0 + lane] == i);
    if (hit) return e0 + __ffs(hit) - 1;
  }
  return nd;
}

__device__ __forceinline__ unsigned long long pack_key(double v, int logical) {
  return (static_cast<unsigned long long>(__double_as_longlong(fabs(v))) & ~0xFFFFull) |
         static_cast<unsigned long long>(0xFFFF - logical);
}

// One CTA's candidate for the pivot search: its argmax key (see pack_key),
// the signed value and physical row there, and -- in the CTA owning the
// column's own row -- the diagonal entry.  Read remotely by every warp.
struct Rec {
  unsigned long long key;
  double val;
  double diag;
  int phys;
  int pad;
};

__device__ __forceinline__ void take_max(unsigned long long& key, double& val, int& phys, unsigned long long k2,
                                         double v2, int p2) {
  if (k2 > key) {
    key = k2;
    val = v2;
    phys = p2;
  }
}

// CTA-wide (key, value, row) maximum into rec (one CTA barrier; the cluster
// barrier that follows publishes it)
__device__ __forceinline__ void cta_best(unsigned long long key, double val, int phys, Rec* rec,
                                         unsigned long long* kwk, double* kwv, int* kwp) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long k2 = __shfl_xor_sync(0xffffffffu, key, o);
    const double v2 = __shfl_xor_sync(0xffffffffu, val, o);
    const int p2 = __shfl_xor_sync(0xffffffffu, phys, o);
    take_max(key, val, phys, k2, v2, p2);
  }
  if (lane == 0) {
    kwk[warp] = key;
    kwv[warp] = val;
    kwp[warp] = phys;
  }
  __syncthreads();
  if (warp == 0) {
    key = lane < kWarps ? kwk[lane] : 0ull;
    val = lane < kWarps ? kwv[lane] : 0.0;
    phys = lane < kWarps ? kwp[lane] : -1;
#pragma unroll
    for (int o = kWarps / 2; o > 0; o >>= 1) {
      const unsigned long long k2 = __shfl_xor_sync(0xffffffffu, key, o);
      const double v2 = __shfl_xor_sync(0xffffffffu, val, o);
      const int p2 = __shfl_xor_sync(0xffffffffu, phys, o);
      take_max(key, val, phys, k2, v2, p2);
    }
    if (lane == 0) {
      rec->key = key;
      rec->val = val;
      rec->phys = phys;
    }
  }
}

// The cluster's maximum from the kCl records (lanes 0..kCl-1 of every warp read
// one each, in parallel): its logical index (-1: no candidate), signed value
// and physical row, plus the diagonal held by CTA `owner`
template <int kCl>
__device__ __forceinline__ int cluster_best(cg::cluster_group& cluster, Rec* rec, int owner, double& val, int& phys,
                                            double& diag) {
  const int lane = threadIdx.x & 31;
  unsigned long long key = 0;
  double v = 0.0, dg = 0.0;
  int ph = -1;
  if (lane < kCl) {
    const Rec* r = cluster.map_shared_rank(rec, lane);
    key = r->key;
    v = r->val;
    dg = r->diag;
    ph = r->phys;
  }
  diag = __shfl_sync(0xffffffffu, dg, owner);
#pragma unroll
  for (int o = kCl / 2; o > 0; o >>= 1) {
    const unsigned long long k2 = __shfl_xor_sync(0xffffffffu, key, o);
    const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
    const int p2 = __shfl_xor_sync(0xffffffffu, ph, o);
    take_max(key, v, ph, k2, v2, p2);
  }
  key = __shfl_sync(0xffffffffu, key, 0);
  val = __shfl_sync(0xffffffffu, v, 0);
  phys = __shfl_sync(0xffffffffu, ph, 0);
  return key == 0 ? -1 : 0xFFFF - static_cast<int>(key & 0xFFFF);
}

// sum_c W(row, c) z_c over the panel's first jj columns (slot offsets soff)
__device__ __forceinline__ double panel_dot(const double* Wl, const int* soff, const double* z, int jj, int row) {
  double s0 = 0.0, s1 = 0.0;
  int c = 0;
  for (; c + 1 < jj; c += 2) {
    s0 = fma(Wl[soff[c] + row], z[c], s0);
    s1 = fma(Wl[soff[c + 1] + row], z[c + 1], s1);
  }
  if (c < jj) s0 = fma(Wl[soff[c] + row], z[c], s0);
  return s0 + s1;
}

__device__ __forceinline__ void cp_async8(void* smem_dst, const void* src, bool valid) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(valid ? 8 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

// D = A(8x4, row) * B(4x8, col) + D on the FP64 tensor pipe (DMMA.8x8x4):
// lane l holds A(l / 4, l % 4), B(l % 4, l / 4), D(l / 4, 2 (l % 4) + {0, 1})
__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}

// A'(i, j) = A(loc i, loc j) - sum_c L(loc i, c) W(loc j, c) for i, j in
// [k1, n): one 64 x 64 tile of the lower triangle per CTA pass (written
// with its mirror: A' stays symmetric), several CTAs per SM (their load,
// tensor-pipe and store phases overlap), on the FP64 tensor pipe: each of
// the 8 warps a 16 x 32 block = 2 x 4 DMMA 8x8x4 tiles, K = the panel
// width.  The A block, the L rows and the W rows are gathered with 8-byte
// cp.async (rows and columns through loc), L / W staged as [c][kLdi]
// (conflict-free writes and fragment loads); the result goes back through
// shared memory so A' is written in 512-byte rows.
__device__ void trailing_update(const double* __restrict__ a, double* __restrict__ a2,
                                const double* __restrict__ pl, const double* __restrict__ pw,
                                const int* __restrict__ locg, int n, int k1, int width, double* stage,
                                long long* tr) {
  const bool tracing = tr != nullptr && blockIdx.x == 0 && threadIdx.x == 0;
  long long tl = clock64(), t_issue = 0, t_wait = 0, t_fma = 0, t_store = 0;
  auto tmark = [&](long long& acc_) {
    if (tracing) {
      const long long now = clock64();
      acc_ += now - tl;
      tl = now;
    }
  };
  const int m = n - k1;
  const int tm = (m + kT - 1) / kT, tiles = tm * (tm + 1) / 2;  // the lower triangle of tiles
  const int kw = (width + 3) & ~3;          // K rounded to the DMMA step (zero-filled)
  double* A_ = stage;                       // [kT][kLdA]
  double* L_ = A_ + kT * kLdA;              // [kMaxNb][kLdi]
  double* W_ = L_ + kMaxNb * kLdi;          // [kMaxNb][kLdi]
  int* li = reinterpret_cast<int*>(W_ + kMaxNb * kLdi);  // [kT] loc of the tile's rows
  int* lj = li + kT;                                      // [kT] and columns
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wr = (warp >> 1) * 16, wc = (warp & 1) * 32;  // the warp's 16 x 32 block
  const int fr = lane >> 2, fk = lane & 3;                 // fragment row / k (col pair for D)
  for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    // tile = I (I + 1) / 2 + J, J <= I
    int I = static_cast<int>((sqrtf(8.0f * static_cast<float>(tile) + 1.0f) - 1.0f) * 0.5f);
    while (I * (I + 1) / 2 > tile) --I;
    while ((I + 1) * (I + 2) / 2 <= tile) ++I;
    const int J = tile - I * (I + 1) / 2;
    const int i0 = k1 + I * kT, j0 = k1 + J * kT;
    if (tid < 2 * kT) {
      const int x = tid < kT ? i0 + tid : j0 + tid - kT;
      li[tid] = x < n ? __ldcg(locg + x) : 0;  // li and lj are contiguous
    }
    __syncthreads();
#pragma unroll 4
    for (int u = 0; u < kT * kT / kUpdThreads; ++u) {
      const int x = tid + u * kUpdThreads, r = x / kT, c = x % kT;
      const bool ok = i0 + r < n && j0 + c < n;
      cp_async8(A_ + r * kLdA + c, ok ? a + static_cast<int64_t>(li[r]) * n + lj[c] : a, ok);
    }
#pragma unroll 4
    for (int u = 0; u < kMaxNb * kT / kUpdThreads; ++u) {
      const int x = tid + u * kUpdThreads, c = x / kT, i = x % kT;
      if (c < kw) {
        const bool oki = c < width && i0 + i < n, okj = c < width && j0 + i < n;
        cp_async8(L_ + c * kLdi + i, oki ? pl + static_cast<int64_t>(c) * n + li[i] : pl, oki);
        cp_async8(W_ + c * kLdi + i, okj ? pw + static_cast<int64_t>(c) * n + lj[i] : pw, okj);
      }
    }
    cp_async_commit();
    tmark(t_issue);
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncthreads();
    tmark(t_wait);
    double acc[2][4][2];
#pragma unroll
    for (int mb = 0; mb < 2; ++mb)
#pragma unroll
      for (int nb_ = 0; nb_ < 4; ++nb_) {
        const double* v = A_ + (wr + 8 * mb + fr) * kLdA + wc + 8 * nb_ + 2 * fk;
        acc[mb][nb_][0] = v[0];
        acc[mb][nb_][1] = v[1];
      }
    for (int c0 = 0; c0 < kw; c0 += 4) {
      double fa[2], fb[4];
#pragma unroll
      for (int mb = 0; mb < 2; ++mb) fa[mb] = -L_[(c0 + fk) * kLdi + wr + 8 * mb + fr];
#pragma unroll
      for (int nb_ = 0; nb_ < 4; ++nb_) fb[nb_] = W_[(c0 + fk) * kLdi + wc + 8 * nb_ + fr];
#pragma unroll
      for (int mb = 0; mb < 2; ++mb)
#pragma unroll
        for (int nb_ = 0; nb_ < 4; ++nb_) dmma884(acc[mb][nb_], fa[mb], fb[nb_]);
    }
    // back through shared memory (each warp rewrites its own block of A_)
#pragma unroll
    for (int mb = 0; mb < 2; ++mb)
#pragma unroll
      for (int nb_ = 0; nb_ < 4; ++nb_) {
        double* v = A_ + (wr + 8 * mb + fr) * kLdA + wc + 8 * nb_ + 2 * fk;
        v[0] = acc[mb][nb_][0];
        v[1] = acc[mb][nb_][1];
      }
    __syncthreads();
    tmark(t_fma);
#pragma unroll 4
    for (int u = 0; u < kT * kT / kUpdThreads; ++u) {
      const int x = tid + u * kUpdThreads, r = x / kT, c = x % kT;
      if (i0 + r < n && j0 + c < n) __stcg(a2 + static_cast<int64_t>(i0 + r) * n + j0 + c, A_[r * kLdA + c]);
    }
    if (I != J) {  // the mirror block A'(j, i) = A'(i, j): columns of the staged tile
#pragma unroll 4
      for (int u = 0; u < kT * kT / kUpdThreads; ++u) {
        const int x = tid + u * kUpdThreads, c = x / kT, r = x % kT;
        if (i0 + r < n && j0 + c < n) __stcg(a2 + static_cast<int64_t>(j0 + c) * n + i0 + r, A_[r * kLdA + c]);
      }
    }
    __syncthreads();  // A_, L_, W_, li / lj reusable
    tmark(t_store);
  }
  if (tracing) {
    tr[10] += t_issue;
    tr[11] += t_wait;
    tr[12] += t_fma;
    tr[13] += t_store;
  }
}

// One panel: the cluster (the whole launch, kCl CTAs) factors the nb columns
// from logical k0 = ctl[0] of the compact storage A (rows mapped to original
// rows by orig); publishes W / L by storage row, L by original row, loc
// (locg), the next buffer's orig (orig2) and the final perm entries of the
// panel, ctl[0] = k0 + width and ctl[1] = width.  No-op once k0 >= n.
template <int kCl>
__global__ void __cluster_dims__(kCl, 1, 1) __launch_bounds__(kThreads, 1)
    bkq_panel_kernel(Params p, const double* __restrict__ A, const int* __restrict__ orig, int* __restrict__ orig2) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ unsigned long long kwk[kWarps];
  __shared__ double kwv[kWarps];
  __shared__ int kwp[kWarps];
  __shared__ Rec crec[2][2];  // [pivot parity][column k, column r]
  __shared__ int soff[kMaxNb + 4];  // panel column c lives at Wl + soff[c]
  __shared__ double zs[kMaxNb], zr[kMaxNb], g0[kMaxNb], g1[kMaxNb];
  __shared__ int pp[kMaxNb];
  __shared__ int dpos[kMaxNb + 2], dval[kMaxNb + 2];  // loc's displaced positions (this panel)
  __shared__ int fin[kMaxNb + 2];                     // loc of the panel's own positions k0 + c
  __shared__ int s_nd;
  cg::cluster_group cluster = cg::this_cluster();
  const int n = p.n, nb = p.nb;
  const int k0 = __ldcg(p.ctl);
  if (k0 >= n) return;
  const int rank = static_cast<int>(blockIdx.x);  // = cluster rank
  const int lr = (n + kCl - 1) / kCl;   // local slice rows
  const int tid = threadIdx.x;
  long long tacc[10] = {};
  long long tlast = clock64();
  auto mark = [&](int i) {
    if (p.trace && blockIdx.x == 0 && tid == 0) {
      const long long t = clock64();
      tacc[i] += t - tlast;
      tlast = t;
    }
  };

  double* Wl = reinterpret_cast<double*>(smem_raw);  // [nb + 2][lr]: W columns of this CTA's rows

  // element P of the W column at slot offset `off` in P's owner's slice
  // (generic pointer, DSMEM when remote)
  auto wref = [&](int off, int P) -> const double* {
    return cluster.map_shared_rank(Wl, P % kCl) + off + P / kCl;
  };

  int parity = 0;
  {
    {
      // ---------------- panel (cluster 0) ----------------
      int k = k0, jj = 0;
      if (tid <= nb) soff[tid] = tid * lr;
      if (tid == 0) s_nd = 0;
      // this thread's rows: local index tid + t * kThreads, storage row P_t;
      // storage order = logical order at the panel's start
      int inv_t[kR];   // logical index of P_t
      bool act_t[kR];  // P_t not yet pivoted
      double arow[kR], anext[kR];
#pragma unroll
      for (int t = 0; t < kR; ++t) {
        const int P = (tid + t * kThreads) * kCl + rank;
        inv_t[t] = P;
        act_t[t] = tid + t * kThreads < lr && P < n && P >= k0;
        anext[t] = act_t[t] ? __ldcg(A + static_cast<int64_t>(k0) * n + P) : 0.0;
      }
      int q_next = k0;
      cluster.sync();  // every slice and the replicated state are current
      while (jj < nb && k < n) {
        const int nd = s_nd;
        const int q = loc_of(k, dpos, dval, nd);
#pragma unroll
        for (int t = 0; t < kR; ++t) {
          const int P = (tid + t * kThreads) * kCl + rank;
          arow[t] = q == q_next ? anext[t] : (act_t[t] ? __ldcg(A + static_cast<int64_t>(q) * n + P) : 0.0);
        }
        // 1. zs = D^{-1} W(q, 0:jj) from q's owner
        mark(9);
        if (tid < jj) zs[tid] = g0[tid] * *wref(soff[tid], q) + g1[tid] * *wref(soff[pp[tid]], q);
        __syncthreads();
        mark(0);
        // prefetch the likely next pivot row (logical k + 1)
        const int qn = k + 1 < n && jj + 1 < nb ? loc_of(k + 1, dpos, dval, nd) : -1;
        q_next = qn;
#pragma unroll
        for (int t = 0; t < kR; ++t) {
          const int P = (tid + t * kThreads) * kCl + rank;
          if (qn >= 0 && act_t[t]) anext[t] = __ldcg(A + static_cast<int64_t>(qn) * n + P);
        }
        // 2. this CTA's entries of the updated column, its (key, value, row) maximum
        unsigned long long key = 0;
        double val = 0.0;
        int phys = -1;
#pragma unroll
        for (int t = 0; t < kR; ++t) {
          if (!act_t[t]) continue;
          const int li = tid + t * kThreads, P = li * kCl + rank;
          const double v = arow[t] - panel_dot(Wl, soff, zs, jj, li);
          Wl[soff[jj] + li] = v;
          if (P != q) {
            take_max(key, val, phys, pack_key(v, inv_t[t]), v, P);
          } else {
            crec[parity][0].diag = v;
          }
        }
        cta_best(key, val, phys, &crec[parity][0], kwk, kwv, kwp);
        mark(1);
        cluster.sync();
        mark(2);
        // 3. the cluster's maximum and the diagonal, one DSMEM round trip
        double wkr, wkq;  // W(loc[r], k) signed (the column maximum), W(q, k) (the diagonal)
        int pr;           // loc[r]
        const int r = cluster_best<kCl>(cluster, &crec[parity][0], q % kCl, wkr, pr, wkq);
        const double lambda = fabs(wkr), absakk = fabs(wkq);
        int kind = 0;  // 0: 1x1 at k; 1: 1x1 at r (swap k <-> r); 2: 2x2 (k, r) (swap k+1 <-> r)
        const bool negl = !(fmax(absakk, lambda) > p.eps);  // linalg.cpp:143-157
        double wrr = 0.0;  // W_r(loc[r]): column r's diagonal
        mark(3);
        if (r >= 0 && !negl && absakk < kAlpha * lambda) {
          // 4. column r into the scratch slot of column jj + 1
          double ar[kR];
#pragma unroll
          for (int t = 0; t < kR; ++t) {
            const int P = (tid + t * kThreads) * kCl + rank;
            ar[t] = act_t[t] ? __ldcg(A + static_cast<int64_t>(pr) * n + P) : 0.0;
          }
          if (tid < jj) zr[tid] = g0[tid] * *wref(soff[tid], pr) + g1[tid] * *wref(soff[pp[tid]], pr);
          __syncthreads();
          unsigned long long key2 = 0;
          double val2 = 0.0;
          int phys2 = -1;
#pragma unroll
          for (int t = 0; t < kR; ++t) {
            if (!act_t[t]) continue;
            const int li = tid + t * kThreads, P = li * kCl + rank;
            const double v = ar[t] - panel_dot(Wl, soff, zr, jj, li);
            Wl[soff[jj + 1] + li] = v;
            if (P != pr) {
              take_max(key2, val2, phys2, pack_key(v, inv_t[t]), v, P);
            } else {
              crec[parity][1].diag = v;
            }
          }
          cta_best(key2, val2, phys2, &crec[parity][1], kwk, kwv, kwp);
          cluster.sync();
          double wsr;
          int pr2;
          cluster_best<kCl>(cluster, &crec[parity][1], pr % kCl, wsr, pr2, wrr);
          const double sigma = fabs(wsr);
          if (absakk * sigma >= kAlpha * lambda * lambda)
            kind = 0;
          else if (fabs(wrr) >= kAlpha * sigma)
            kind = 1;
          else
            kind = 2;
          mark(4);
        }
        if (kind == 2 && jj + 1 >= nb) break;  // no room for the 2x2 block: it opens the next panel
        // interchange (logical labels only, replicated in every CTA), retire the pivot rows
        const int a_ = kind == 1 ? k : k + 1;
        const int pa = kind != 0 && a_ != r ? (kind == 1 ? q : loc_of(k + 1, dpos, dval, nd)) : -1;
        const int e_r = pa >= 0 ? loc_slot(r, dpos, nd) : 0;  // where position r goes in the table
        const int p0 = kind == 1 ? pr : q;
        const int p1 = kind == 2 ? pr : -1;
        const double dk = negl ? 0.0 : (kind == 1 ? wrr : wkq);
        double gk0, gk1 = 0.0, gr0 = 0.0;
        if (kind != 2) {
          gk0 = fabs(dk) > p.eps ? 1.0 / dk : 0.0;  // |d| <= eps: zero L column (linalg.cpp:226-229)
        } else {
          const double det = wkq * wrr - wkr * wkr;  // [[W(p0,k), W(p1,k)], [W(p1,k), W_r(p1)]]
          gk0 = wrr / det;
          gk1 = -wkr / det;
          gr0 = wkq / det;
        }
        // the owners update their rows' registers
#pragma unroll
        for (int t = 0; t < kR; ++t) {
          const int P = (tid + t * kThreads) * kCl + rank;
          if (pa >= 0) {
            if (P == pr) inv_t[t] = a_;
            if (P == pa) inv_t[t] = r;
          }
          if (P == p0 || P == p1) act_t[t] = false;
        }
        __syncthreads();  // every thread has read the loc table and soff
        if (tid == 0) {
          // loc: positions k (, k + 1) are final; position r takes pa
          fin[jj] = p0;
          if (kind == 2) fin[jj + 1] = p1;
          if (pa >= 0) {
            dpos[e_r] = r;
            dval[e_r] = pa;
            if (e_r == nd) s_nd = nd + 1;
          }
          if (kind == 1) {  // the pivot column is column r: swap the slots, move no data
            const int t = soff[jj];
            soff[jj] = soff[jj + 1];
            soff[jj + 1] = t;
          }
          // D and D^{-1} from the values every CTA already holds
          g0[jj] = gk0;
          g1[jj] = gk1;
          pp[jj] = kind == 2 ? jj + 1 : jj;
          if (kind == 2) {
            g0[jj + 1] = gr0;
            g1[jj + 1] = gk1;
            pp[jj + 1] = jj;
          }
          if (rank == 0) {
            p.d[k] = kind == 2 ? wkq : dk;
            p.e[k] = kind == 2 ? wkr : 0.0;
            p.piv[k] = kind == 2 ? 2 : 1;
            if (kind == 2) {
              p.d[k + 1] = wrr;
              p.e[k + 1] = 0.0;
              p.piv[k + 1] = -2;
            }
          }
        }
        __syncthreads();
        mark(5);
        parity ^= 1;
        const int step = kind == 2 ? 2 : 1;
        k += step;
        jj += step;
      }
      // publish the panel: W and L columns by storage row for the update,
      // L by original row for the output (each CTA its rows); rank 0: loc
      // over [k0, n) and the width
#pragma unroll
      for (int t = 0; t < kR; ++t) {
        const int li = tid + t * kThreads, P = li * kCl + rank;
        if (li >= lr || P >= n || P < k0) continue;
        const int o = __ldcg(orig + P);
        for (int c = 0; c < jj; ++c) {
          const double w = Wl[soff[c] + li];
          const double l = g0[c] * w + g1[c] * Wl[soff[pp[c]] + li];
          __stcg(p.pan_w + static_cast<int64_t>(c) * n + P, w);
          __stcg(p.pan_l + static_cast<int64_t>(c) * n + P, l);
          __stcg(p.lcols + static_cast<int64_t>(k0 + c) * n + o, l);
        }
      }
      if (rank == 0) {
        for (int i = k0 + jj + tid; i < n; i += kThreads) p.locg[i] = i;
        __syncthreads();
        const int nd = s_nd;
        if (tid < nd && dpos[tid] >= k0 + jj) p.locg[dpos[tid]] = dval[tid];
        if (tid < jj) p.locg[k0 + tid] = fin[tid];
      }
      cluster.sync();  // the slices are read remotely until here; locg is complete
      // positions [k0, k1) are final (perm); the rest maps the next buffer
      const int k1 = k0 + jj;
      for (int i = k0 + rank * kThreads + tid; i < n; i += kCl * kThreads)
        (i < k1 ? p.perm : orig2)[i] = __ldcg(orig + __ldcg(p.locg + i));
      if (rank == 0 && tid == 0) {
        p.ctl[0] = k1;
        p.ctl[1] = jj;
      }
      mark(6);
    }
  }
  if (p.trace && blockIdx.x == 0 && tid == 0)
    for (int i = 0; i < 10; ++i) p.trace[i] += tacc[i];
}

// The panel's trailing update into the other buffer (no-op once k1 >= n)
__global__ void __launch_bounds__(kUpdThreads, 3) bkq_update_kernel(Params p, const double* __restrict__ A,
                                                                 double* __restrict__ A2) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int n = p.n, k1 = __ldcg(p.ctl), width = __ldcg(p.ctl + 1);
  if (k1 >= n) return;
  trailing_update(A, A2, p.pan_l, p.pan_w, p.locg, n, k1, width, reinterpret_cast<double*>(smem_raw), p.trace);
}

// storage -> original map of the first buffer (the identity), ctl[0] = 0
__global__ void bkq_init_kernel(Params p) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < p.n; i += gridDim.x * blockDim.x) p.orig_a[i] = i;
  if (blockIdx.x == 0 && threadIdx.x == 0) p.ctl[0] = 0;
}

// L in logical order: L(i, c) = lcols[c][perm[i]], c < i
__global__ void bkq_gather_kernel(Params p) {
  const int n = p.n;
  for (int i = blockIdx.x; i < n; i += gridDim.x) {
    const int P = __ldcg(p.perm + i);
    double* dst = p.l + static_cast<int64_t>(i) * p.ldl;
    for (int c = threadIdx.x; c < i; c += blockDim.x) dst[c] = __ldcg(p.lcols + static_cast<int64_t>(c) * n + P);
  }
}

}  // namespace bkq
}  // namespace gbb
