// Bunch-Kaufman LDL^T of a small dense symmetric matrix held entirely in
// the distributed shared memory of ONE 16-CTA thread-block cluster
// (right-looking, the KKT systems of the reduced-space IPM,
// n ~ 800).  Same contract and output format as the cooperative-grid kernel
// in ldlt_bk.cuh (P A P^T = L D L^T, (P b)_i = b[perm[i]], piv 1 / 2 / -2),
// same pivoting rule as the reference (proj/src/linalg.cpp:101-287, LAPACK
// dsytf2 lower, alpha = (1 + sqrt 17) / 8, ties to the smaller index).
//
// Why: at n ~ 800 the left-looking grid kernel is latency-bound (~8 us per
// pivot: L2 round trips plus ~1.2 us grid barriers).  Here the lower
// triangle (n^2 / 2 doubles, 3.1 MB at n = 882) stays on chip and a pivot
// step is two cluster barriers, column gathers over distributed shared
// memory and a rank-1 (or rank-2) update from shared memory.
//
// Distribution: the pair {i, j} (i >= j, physical indices) lives in CTA
// (i + j) mod 16, so every row AND every column is spread evenly over the
// 16 CTAs: gathering a column reads n / 16 values from each CTA, and each
// CTA updates 1/16 of every trailing row.  CTA c stores, row after row, the
// entries j = j0(i), j0(i) + 16, ... <= i of row i, j0(i) = (c - i) mod 16;
// row_off(i, c) is the start of row i.
//
// Symmetric interchanges move no data: physical row P always holds original
// row P; `loc` maps the logical (pivot-order) index to its physical row and
// `inv` back, so an interchange k <-> r swaps two entries of loc.  A
// physical index is "active" while its logical index has not been pivoted;
// retired pairs hold L entries (and D in the pivot slots).
//
// Per step k (logical):
//   1. every CTA gathers column k of the trailing matrix (physical indexing,
//      stored residue-major so the update reads it without bank conflicts)
//      and, when |a_kk| < alpha lambda, column r; every CTA makes the same
//      pivot decision from its copies; cluster barrier;
//   2. loc / inv are swapped, the pivot indices retired;
//   3. each CTA writes the L entries of its pairs in the pivot column(s) and
//      applies A -= w w^T / d (or the 2x2 form) to its pairs; cluster barrier.
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace gbb {
namespace bkc {

namespace cg = cooperative_groups;

constexpr int kCtas = 16;      // cluster size (non-portable; B200 GPCs hold 16 SMs)
constexpr int kThreads = 512;  // per CTA
constexpr int kWarps = kThreads / 32;
constexpr double kAlpha = 0.64038820320220756872;  // (1 + sqrt(17)) / 8

struct Params {
  const double* a;  // [n][n] symmetric input, row-major (the equilibrated matrix)
  double* l;        // [n][ldl] unit lower factor, logical order (strict lower part written)
  int ldl;
  double* d;        // [n]
  double* e;        // [n]
  int* piv;         // [n]
  int* perm;        // [n]
  int n;
  double eps;  // zero-pivot threshold 1e-11 max|SAS| (linalg.cpp:101, 143-157, 226-229)
  long long* trace;  // diagnostics (GBOPT_LDLT_TIMING): rank 0's clock at 6 points per step, or null
};

// rows b in [0, 16) of a 16-row block whose entry count in CTA c gets +1:
// b >= (c - b) mod 16
__host__ __device__ inline unsigned extra_mask(int c) {
  unsigned m = 0;
  for (int b = 0; b < 16; ++b)
    if (b >= ((c - b) & 15)) m |= 1u << b;
  return m;
}
__host__ __device__ inline int popc16(unsigned v) {
#ifdef __CUDA_ARCH__
  return __popc(v);
#else
  return __builtin_popcount(v);
#endif
}
// entries of rows [0, i) stored in CTA c: row 16a + b holds a + [b in mask]
__host__ __device__ inline int64_t row_off(int i, unsigned mask) {
  const int64_t A = i >> 4, B = i & 15;
  return 8 * A * (A - 1) + A * popc16(mask) + A * B + popc16(mask & ((1u << B) - 1u));
}
// padded column-buffer length (residue-major: [16][cols16])
__host__ __device__ inline int cols16(int n) { return (n + 15) / 16; }

__host__ __device__ inline int64_t max_pairs(int n) {
  int64_t m = 0;
  for (int c = 0; c < kCtas; ++c) {
    const int64_t r = row_off(n, extra_mask(c));
    m = r > m ? r : m;
  }
  return m;
}

// Shared-memory bytes the kernel needs for dimension n
inline int64_t smem_bytes(int n) {
  const int64_t dbl = max_pairs(n) + 2 * 16 * static_cast<int64_t>(cols16(n));  // pairs | col | colr
  return 8 * dbl + 8 * static_cast<int64_t>(n) /* loc, inv */ + 2 * static_cast<int64_t>(n) /* active, pivk */ + 16;
}

// (value, index) maximum with ties to the smaller index (index < 0: none)
__device__ __forceinline__ void max_pair(double& v, int& i, double v2, int i2) {
  if (i2 >= 0 && (i < 0 || v2 > v || (v2 == v && i2 < i))) {
    v = v2;
    i = i2;
  }
}

struct Smem {
  double* pairs;  // this CTA's pairs, row after row
  double* col;    // gathered column k, residue-major: col[(Q & 15) * c16 + (Q >> 4)]
  double* colr;   // gathered column r, same layout
  int* loc;
  int* inv;
  unsigned char* active;
  signed char* pivk;  // [n] per logical index: 1, or 2 / -2 for the rows of a 2x2 block
  int c16;
};

__device__ __forceinline__ int cix(const Smem& s, int Q) { return (Q & 15) * s.c16 + (Q >> 4); }

// CTA-wide (value, index) maximum; result in every thread
__device__ void cta_max(double& v, int& i, double* rv, int* ri) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
    const int i2 = __shfl_xor_sync(0xffffffffu, i, o);
    max_pair(v, i, v2, i2);
  }
  __syncthreads();
  if (lane == 0) {
    rv[warp] = v;
    ri[warp] = i;
  }
  __syncthreads();
  v = -1.0;
  i = -1;
  for (int w = 0; w < kWarps; ++w) max_pair(v, i, rv[w], ri[w]);
}

// Gather column `q` (physical) of the active trailing matrix into this CTA's
// `buf` with distributed-shared-memory loads -- pair {Q, q} from CTA
// (Q + q) mod 16 -- and return its off-diagonal maximum (|value|, logical
// index), identical in every CTA and every thread.
__device__ double column_pull(cg::cluster_group& cluster, const Smem& s, const unsigned* masks, int n, int q,
                              double* buf, int& idx, double* rv, int* ri) {
  double m = -1.0;
  int mi = -1;
#pragma unroll 1
  for (int Q0 = threadIdx.x; Q0 < n; Q0 += 2 * kThreads) {
    double v[2];
    bool ok[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int Q = Q0 + u * kThreads;
      ok[u] = Q < n && s.active[Q];
      if (ok[u]) {
        const int hi = Q > q ? Q : q, lo = Q > q ? q : Q;
        const int owner = (hi + lo) & 15;
        const int64_t off = row_off(hi, masks[owner]) + ((lo - ((owner - hi) & 15)) >> 4);
        v[u] = *cluster.map_shared_rank(s.pairs + off, owner);
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int Q = Q0 + u * kThreads;
      if (Q >= n) continue;
      buf[cix(s, Q)] = ok[u] ? v[u] : 0.0;  // retired entries read as 0: the update leaves them alone
      if (ok[u] && Q != q) max_pair(m, mi, fabs(v[u]), s.inv[Q]);
    }
  }
  cta_max(m, mi, rv, ri);
  idx = mi;
  return m;
}

__global__ void __launch_bounds__(kThreads, 1) bkc_factor_kernel(Params p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ double rv[kWarps];
  __shared__ int ri[kWarps];
  __shared__ unsigned masks[kCtas];
  __shared__ int s_qmin;
  cg::cluster_group cluster = cg::this_cluster();
  const int n = p.n;
  const int rank = static_cast<int>(cluster.block_rank());
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x < kCtas) masks[threadIdx.x] = extra_mask(threadIdx.x);

  Smem s;
  s.c16 = cols16(n);
  double* dp = reinterpret_cast<double*>(smem_raw);
  s.pairs = dp;
  dp += max_pairs(n);
  s.col = dp;
  s.colr = dp + 16 * s.c16;
  dp += 32 * s.c16;
  s.loc = reinterpret_cast<int*>(dp);
  s.inv = s.loc + n;
  s.active = reinterpret_cast<unsigned char*>(s.inv + n);
  s.pivk = reinterpret_cast<signed char*>(s.active + n);
  __syncthreads();
  const unsigned mymask = masks[rank];

  // ---- load this CTA's pairs: row i, j = j0(i) + 16 u <= i ----
  for (int i = warp; i < n; i += kWarps) {
    const int j0 = (rank - i) & 15;
    double* rp = s.pairs + row_off(i, mymask);
    const double* ap = p.a + static_cast<int64_t>(i) * n;
    for (int u = lane; j0 + 16 * u <= i; u += 32) rp[u] = __ldg(ap + j0 + 16 * u);
  }
  for (int i = threadIdx.x; i < n; i += kThreads) {
    s.loc[i] = i;
    s.inv[i] = i;
    s.active[i] = 1;
  }
  if (threadIdx.x == 0) {
    s_qmin = 0;
  }
  __syncthreads();
  cluster.sync();  // every CTA's pairs loaded before any remote read

  auto mark = [&](int k, int i) {
    if (p.trace && rank == 0 && threadIdx.x == 0) p.trace[6 * k + i] = clock64();
  };
  for (int k = 0; k < n;) {
    mark(k, 0);
    int r;
    const double lambda = fmax(column_pull(cluster, s, masks, n, s.loc[k], s.col, r, rv, ri), 0.0);
    const double absakk = fabs(s.col[cix(s, s.loc[k])]);
    int kind = 0;  // 0: 1x1 at k; 1: 1x1 at r (swap k <-> r); 2: 2x2 (k, r) (swap k+1 <-> r)
    if (r >= 0 && fmax(absakk, lambda) > p.eps && absakk < kAlpha * lambda) {
      int r2;
      const double sigma = fmax(column_pull(cluster, s, masks, n, s.loc[r], s.colr, r2, rv, ri), 0.0);
      if (absakk * sigma >= kAlpha * lambda * lambda)
        kind = 0;
      else if (fabs(s.colr[cix(s, s.loc[r])]) >= kAlpha * sigma)
        kind = 1;
      else
        kind = 2;
    }
    mark(k, 1);
    cluster.sync();  // every CTA has read the matrix for this step before any pair changes
    mark(k, 2);
    if (threadIdx.x == 0) {
      const int a = kind == 1 ? k : k + 1;
      if (kind != 0 && a != r) {
        const int pa = s.loc[a], pr = s.loc[r];
        s.loc[a] = pr;
        s.loc[r] = pa;
        s.inv[pr] = a;
        s.inv[pa] = r;
      }
      // retire the pivot indices; qmin = the smallest active physical index
      s.active[s.loc[k]] = 0;
      if (kind == 2) s.active[s.loc[k + 1]] = 0;
      int q = s_qmin;
      while (q < n && !s.active[q]) ++q;
      s_qmin = q;
      s.pivk[k] = kind == 2 ? 2 : 1;
      if (kind == 2) s.pivk[k + 1] = -2;
    }
    __syncthreads();
    mark(k, 3);
    const int p0 = s.loc[k];
    const int p1 = kind == 2 ? s.loc[k + 1] : -1;
    const int qmin = s_qmin;
    double* wa = kind == 1 ? s.colr : s.col;  // pivot column
    double* wb = s.colr;                       // second pivot column (2x2)
    // D block; for 2x2, [L(i,k) L(i,k+1)] = [wa_i wb_i] D^{-1}
    const double a2 = wa[cix(s, p0)], b2 = kind == 2 ? wa[cix(s, p1)] : 0.0, c2 = kind == 2 ? wb[cix(s, p1)] : 0.0;
    const double det = a2 * c2 - b2 * b2;
    const double rdk = fabs(a2) > p.eps ? 1.0 / a2 : 0.0;  // |d| <= eps: no update (linalg.cpp:226-229)
    __syncthreads();  // D read by every thread before the pivot entries are cleared
    if (threadIdx.x == 0) {
      // the pivot indices are retired: their column entries must not update anything
      wa[cix(s, p0)] = 0.0;
      if (kind == 2) {
        wa[cix(s, p1)] = 0.0;
        wb[cix(s, p0)] = 0.0;
        wb[cix(s, p1)] = 0.0;
      }
    }
    __syncthreads();
    // the update of this CTA's active pairs {P, Q}, qmin <= Q <= P:
    // kLanesRow threads per row (rows hold only ~(P - qmin) / 16 entries
    // here), thread s of a row taking entries u0 + s + kLanesRow e so
    // neighbouring threads touch neighbouring words.  Retired Q read a zero
    // column entry: their pairs (L entries) are rewritten unchanged.
    constexpr int kLanesRow = 8;
    const int nact = n - qmin;
    for (int x = threadIdx.x; x < nact * kLanesRow; x += kThreads) {
      const int P = qmin + x / kLanesRow;
      if (!s.active[P]) continue;
      const int j0 = (rank - P) & 15;
      // stored entries j = j0 + 16 u, u in [u0, cnt): those at or after qmin
      const int u0 = (qmin > j0 ? (qmin - j0 + 15) >> 4 : 0) + (x % kLanesRow);
      const int cnt = P >= j0 ? ((P - j0) >> 4) + 1 : 0;
      double* rp = s.pairs + row_off(P, mymask);
      const double* wra = wa + j0 * s.c16;  // column entries j = j0 + 16 u at wra[u]
      const double* wrb = wb + j0 * s.c16;
      if (kind != 2) {
        const double lp = wa[cix(s, P)] * rdk;
        for (int u = u0; u < cnt; u += 4 * kLanesRow) {
          double av[4], wv[4];
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (u + kLanesRow * e < cnt) {
              av[e] = rp[u + kLanesRow * e];
              wv[e] = wra[u + kLanesRow * e];
            }
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (u + kLanesRow * e < cnt) rp[u + kLanesRow * e] = fma(-lp, wv[e], av[e]);
        }
      } else {
        const double x0 = wa[cix(s, P)], x1 = wb[cix(s, P)];
        const double l0 = (x0 * c2 - x1 * b2) / det, l1 = (x1 * a2 - x0 * b2) / det;
        for (int u = u0; u < cnt; u += 4 * kLanesRow) {
          double av[4], w0v[4], w1v[4];
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (u + kLanesRow * e < cnt) {
              av[e] = rp[u + kLanesRow * e];
              w0v[e] = wra[u + kLanesRow * e];
              w1v[e] = wrb[u + kLanesRow * e];
            }
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (u + kLanesRow * e < cnt) rp[u + kLanesRow * e] = fma(-l0, w0v[e], fma(-l1, w1v[e], av[e]));
        }
      }
    }
    __syncthreads();  // the update's read-modify-writes are done before the L entries land
    // this CTA's pairs {Q, p} of the pivot column(s), Q active: L(Q, k) / L(Q, k + 1)
    for (int h = 0; h < (kind == 2 ? 2 : 1); ++h) {
      const int pp = h == 0 ? p0 : p1;
      const int qres = (rank - pp) & 15;
      for (int t = threadIdx.x; qres + 16 * t < n; t += kThreads) {
        const int Q = qres + 16 * t;
        if (!s.active[Q]) continue;
        const int hi = Q > pp ? Q : pp, lo = Q > pp ? pp : Q;
        double* slot = s.pairs + row_off(hi, mymask) + ((lo - ((rank - hi) & 15)) >> 4);
        const double x0 = wa[cix(s, Q)];
        if (kind != 2) {
          *slot = x0 * rdk;
        } else {
          const double x1 = wb[cix(s, Q)];
          *slot = h == 0 ? (x0 * c2 - x1 * b2) / det : (x1 * a2 - x0 * b2) / det;
        }
      }
    }
    mark(k, 4);
    cluster.sync();  // every pair updated before the next column is gathered
    mark(k, 5);
    k += kind == 2 ? 2 : 1;
  }

  // ---- outputs: perm, piv, D (diagonal and 2x2 pair slots), and L in
  //      logical order (pairs inside a 2x2 block -> 0) ----
  if (rank == 0)
    for (int i = threadIdx.x; i < n; i += kThreads) {
      p.perm[i] = s.loc[i];
      p.piv[i] = s.pivk[i];
    }
  for (int P = warp; P < n; P += kWarps) {
    const int j0 = (rank - P) & 15;
    const double* rp = s.pairs + row_off(P, mymask);
    const int i = s.inv[P];
    for (int u = lane; j0 + 16 * u <= P; u += 32) {
      const int Q = j0 + 16 * u;
      const double v = rp[u];
      if (Q == P) {
        p.d[i] = v;
        if (s.pivk[i] != 2) p.e[i] = 0.0;
        continue;
      }
      const int j = s.inv[Q];
      const int hi = i > j ? i : j, lo = i > j ? j : i;
      const bool blk = hi == lo + 1 && s.pivk[lo] == 2;
      if (blk) p.e[lo] = v;
      p.l[static_cast<int64_t>(hi) * p.ldl + lo] = blk ? 0.0 : v;
    }
  }
}

}  // namespace bkc
}  // namespace gbb
