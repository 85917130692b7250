// Bunch-Kaufman LDL^T of a dense symmetric matrix on the device: one
// cooperative (grid-synchronised) launch for the whole factorisation, one
// single-CTA launch per solve.  Replaces cuSOLVER's dsytrf / sytrs for the
// KKT row f3 (reference proj/src/linalg.cpp:101-287 factor, 393-438 solve).
//
// Factorisation, left-looking, one pivot (1x1 or 2x2) per step:
//   column k of the updated matrix is  w = A(:, k) - L(:, 0:k) * (D L(k, 0:k)^T)
//   (a GEMV over the rows of L; the original matrix A is only permuted, never
//   updated), so a step touches L's rows below k once and needs no trailing
//   update.  The Bunch-Kaufman test (alpha = (1 + sqrt 17) / 8) picks, from
//   the column maximum lambda of w and -- when |w_k| < alpha lambda -- the
//   updated column r of that maximum and its off-diagonal maximum sigma:
//     1x1 at k;  1x1 at r (swap k <-> r);  or 2x2 at (k, r) (swap k+1 <-> r)
//   exactly as LAPACK's dsytf2 / the reference's panel code.  Symmetric
//   interchanges are applied to the trailing part of A, to the rows of L
//   computed so far, and recorded in perm, so that on exit
//       P A P^T = L D L^T,   (P b)_i = b[perm[i]].
//   Per step: every CTA recomputes v = D L(k, 0:k)^T into shared memory; warps
//   take rows i >= k; a grid-wide barrier publishes the column maxima, a
//   second (only for non-trivial pivots) those of column r, a third the swap
//   and the new L column(s).  Ties in the maxima resolve to the smallest row
//   index, and every reduction has a fixed order: the factorisation is
//   deterministic.
//
// Solve (x = P^T L^-T D^-1 L^-1 P b): one cooperative launch, forward /
// backward substitution in 32-row blocks (block updates by the whole grid,
// the 32 x 32 triangle by one warp from shared memory), block-diagonal D in
// between.
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace gbb {
namespace bk {

namespace cg = cooperative_groups;

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr double kAlpha = 0.64038820320220756872;  // (1 + sqrt(17)) / 8

struct Factor {
  double* a;      // [n][n] full symmetric (permuted in place; only rows/cols >= k are read at step k)
  double* l;      // [n][ldl] unit lower factor, row-major (row i holds L(i, 0:i)); ldl even (16-B rows)
  double* wd;     // [n][ldl] W = L D: row k of W is v = D L(k, 0:k)^T, the GEMV vector of step k
                  // (W's new columns are the updated columns themselves, before the pivot division)
  double* d;      // [n] D diagonal
  double* e;      // [n] D subdiagonal (e[k] = D(k+1, k) of a 2x2 block, else 0)
  int* piv;       // [n] 1: 1x1 block; 2 / -2: first / second row of a 2x2 block
  int* perm;      // [n] P: row i of the factorisation is original row perm[i]
  double* w;      // [n] updated column k (ping-pong with w2 across look-ahead steps)
  double* w2;     // [n]
  double* wr;     // [n] updated column r
  double* part;   // [2 * grid] per-CTA maxima of column k (value, index as double); ping-pong with part3
  double* part3;  // [2 * grid]
  double* part2;  // [2 * grid] the same for column r (separate: CTAs may still read part)
  int n;
  int ldl;
  double eps;  // zero-pivot threshold 1e-11 max|SAS| (linalg.cpp:101, 143-157, 226-229)
  int nb;  // > 0: blocked -- column updates span only the current panel's
           // columns, and the trailing A takes a rank-nb update per panel
  long long* trace;  // null, or [16]: CTA 0's clocks -- trailing updates (incl. their barrier), whole kernel,
                     // phases (column k, decision, column r, look-ahead, interchange + new column), phase counts
};

// (value, index) maximum with ties to the smaller index
__device__ __forceinline__ void max_pair(double& v, int& i, double v2, int i2) {
  if (v2 > v || (v2 == v && i2 >= 0 && (i < 0 || i2 < i))) {
    v = v2;
    i = i2;
  }
}

// CTA-wide (value, index) maximum, result valid in every thread
__device__ double cta_max(double v, int& idx, double* sv, int* si) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
    const int i2 = __shfl_xor_sync(0xffffffffu, idx, o);
    max_pair(v, idx, v2, i2);
  }
  __syncthreads();
  if (lane == 0) {
    sv[warp] = v;
    si[warp] = idx;
  }
  __syncthreads();
  v = -1.0;
  idx = -1;
  for (int k = 0; k < kWarps; ++k) max_pair(v, idx, sv[k], si[k]);
  return v;
}

// grid-wide (value, index) maximum over the per-CTA partials
__device__ double grid_max(const double* part, int& idx, double* sv, int* si) {
  double v = -1.0;
  idx = -1;
  // up to 2 partials per thread (grid <= 2 kThreads), both loads in flight before the compares
  const int c0 = threadIdx.x, c1 = threadIdx.x + kThreads, g = static_cast<int>(gridDim.x);
  const double v0 = c0 < g ? __ldcg(part + 2 * c0) : -1.0, i0 = c0 < g ? __ldcg(part + 2 * c0 + 1) : -1.0;
  const double v1 = c1 < g ? __ldcg(part + 2 * c1) : -1.0, i1 = c1 < g ? __ldcg(part + 2 * c1 + 1) : -1.0;
  if (c0 < g) max_pair(v, idx, v0, static_cast<int>(i0));
  if (c1 < g) max_pair(v, idx, v1, static_cast<int>(i1));
  for (int c = threadIdx.x + 2 * kThreads; c < g; c += kThreads)
    max_pair(v, idx, __ldcg(part + 2 * c), static_cast<int>(__ldcg(part + 2 * c + 1)));
  return cta_max(v, idx, sv, si);
}

// v[j0:k] = W(row, j0:k) = (D L(row, j0:k)^T)^T into shared memory (16-byte
// loads; j0 even, v[j0 .. k0) zeroed by the caller's choice of k0)
__device__ void d_times_lrow(const Factor& F, int row, int k0, int k, double* v) {
  const double* wr = F.wd + static_cast<int64_t>(row) * F.ldl;
  const int j0 = k0 & ~1;
  for (int j = j0 + 2 * threadIdx.x; j < k; j += 2 * kThreads) {
    if (j + 1 < k) {
      const double2 t = __ldcg(reinterpret_cast<const double2*>(wr + j));
      v[j] = j < k0 ? 0.0 : t.x;  // only j0 = k0 - 1 can be outside the panel
      v[j + 1] = t.y;
    } else {
      v[j] = j < k0 ? 0.0 : __ldcg(wr + j);
    }
  }
}

// Narrow panels (k - (k0 & ~1) <= 128, the blocked mode): kRowBatch rows per
// warp pass with every load in flight before the first FMA -- a warp owns
// several rows at large n, and one row per round trip made the column
// phases latency-bound.  Lane l covers columns jb + 2l and jb + 2l + 64.
constexpr int kRowBatch = 4;
__device__ __forceinline__ void panel_dots(const Factor& F, int k0, int k, const double* v, int ibase, int stride,
                                           double (&sum)[kRowBatch]) {
  const int lane = threadIdx.x & 31, jb = k0 & ~1;
  double2 a[kRowBatch][2];
#pragma unroll
  for (int r = 0; r < kRowBatch; ++r) {
    const int i = ibase + r * stride;
    const double* li = F.l + static_cast<int64_t>(i < F.n ? i : 0) * F.ldl;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = jb + 2 * lane + 64 * h;
      if (i < F.n && j + 1 < k)
        a[r][h] = __ldcg(reinterpret_cast<const double2*>(li + j));
      else
        a[r][h] = make_double2(i < F.n && j < k ? __ldcg(li + j) : 0.0, 0.0);
    }
  }
  double2 vv[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int j = jb + 2 * lane + 64 * h;
    vv[h] = make_double2(j < k ? v[j] : 0.0, j + 1 < k ? v[j + 1] : 0.0);
  }
#pragma unroll
  for (int r = 0; r < kRowBatch; ++r) {
    double t = fma(a[r][0].x, vv[0].x, fma(a[r][0].y, vv[0].y, 0.0));
    t = fma(a[r][1].x, vv[1].x, fma(a[r][1].y, vv[1].y, t));
    sum[r] = t;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int r = 0; r < kRowBatch; ++r) sum[r] += __shfl_xor_sync(0xffffffffu, sum[r], o);
}

// out[i] = A[i][col] - L(i, 0:k) . v for i >= k (one warp per row), and the
// CTA's maximum of |out[i]| over i >= k, i != skip
__device__ double column_update(const Factor& F, int col, int k0, int k, const double* v, double* out, int skip,
                                int& idx, double* sv, int* si) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gw = blockIdx.x * kWarps + warp, nw = gridDim.x * kWarps;
  double m = -1.0;
  idx = -1;
  if (k - (k0 & ~1) <= 128) {
    for (int ib = k + gw; ib < F.n; ib += kRowBatch * nw) {
      double av[kRowBatch], sum[kRowBatch];
#pragma unroll
      for (int r = 0; r < kRowBatch; ++r) {
        const int i = ib + r * nw;
        av[r] = i < F.n ? __ldcg(F.a + static_cast<int64_t>(col) * F.n + i) : 0.0;
      }
      panel_dots(F, k0, k, v, ib, nw, sum);
#pragma unroll
      for (int r = 0; r < kRowBatch; ++r) {
        const int i = ib + r * nw;
        if (i >= F.n) break;
        const double wi = av[r] - sum[r];
        if (lane == 0) out[i] = wi;
        if (i != skip) max_pair(m, idx, fabs(wi), i);
      }
    }
    return cta_max(m, idx, sv, si);
  }
  for (int i = k + gw; i < F.n; i += nw) {
    const double* li = F.l + static_cast<int64_t>(i) * F.ldl;
    // 16-byte loads, four in flight per lane (the rows are latency-bound
    // otherwise: one dependent load per 32 lanes per iteration)
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int j = (k0 & ~1) + 2 * lane;  // the panel's columns (v is 0 before k0)
    for (; j + 192 + 1 < k; j += 256) {
      const double2 a0 = __ldcg(reinterpret_cast<const double2*>(li + j));
      const double2 a1 = __ldcg(reinterpret_cast<const double2*>(li + j + 64));
      const double2 a2 = __ldcg(reinterpret_cast<const double2*>(li + j + 128));
      const double2 a3 = __ldcg(reinterpret_cast<const double2*>(li + j + 192));
      const double2 v0 = *reinterpret_cast<const double2*>(v + j);
      const double2 v1 = *reinterpret_cast<const double2*>(v + j + 64);
      const double2 v2 = *reinterpret_cast<const double2*>(v + j + 128);
      const double2 v3 = *reinterpret_cast<const double2*>(v + j + 192);
      s0 = fma(a0.x, v0.x, fma(a0.y, v0.y, s0));
      s1 = fma(a1.x, v1.x, fma(a1.y, v1.y, s1));
      s2 = fma(a2.x, v2.x, fma(a2.y, v2.y, s2));
      s3 = fma(a3.x, v3.x, fma(a3.y, v3.y, s3));
    }
    for (; j < k; j += 64) {
      if (j + 1 < k) {
        const double2 a0 = __ldcg(reinterpret_cast<const double2*>(li + j));
        s0 = fma(a0.x, v[j], fma(a0.y, v[j + 1], s0));
      } else {
        s0 = fma(__ldcg(li + j), v[j], s0);
      }
    }
    double s = (s0 + s1) + (s2 + s3);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const double wi = __ldcg(F.a + static_cast<int64_t>(col) * F.n + i) - s;  // A symmetric: row col, coalesced
    if (lane == 0) out[i] = wi;
    if (i != skip) max_pair(m, idx, fabs(wi), i);
  }
  return cta_max(m, idx, sv, si);
}

// Look-ahead after a 1x1 pivot without interchange at k (the common case):
// in one pass over the rows i > k, write column k of L and W
// (L(i,k) = w_i / d_k, W(i,k) = w_i) and compute column k+1 of the next
// step, w'_i = A(i,k+1) - L(i,0:k) W(k+1,0:k)^T - L(i,k) W(k+1,k), with the
// new column applied as a rank-1 term from registers -- one grid barrier
// per such pivot instead of two.  v[0:k] = W(k+1, 0:k) must be staged.
__device__ double lookahead_update(const Factor& F, int k0, int k, double dk, const double* w, const double* v,
                                   double vk, double* wn, int& idx, double* sv, int* si) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gw = blockIdx.x * kWarps + warp, nw = gridDim.x * kWarps;
  double m = -1.0;
  idx = -1;
  if (k - (k0 & ~1) <= 128) {
    for (int ib = k + 1 + gw; ib < F.n; ib += kRowBatch * nw) {
      double av[kRowBatch], xv[kRowBatch], sum[kRowBatch];
#pragma unroll
      for (int r = 0; r < kRowBatch; ++r) {
        const int i = ib + r * nw;
        av[r] = i < F.n ? __ldcg(F.a + static_cast<int64_t>(k + 1) * F.n + i) : 0.0;
        xv[r] = i < F.n ? __ldcg(w + i) : 0.0;
      }
      panel_dots(F, k0, k, v, ib, nw, sum);
#pragma unroll
      for (int r = 0; r < kRowBatch; ++r) {
        const int i = ib + r * nw;
        if (i >= F.n) break;
        const double x = xv[r];
        const double lik = fabs(dk) > F.eps ? x / dk : 0.0;
        const double s = fma(lik, vk, sum[r]);  // the new column k (fixed order: after the reduction)
        const double wi = av[r] - s;
        if (lane == 0) {
          F.l[static_cast<int64_t>(i) * F.ldl + k] = lik;
          F.wd[static_cast<int64_t>(i) * F.ldl + k] = fabs(dk) > F.eps ? x : 0.0;
          wn[i] = wi;
        }
        if (i != k + 1) max_pair(m, idx, fabs(wi), i);
      }
    }
    return cta_max(m, idx, sv, si);
  }
  for (int i = k + 1 + gw; i < F.n; i += nw) {
    const double* li = F.l + static_cast<int64_t>(i) * F.ldl;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int j = (k0 & ~1) + 2 * lane;  // the panel's columns (v is 0 before k0)
    for (; j + 192 + 1 < k; j += 256) {
      const double2 a0 = __ldcg(reinterpret_cast<const double2*>(li + j));
      const double2 a1 = __ldcg(reinterpret_cast<const double2*>(li + j + 64));
      const double2 a2 = __ldcg(reinterpret_cast<const double2*>(li + j + 128));
      const double2 a3 = __ldcg(reinterpret_cast<const double2*>(li + j + 192));
      const double2 v0 = *reinterpret_cast<const double2*>(v + j);
      const double2 v1 = *reinterpret_cast<const double2*>(v + j + 64);
      const double2 v2 = *reinterpret_cast<const double2*>(v + j + 128);
      const double2 v3 = *reinterpret_cast<const double2*>(v + j + 192);
      s0 = fma(a0.x, v0.x, fma(a0.y, v0.y, s0));
      s1 = fma(a1.x, v1.x, fma(a1.y, v1.y, s1));
      s2 = fma(a2.x, v2.x, fma(a2.y, v2.y, s2));
      s3 = fma(a3.x, v3.x, fma(a3.y, v3.y, s3));
    }
    for (; j < k; j += 64) {
      if (j + 1 < k) {
        const double2 a0 = __ldcg(reinterpret_cast<const double2*>(li + j));
        s0 = fma(a0.x, v[j], fma(a0.y, v[j + 1], s0));
      } else {
        s0 = fma(__ldcg(li + j), v[j], s0);
      }
    }
    double s = (s0 + s1) + (s2 + s3);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const double x = __ldcg(w + i);
    const double lik = fabs(dk) > F.eps ? x / dk : 0.0;
    s = fma(lik, vk, s);  // the new column k (fixed order: after the reduction)
    const double wi = __ldcg(F.a + static_cast<int64_t>(k + 1) * F.n + i) - s;
    if (lane == 0) {
      F.l[static_cast<int64_t>(i) * F.ldl + k] = lik;
      F.wd[static_cast<int64_t>(i) * F.ldl + k] = fabs(dk) > F.eps ? x : 0.0;
      wn[i] = wi;
    }
    if (i != k + 1) max_pair(m, idx, fabs(wi), i);
  }
  return cta_max(m, idx, sv, si);
}

// Blocked mode: the trailing update runs on the FP64 tensor pipe
// (mma.sync m8n8k4 DMMA) over 64 x 64 tiles; a tile's L rows and W rows
// (panel columns, zero-padded to a multiple of 4) are staged row-major with
// a pitch of 4 mod 16 doubles, which makes both the coalesced staging stores
// and the fragment loads (8 rows x 4 columns per warp) bank-conflict-free.
constexpr int kTile = 64;
constexpr int kMaxGridNb = 128;  // panel width cap (a panel may end one column late, at a 2x2 pivot)

// staged columns: [k0 & ~1, k1) rounded up to 4 (a panel is at most nb + 1 wide)
__host__ __device__ constexpr int tile_pitch(int nb) { return (((nb + 2 + 3) / 4 * 4 - 4 + 15) / 16) * 16 + 4; }
// staged L / W tiles, reused for the 64 x 65 product tile of the epilogue
__host__ __device__ constexpr int trailing_smem_doubles(int nb) {
  return nb <= 0 ? 0 : (2 * kTile * tile_pitch(nb) > kTile * (kTile + 1) ? 2 * kTile * tile_pitch(nb) : kTile * (kTile + 1));
}

// 16-byte global -> shared copy through L2 only (the panel's columns were
// written by other CTAs: no L1), bypassing registers; the bytes past
// src_bytes are zero-filled
__device__ __forceinline__ void cp_async16(double* dst, const double* src, int src_bytes) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(src_bytes) : "memory");
}

// D(8x8) += A(8x4, row) B(4x8, col) on the FP64 tensor pipe
__device__ __forceinline__ void dmma884_bk(double (&d)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}

// A(i, j) -= sum_{c in [k0, k1)} L(i, c) W(j, c) for i, j in [k1, n): the
// panel's rank-(k1 - k0) update of the trailing square, so that the next
// panel's column updates span only its own columns.  64 x 64 tiles strided
// over the grid; 8 warps as 2 x 4, a warp owning 32 rows x 16 columns
// (4 x 2 DMMA tiles); the k order is fixed (deterministic).
__device__ void trailing_update(const Factor& F, int k0, int k1, double* sm) {
  const int n = F.n, w = k1 - k0, m = n - k1;
  if (m <= 0 || w <= 0) return;
  const int jb = k0 & ~1;                          // 16-byte aligned first staged column
  const int w4 = (k1 - jb + 3) & ~3, pitch = tile_pitch(F.nb);
  const int tiles = (m + kTile - 1) / kTile;
  double* const ls = sm;                  // [64][pitch]: ls[r][c] = L(i0 + r, jb + c) (0 for columns < k0)
  double* const ws = sm + kTile * pitch;  // [64][pitch]: ws[r][c] = W(j0 + r, jb + c)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wr0 = (warp >> 2) * 32, wc0 = (warp & 3) * 16;  // the warp's sub-tile
  const int fr = lane >> 2, fk = lane & 3;                    // fragment row / k of this lane
  for (int t = blockIdx.x; t < tiles * (tiles + 1) / 2; t += gridDim.x) {
    // lower tiles (ti >= tj) only; the update is mirrored, so A stays exactly symmetric
    int ti = static_cast<int>((sqrtf(8.0f * t + 1.0f) - 1.0f) * 0.5f);
    while (ti * (ti + 1) / 2 > t) --ti;
    while ((ti + 1) * (ti + 2) / 2 <= t) ++ti;
    const int tj = t - ti * (ti + 1) / 2;
    const int i0 = k1 + ti * kTile, j0 = k1 + tj * kTile;
    __syncthreads();  // the previous tile's reads (or v) are done
    // asynchronous 8-byte copies (zero-filled outside the matrix / panel):
    // every load of the tile in flight at once
    for (int e = threadIdx.x; e < kTile * (w4 / 2); e += kThreads) {
      const int r = e / (w4 / 2), c = 2 * (e - r * (w4 / 2));
      const int i = i0 + r, j = j0 + r;
      const int valid = 8 * max(0, min(2, k1 - (jb + c)));
      const int cs = valid ? c : 0;
      cp_async16(ls + r * pitch + c, F.l + static_cast<int64_t>(i < n ? i : k1) * F.ldl + jb + cs, i < n ? valid : 0);
      cp_async16(ws + r * pitch + c, F.wd + static_cast<int64_t>(j < n ? j : k1) * F.ldl + jb + cs, j < n ? valid : 0);
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    if (jb < k0) {  // odd panel start: column k0 - 1 belongs to the previous panel
      __syncthreads();
      if (threadIdx.x < kTile) ls[threadIdx.x * pitch] = 0.0;
    }
    __syncthreads();
    double acc[4][2][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    const double* la = ls + (wr0 + fr) * pitch + fk;
    const double* wb = ws + (wc0 + fr) * pitch + fk;
#pragma unroll 2
    for (int kk = 0; kk < w4; kk += 4) {
      double af[4], bf[2];
#pragma unroll
      for (int a = 0; a < 4; ++a) af[a] = la[a * 8 * pitch + kk];
#pragma unroll
      for (int b = 0; b < 2; ++b) bf[b] = wb[b * 8 * pitch + kk];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) dmma884_bk(acc[a][b], af[a], bf[b]);
    }
    // epilogue through shared memory: the tile's products land in ct
    // [64][65], then A's tile rows are read / written as whole 512-byte row
    // segments, and the mirror (upper) tile is written from ct transposed
    __syncthreads();  // every warp is done with ls / ws
    double* const ct = sm;  // [64][kTile + 1]
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int h = 0; h < 2; ++h) ct[(wr0 + a * 8 + fr) * (kTile + 1) + wc0 + b * 8 + 2 * fk + h] = acc[a][b][h];
    __syncthreads();
    constexpr int kPer = kTile * kTile / kThreads;  // 16 elements per thread
    const int cc = threadIdx.x & (kTile - 1), r0 = threadIdx.x / kTile;
    double old[kPer];
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const int i = i0 + r0 + 4 * q, j = j0 + cc;
      old[q] = (i < n && j < n && j <= i) ? __ldcg(F.a + static_cast<int64_t>(i) * n + j) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const int r = r0 + 4 * q, i = i0 + r, j = j0 + cc;
      if (i < n && j < n && j <= i) {
        const double x = old[q] - ct[r * (kTile + 1) + cc];
        F.a[static_cast<int64_t>(i) * n + j] = x;
        ct[r * (kTile + 1) + cc] = x;
      }
    }
    __syncthreads();
    // mirror: A(j, i) = A(i, j) for i > j; row j of the upper tile is column j of ct
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const int rr = r0 + 4 * q, j = j0 + rr, i = i0 + cc;
      if (i < n && j < n && i > j) F.a[static_cast<int64_t>(j) * n + i] = ct[cc * (kTile + 1) + rr];
    }
  }
}

__global__ void __launch_bounds__(kThreads, 2) bk_factor_kernel(Factor F) {
  extern __shared__ double smem[];
  // v = W(row, panel) for the column updates.  Blocked mode (F.nb > 0): only
  // the panel's columns [k0 & ~1, k) are live, so v is panel-relative (its
  // base shifted by k0 & ~1; the functions index it by absolute column) and
  // shared memory no longer grows with n -- no size limit on n.  Unblocked
  // mode: absolute, [n].
  __shared__ double sv[kWarps];
  __shared__ int si[kWarps];
  cg::grid_group grid = cg::this_grid();
  const int n = F.n;
  const int tid = blockIdx.x * kThreads + threadIdx.x, nt = gridDim.x * kThreads;

  // A := the symmetric matrix of its lower triangle (LAPACK's 'L' view; the
  // input is symmetric to 1e-12): 32 x 32 tiles below the diagonal are
  // transposed through shared memory onto their mirror.  From here on every
  // step keeps A exactly symmetric, so column reads become row reads.
  {
    double(*tile)[33] = reinterpret_cast<double(*)[33]>(smem);
    const int tb = (n + 31) / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int t = blockIdx.x; t < tb * (tb + 1) / 2; t += gridDim.x) {
      int ti = static_cast<int>((sqrtf(8.0f * t + 1.0f) - 1.0f) * 0.5f);
      while (ti * (ti + 1) / 2 > t) --ti;
      while ((ti + 1) * (ti + 2) / 2 <= t) ++ti;
      const int tj = t - ti * (ti + 1) / 2;
      __syncthreads();
      for (int r = warp; r < 32; r += kWarps) {
        const int i = ti * 32 + r, j = tj * 32 + lane;
        tile[r][lane] = (i < n && j < n) ? __ldcg(F.a + static_cast<int64_t>(i) * n + j) : 0.0;
      }
      __syncthreads();
      for (int r = warp; r < 32; r += kWarps) {
        const int j = tj * 32 + r, i = ti * 32 + lane;  // element (i, j) -> (j, i)
        if (i < n && j < n && i > j) F.a[static_cast<int64_t>(j) * n + i] = tile[lane][r];
      }
    }
    grid.sync();
  }

  int cur = 0;        // which of (w, part) / (w2, part3) holds the current column
  bool pre = false;   // column k already computed (and its maxima published) by a look-ahead
  int k0 = 0;         // first column of the current panel (blocked mode; 0 throughout otherwise)
  const long long c_start = clock64();
  // phase clocks / counts in shared memory (CTA 0, thread 0): no registers held across the kernel
  __shared__ long long s_ph[11];  // [0..4] clocks, [5..9] counts, [10] trailing updates
  if (threadIdx.x == 0)
    for (int q = 0; q < 11; ++q) s_ph[q] = 0;
  long long c_mark = c_start;
  const bool tracing = F.trace != nullptr && blockIdx.x == 0 && threadIdx.x == 0;
  auto mark = [&](int q) {
    if (!tracing) return;
    const long long t = clock64();
    s_ph[q] += t - c_mark;
    s_ph[5 + q] += 1;
    c_mark = t;
  };
  for (int k = 0; k < n;) {
    double* const v = F.nb > 0 ? smem - (k0 & ~1) : smem;
    double* const wk = cur ? F.w2 : F.w;
    double* const pk = cur ? F.part3 : F.part;
    if (!pre) {
      // ---- updated column k and its maximum below the diagonal ----
      d_times_lrow(F, k, k0, k, v);
      __syncthreads();
      int idx;
      double m = column_update(F, k, k0, k, v, wk, k, idx, sv, si);
      if (threadIdx.x == 0) {
        pk[2 * blockIdx.x] = m;
        pk[2 * blockIdx.x + 1] = idx;
      }
      grid.sync();
      mark(0);
    }
    // Speculative loads for the common outcome (a 1x1 pivot at k followed by
    // the look-ahead): W(k+1, panel) into v and w_k, w_{k+1}, in flight
    // together with the maxima (cta_max's barriers publish v)
    const bool may_look = k + 1 < n && (F.nb <= 0 || k + 1 - k0 < F.nb);
    if (may_look) d_times_lrow(F, k + 1, k0, k, v);
    const double wkk = __ldcg(wk + k);
    const double wk1 = may_look ? __ldcg(wk + k + 1) : 0.0;
    bool v_next = may_look;  // v holds W(k+1, panel)
    int r;
    const double lambda = fmax(grid_max(pk, r, sv, si), 0.0);
    const double absakk = fabs(wkk);
    int kind = 0;  // 0: 1x1 at k; 1: 1x1 at r (swap k <-> r); 2: 2x2 (k, r) (swap k+1 <-> r)
    mark(1);
    // the reference's negligible column (linalg.cpp:143-157): an exact zero
    // pivot, no interchange, a zero column of L
    const bool negl = !(fmax(absakk, lambda) > F.eps);
    if (r >= 0 && !negl && absakk < kAlpha * lambda) {
      // ---- updated column r and its off-diagonal maximum ----
      __syncthreads();  // v is reused
      v_next = false;
      d_times_lrow(F, r, k0, k, v);
      __syncthreads();
      int idx2;
      double m2 = column_update(F, r, k0, k, v, F.wr, r, idx2, sv, si);
      __syncthreads();
      if (threadIdx.x == 0) {
        F.part2[2 * blockIdx.x] = m2;
        F.part2[2 * blockIdx.x + 1] = idx2;
      }
      grid.sync();
      int r2;
      const double sigma = fmax(grid_max(F.part2, r2, sv, si), 0.0);
      if (absakk * sigma >= kAlpha * lambda * lambda)
        kind = 0;
      else if (fabs(__ldcg(F.wr + r)) >= kAlpha * sigma)
        kind = 1;
      else
        kind = 2;
      mark(2);
    }
    // (no look-ahead into the next panel: its columns need the trailing update first)
    if (kind == 0 && may_look) {
      // ---- look-ahead: column k of L / W and column k+1, one barrier ----
      const double dk = negl ? 0.0 : wkk;
      if (!v_next) {
        __syncthreads();  // v is reused
        d_times_lrow(F, k + 1, k0, k, v);
        __syncthreads();
      }
      const double vk = fabs(dk) > F.eps ? wk1 : 0.0;  // W(k+1, k)
      double* const wn = cur ? F.w : F.w2;
      double* const pn = cur ? F.part : F.part3;
      int idx;
      const double m = lookahead_update(F, k0, k, dk, wk, v, vk, wn, idx, sv, si);
      if (threadIdx.x == 0) {
        pn[2 * blockIdx.x] = m;
        pn[2 * blockIdx.x + 1] = idx;
      }
      if (tid == 0) {
        F.d[k] = dk;
        F.e[k] = 0.0;
        F.piv[k] = 1;
        F.l[static_cast<int64_t>(k) * F.ldl + k] = 1.0;
        F.wd[static_cast<int64_t>(k) * F.ldl + k] = dk;
      }
      grid.sync();
      mark(3);
      cur ^= 1;
      pre = true;
      k += 1;
      continue;
    }
    pre = false;
    // ---- symmetric interchange p <-> r of the trailing A, of L's rows so
    //      far, and of perm ----
    const int p = kind == 1 ? k : kind == 2 ? k + 1 : -1;
    if (p >= 0 && p != r) {
      for (int j = k + tid; j < n; j += nt) {
        if (j == p || j == r) continue;
        double* ap = F.a + static_cast<int64_t>(p) * n;
        double* ar = F.a + static_cast<int64_t>(r) * n;
        // (L2 loads: other CTAs' trailing updates wrote A, L1 may be stale)
        const double x = __ldcg(ap + j), y = __ldcg(ar + j);
        ap[j] = y;
        ar[j] = x;
        double* aj = F.a + static_cast<int64_t>(j) * n;
        const double u = __ldcg(aj + p), q = __ldcg(aj + r);
        aj[p] = q;
        aj[r] = u;
      }
      for (int j = tid; j < k; j += nt) {
        double* lp = F.l + static_cast<int64_t>(p) * F.ldl;
        double* lr = F.l + static_cast<int64_t>(r) * F.ldl;
        double* wp = F.wd + static_cast<int64_t>(p) * F.ldl;
        double* wq = F.wd + static_cast<int64_t>(r) * F.ldl;
        const double l0 = __ldcg(lp + j), l1 = __ldcg(lr + j), w0 = __ldcg(wp + j), w1 = __ldcg(wq + j);
        lp[j] = l1;
        lr[j] = l0;
        wp[j] = w1;
        wq[j] = w0;
      }
      if (tid == 0) {
        const double t = __ldcg(F.a + static_cast<int64_t>(p) * n + p);
        F.a[static_cast<int64_t>(p) * n + p] = __ldcg(F.a + static_cast<int64_t>(r) * n + r);
        F.a[static_cast<int64_t>(r) * n + r] = t;
        const int pt = F.perm[p];
        F.perm[p] = F.perm[r];
        F.perm[r] = pt;
      }
    }
    // ---- D block and the new column(s) of L (rows below the block) ----
    // sigma_swap(i): index of row i before the interchange p <-> r
    auto src = [&](int i) { return (p >= 0 && p != r) ? (i == p ? r : (i == r ? p : i)) : i; };
    if (kind == 0) {
      const double dk = negl ? 0.0 : __ldcg(wk + k);
      if (tid == 0) {
        F.d[k] = dk;
        F.e[k] = 0.0;
        F.piv[k] = 1;
        F.l[static_cast<int64_t>(k) * F.ldl + k] = 1.0;
      }
      for (int i = k + 1 + tid; i < n; i += nt) {
        const double x = __ldcg(wk + i);
        F.l[static_cast<int64_t>(i) * F.ldl + k] = fabs(dk) > F.eps ? x / dk : 0.0;
        F.wd[static_cast<int64_t>(i) * F.ldl + k] = fabs(dk) > F.eps ? x : 0.0;
      }
    } else if (kind == 1) {
      const double dk = __ldcg(F.wr + r);
      if (tid == 0) {
        F.d[k] = dk;
        F.e[k] = 0.0;
        F.piv[k] = 1;
        F.l[static_cast<int64_t>(k) * F.ldl + k] = 1.0;
      }
      for (int i = k + 1 + tid; i < n; i += nt) {
        const double x = __ldcg(F.wr + src(i));
        F.l[static_cast<int64_t>(i) * F.ldl + k] = fabs(dk) > F.eps ? x / dk : 0.0;
        F.wd[static_cast<int64_t>(i) * F.ldl + k] = fabs(dk) > F.eps ? x : 0.0;
      }
    } else {
      const double a = __ldcg(wk + k), b = __ldcg(wk + r), c = __ldcg(F.wr + r);
      const double det = a * c - b * b;
      if (tid == 0) {
        F.d[k] = a;
        F.d[k + 1] = c;
        F.e[k] = b;
        F.e[k + 1] = 0.0;
        F.piv[k] = 2;
        F.piv[k + 1] = -2;
        F.l[static_cast<int64_t>(k) * F.ldl + k] = 1.0;
        F.l[static_cast<int64_t>(k + 1) * F.ldl + k] = 0.0;
        F.l[static_cast<int64_t>(k + 1) * F.ldl + k + 1] = 1.0;
        F.wd[static_cast<int64_t>(k + 1) * F.ldl + k] = b;  // (L D)(k+1, k) = 0 a + 1 b
      }
      for (int i = k + 2 + tid; i < n; i += nt) {
        const int s = src(i);
        const double x0 = __ldcg(wk + s), x1 = __ldcg(F.wr + s);
        // [L(i,k) L(i,k+1)] = [x0 x1] D^{-1},  D^{-1} = [[c, -b], [-b, a]] / det
        F.l[static_cast<int64_t>(i) * F.ldl + k] = (x0 * c - x1 * b) / det;
        F.l[static_cast<int64_t>(i) * F.ldl + k + 1] = (x1 * a - x0 * b) / det;
        F.wd[static_cast<int64_t>(i) * F.ldl + k] = x0;
        F.wd[static_cast<int64_t>(i) * F.ldl + k + 1] = x1;
      }
    }
    grid.sync();
    mark(4);
    k += kind == 2 ? 2 : 1;
    if (F.nb > 0 && k - k0 >= F.nb && k < n) {
      // ---- panel end: rank-(k - k0) update of the trailing square ----
      const long long c0 = clock64();
      trailing_update(F, k0, k, smem);
      grid.sync();
      if (tracing) {
        s_ph[10] += clock64() - c0;
        c_mark = clock64();
      }
      k0 = k;
    }
  }
  if (F.trace && blockIdx.x == 0 && threadIdx.x == 0) {
    F.trace[0] = s_ph[10];
    F.trace[1] = clock64() - c_start;
    for (int q = 0; q < 5; ++q) {
      F.trace[2 + q] = s_ph[q];
      F.trace[7 + q] = s_ph[5 + q];
    }
  }
}

// x = P^T L^-T D^-1 L^-1 P b: one cooperative launch.  The substitutions
// walk 32-row blocks; each block's update from the rows already solved is
// spread over every warp of the grid (fixed-order partial sums), then CTA 0
// reduces the partials and one warp solves the 32 x 32 triangle from shared
// memory (the diagonal tile is staged before the barrier, so its loads
// overlap the partial sums); two grid barriers per block.
//   forward  (row rr of the block, lanes along columns j < b0):
//            tasks (rr, slice), part[rr * kSlices + slice]
//   backward (column c = lane of the block, warps along rows j >= b1):
//            per-CTA sums, part[cta * 32 + c]
constexpr int kSlices = 64;  // warp slices per row of a forward block update

__device__ __forceinline__ void stage_diag_tile(const double* __restrict__ l, int ldl, int b0, int rows, int lane,
                                                double (*tile)[33]) {
#pragma unroll 8
  for (int r = 0; r < 32; ++r)
    tile[r][lane] = (r < rows && lane < rows) ? __ldcg(l + static_cast<int64_t>(b0 + r) * ldl + b0 + lane) : 0.0;
}

__global__ void __launch_bounds__(kThreads) bk_solve_kernel(const double* __restrict__ l, int ldl,
                                                            const double* __restrict__ d, const double* __restrict__ e,
                                                            const int* __restrict__ piv, const int* __restrict__ perm,
                                                            int n, const double* b, double* z, double* x,
                                                            double* part /* >= max(32 kSlices, 32 grid) */) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double tile[32][33];
  __shared__ double red[kWarps][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gw = blockIdx.x * kWarps + warp, nw = gridDim.x * kWarps;
  const int tid = blockIdx.x * kThreads + threadIdx.x, nt = gridDim.x * kThreads;
  const bool lead = blockIdx.x == 0;
  // z = P b
  for (int i = tid; i < n; i += nt) z[i] = b[perm[i]];
  grid.sync();
  // ---- forward: L z = P b (unit lower) ----
  for (int b0 = 0; b0 < n; b0 += 32) {
    const int rows = min(32, n - b0);
    if (lead && warp == 0) stage_diag_tile(l, ldl, b0, rows, lane, tile);
    // task (rr, sl): row b0 + rr, columns j = sl * 32 + lane + 32 * kSlices * t < b0
    for (int task = gw; task < 32 * kSlices; task += nw) {
      const int rr = task / kSlices, sl = task % kSlices;
      double s0 = 0.0, s1 = 0.0;
      if (rr < rows) {
        const double* li = l + static_cast<int64_t>(b0 + rr) * ldl;
        int j = sl * 32 + lane;
        for (; j + 32 * kSlices < b0; j += 64 * kSlices) {
          s0 = fma(__ldcg(li + j), __ldcg(z + j), s0);
          s1 = fma(__ldcg(li + j + 32 * kSlices), __ldcg(z + j + 32 * kSlices), s1);
        }
        if (j < b0) s0 = fma(__ldcg(li + j), __ldcg(z + j), s0);
      }
      double s = s0 + s1;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) part[task] = s;
    }
    grid.sync();
    if (lead) {
      // warp w sums slices [8w, 8w + 8) of row `lane`; warp 0 the warps (fixed order)
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < kSlices / kWarps; ++q) s += __ldcg(part + lane * kSlices + warp * (kSlices / kWarps) + q);
      red[warp][lane] = s;
      __syncthreads();
      if (warp == 0) {
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) t += red[w][lane];
        double zi = lane < rows ? __ldcg(z + b0 + lane) - t : 0.0;
        for (int j = 0; j < rows; ++j) {
          const double zj = __shfl_sync(0xffffffffu, zi, j);
          if (lane > j) zi -= tile[lane][j] * zj;
        }
        if (lane < rows) z[b0 + lane] = zi;
      }
    }
    grid.sync();
  }
  // ---- D ----
  for (int i = tid; i < n; i += nt) {
    if (piv[i] == 1) {
      x[i] = __ldcg(z + i) / d[i];
    } else {
      const bool first = piv[i] == 2;
      const int k = first ? i : i - 1;  // block (k, k+1)
      const double a = d[k], bb = e[k], c = d[k + 1];
      const double det = a * c - bb * bb;
      const double z0 = __ldcg(z + k), z1 = __ldcg(z + k + 1);
      x[i] = first ? (c * z0 - bb * z1) / det : (a * z1 - bb * z0) / det;
    }
  }
  grid.sync();
  // ---- backward: L^T y = x ----
  const int nblk = (n + 31) / 32;
  for (int bi = nblk - 1; bi >= 0; --bi) {
    const int b0 = bi * 32, b1 = min(n, b0 + 32), rows = b1 - b0;
    if (lead && warp == 0) stage_diag_tile(l, ldl, b0, rows, lane, tile);
    // column b0 + lane of L over rows j >= b1, rows strided over the grid's warps
    double s0 = 0.0, s1 = 0.0;
    if (lane < rows) {
      int j = b1 + gw;
      for (; j + nw < n; j += 2 * nw) {
        s0 = fma(__ldcg(l + static_cast<int64_t>(j) * ldl + b0 + lane), __ldcg(x + j), s0);
        s1 = fma(__ldcg(l + static_cast<int64_t>(j + nw) * ldl + b0 + lane), __ldcg(x + j + nw), s1);
      }
      if (j < n) s0 = fma(__ldcg(l + static_cast<int64_t>(j) * ldl + b0 + lane), __ldcg(x + j), s0);
    }
    red[warp][lane] = s0 + s1;
    __syncthreads();
    if (warp == 0) {
      double t = 0.0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) t += red[w][lane];
      part[blockIdx.x * 32 + lane] = t;
    }
    grid.sync();
    if (lead) {
      const int g = gridDim.x;
      double s = 0.0;
      for (int q = warp; q < g; q += kWarps) s += __ldcg(part + q * 32 + lane);
      red[warp][lane] = s;
      __syncthreads();
      if (warp == 0) {
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) t += red[w][lane];
        double yi = lane < rows ? __ldcg(x + b0 + lane) - t : 0.0;
        for (int j = rows - 1; j >= 0; --j) {
          const double yj = __shfl_sync(0xffffffffu, yi, j);
          if (lane < j) yi -= tile[j][lane] * yj;
        }
        if (lane < rows) x[b0 + lane] = yi;
      }
    }
    grid.sync();
  }
  // ---- x_orig[perm[i]] = y_i (through z) ----
  for (int i = tid; i < n; i += nt) z[perm[i]] = __ldcg(x + i);
  grid.sync();
  for (int i = tid; i < n; i += nt) x[i] = __ldcg(z + i);
}

// The same substitutions in ONE CTA of kCtaThreads threads (small and
// medium n): the grid version pays two grid barriers per 32-row block,
// here a block costs two CTA barriers; L (n^2 / 2 words per direction) is
// streamed from L2 by one SM.  Per block: the 32 x b0 (forward) or
// (n - b1) x 32 (backward) update with coalesced row segments -- forward:
// warp w takes row b0 + w, lanes along j; backward: warps take rows j,
// lanes the block's 32 columns, partial sums reduced through shared memory
// in a fixed order -- then warp 0 solves the 32 x 32 triangle from a tile
// staged in shared memory.
constexpr int kCtaThreads = 1024;
constexpr int kCtaWarps = kCtaThreads / 32;

__global__ void __launch_bounds__(kCtaThreads) bk_solve_cta_kernel(const double* __restrict__ l, int ldl,
                                                                   const double* __restrict__ d,
                                                                   const double* __restrict__ e,
                                                                   const int* __restrict__ piv,
                                                                   const int* __restrict__ perm, int n,
                                                                   const double* b, double* z, double* x) {
  __shared__ double tile[32][33];
  __shared__ double red[kCtaWarps][33];
  __shared__ double sblk[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < n; i += kCtaThreads) z[i] = b[perm[i]];
  __syncthreads();
  // ---- forward: L z = P b ----
  for (int b0 = 0; b0 < n; b0 += 32) {
    const int rows = min(32, n - b0);
    // warp w: row b0 + w, sum over j < b0; also stage the diagonal tile row
    if (warp < rows) {
      const double* li = l + static_cast<int64_t>(b0 + warp) * ldl;
      double s0 = 0.0, s1 = 0.0;
      int j = lane;
      for (; j + 32 < b0; j += 64) {
        s0 = fma(__ldcg(li + j), z[j], s0);
        s1 = fma(__ldcg(li + j + 32), z[j + 32], s1);
      }
      if (j < b0) s0 = fma(__ldcg(li + j), z[j], s0);
      double s = s0 + s1;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      tile[warp][lane] = lane < rows ? __ldcg(li + b0 + lane) : 0.0;
      if (lane == 0) sblk[warp] = s;
    }
    __syncthreads();
    if (warp == 0) {
      double zi = lane < rows ? z[b0 + lane] - sblk[lane] : 0.0;
      for (int j = 0; j < rows; ++j) {
        const double zj = __shfl_sync(0xffffffffu, zi, j);
        if (lane > j) zi -= tile[lane][j] * zj;
      }
      if (lane < rows) z[b0 + lane] = zi;
    }
    __syncthreads();
  }
  // ---- D ----
  for (int i = threadIdx.x; i < n; i += kCtaThreads) {
    if (piv[i] == 1) {
      x[i] = z[i] / d[i];
    } else {
      const bool first = piv[i] == 2;
      const int k = first ? i : i - 1;
      const double a = d[k], bb = e[k], c = d[k + 1];
      const double det = a * c - bb * bb;
      const double z0 = z[k], z1 = z[k + 1];
      x[i] = first ? (c * z0 - bb * z1) / det : (a * z1 - bb * z0) / det;
    }
  }
  __syncthreads();
  // ---- backward: L^T y = x ----
  for (int b0 = ((n - 1) / 32) * 32; b0 >= 0; b0 -= 32) {
    const int b1 = min(n, b0 + 32), rows = b1 - b0;
    double s0 = 0.0, s1 = 0.0;
    if (lane < rows) {
      int j = b1 + warp;
      for (; j + kCtaWarps < n; j += 2 * kCtaWarps) {
        s0 = fma(__ldcg(l + static_cast<int64_t>(j) * ldl + b0 + lane), x[j], s0);
        s1 = fma(__ldcg(l + static_cast<int64_t>(j + kCtaWarps) * ldl + b0 + lane), x[j + kCtaWarps], s1);
      }
      if (j < n) s0 = fma(__ldcg(l + static_cast<int64_t>(j) * ldl + b0 + lane), x[j], s0);
    }
    red[warp][lane] = s0 + s1;
    if (warp < rows) tile[warp][lane] = lane < rows ? __ldcg(l + static_cast<int64_t>(b0 + warp) * ldl + b0 + lane) : 0.0;
    __syncthreads();
    if (warp == 0) {
      double t = 0.0;
      for (int w = 0; w < kCtaWarps; ++w) t += red[w][lane];  // fixed order
      double yi = lane < rows ? x[b0 + lane] - t : 0.0;
      for (int j = rows - 1; j >= 0; --j) {
        const double yj = __shfl_sync(0xffffffffu, yi, j);
        if (lane < j) yi -= tile[j][lane] * yj;
      }
      if (lane < rows) x[b0 + lane] = yi;
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < n; i += kCtaThreads) z[perm[i]] = x[i];
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += kCtaThreads) x[i] = z[i];
}

}  // namespace bk
}  // namespace gbb
