// Blocked Bunch-Kaufman LDL^T for the KKT sizes of the reduced-space IPM
// (n up to 2048).  Same contract and output format as
// ldlt_bk.cuh (P A P^T = L D L^T, (P b)_i = b[perm[i]], piv 1 / 2 / -2) and the
// reference's pivot rule (proj/src/linalg.cpp:101-287: LAPACK dsytrf / dlasyf
// lower, alpha = (1 + sqrt 17) / 8, ties to the smaller index).
//
// One cooperative launch, one CTA per SM.  Panels of nb <= 32 columns:
//   * CTA 0 factors the panel alone, the way dlasyf does: column k of the
//     trailing matrix is row loc[k] of A (kept full and symmetric in
//     HBM/L2, current through the previous panel) minus the panel's own
//     contribution  sum_c W(:, c) (D^{-1} W(k, :))_c,  W = L D -- the updated
//     pivot columns -- held in shared memory.  A pivot step costs CTA
//     barriers, not grid barriers, and the next pivot row is prefetched from
//     L2 while the current column is reduced and pivoted;
//   * then every CTA applies the panel's rank-nb update A -= W D^{-1} W^T to
//     its trailing rows (two grid barriers per panel, not per pivot).
// Symmetric interchanges move no data: physical row P keeps original row
// P; loc / inv map logical (pivot-order) indices to physical rows and back.
// Retired physical rows are never read again, so the trailing update runs
// blind over the square [qmin, n)^2 of physical indices.  L = W D^{-1} is
// stored by logical column (lcols[k][P], coalesced) and gathered into
// logical rows at the end.
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace gbb {
namespace bkp {

namespace cg = cooperative_groups;

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxRowsPerThread = 4;  // n <= 2048 (logical indices fit the 12-bit key field)
constexpr int kMaxNb = 32;
constexpr int kUpdRows = 16;  // trailing rows per CTA pass
constexpr double kAlpha = 0.64038820320220756872;  // (1 + sqrt(17)) / 8

struct Params {
  double* a;      // [n][n] full symmetric (equilibrated) matrix; trailing part updated in place
  double* lcols;  // [n][n] L by logical column, physical row (scratch)
  double* l;      // [n][ldl] output: unit lower L, logical order (strict lower part)
  int ldl;
  double* d;      // [n]
  double* e;      // [n]
  int* piv;       // [n]
  int* perm;      // [n]
  double* pan_w;  // [kMaxNb][n]: the panel's W columns (physical rows)
  double* pan_g;  // [kMaxNb][3]: the panel's D^{-1} coefficients g0, g1, partner
  int* ctl;       // [4]: qmin, panel width
  int n;
  int nb;
  double eps;  // zero-pivot threshold 1e-11 max|SAS| (linalg.cpp:101, 143-157, 226-229)
  long long* trace;  // diagnostics (GBOPT_LDLT_TIMING): CTA 0's clocks per phase [8], or null
};

// shared-memory bytes for (n, nb)
__host__ __device__ inline int64_t smem_bytes(int n, int nb) {
  const int64_t wp = 8 * static_cast<int64_t>(nb + 1) * n;                      // W panel + column-r scratch
  const int64_t upd = 8 * (static_cast<int64_t>(nb) * n + kUpdRows * kMaxNb);  // trailing update staging
  return (wp > upd ? wp : upd) + 9 * static_cast<int64_t>(n) + 64;
}

__device__ __forceinline__ void max_pair(double& v, int& i, double v2, int i2) {
  if (i2 >= 0 && (i < 0 || v2 > v || (v2 == v && i2 < i))) {
    v = v2;
    i = i2;
  }
}

// CTA-wide (value, index) maximum, in every thread (two barriers)
__device__ void cta_max(double& v, int& i, double* rv, int* ri) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
    const int i2 = __shfl_xor_sync(0xffffffffu, i, o);
    max_pair(v, i, v2, i2);
  }
  if (lane == 0) {
    rv[warp] = v;
    ri[warp] = i;
  }
  __syncthreads();
  v = lane < kWarps ? rv[lane] : -1.0;
  i = lane < kWarps ? ri[lane] : -1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
    const int i2 = __shfl_xor_sync(0xffffffffu, i, o);
    max_pair(v, i, v2, i2);
  }
  __syncthreads();  // rv / ri reusable
}

struct Panel {
  double* W;   // [nb + 1][n]: W columns, row nb = column-r scratch
  double* zs;  // [kMaxNb]: (D^{-1} W(q, :)) of the current row q
  double* g0;  // [kMaxNb] D^{-1} coefficient on the own column
  double* g1;  // [kMaxNb] on the partner column (2x2 blocks)
  int* pp;     // [kMaxNb] partner column (own index for 1x1)
  int* loc;
  int* inv;
  unsigned char* active;
};

__device__ __forceinline__ void load_row(const Params& p, int n, int q, double* row) {
#pragma unroll
  for (int t = 0; t < kMaxRowsPerThread; ++t) {
    const int P = threadIdx.x + t * kThreads;
    row[t] = P < n ? __ldcg(p.a + static_cast<int64_t>(q) * n + P) : 0.0;
  }
}

// The trailing-matrix column at physical row q with the panel's first jj
// columns applied, into out[P] for active P, and its off-diagonal maximum
// (|value|, logical index).  `arow` holds A[q][P] for the thread's rows;
// when qn >= 0 the thread's entries of row qn (the likely next pivot row)
// are loaded into `next` before the reduction.
__device__ double panel_column(const Params& p, const Panel& s, int n, int q, int jj, const double* arow, int qn,
                               double* next, double* out, double* rv, int* ri, int& idx) {
  if (static_cast<int>(threadIdx.x) < jj) {
    const int c = threadIdx.x;
    s.zs[c] = s.g0[c] * s.W[c * n + q] + s.g1[c] * s.W[s.pp[c] * n + q];
  }
  __syncthreads();
  if (qn >= 0) load_row(p, n, qn, next);
  // off-diagonal argmax as ONE 64-bit key per candidate: |v| with its low 12
  // mantissa bits replaced by (4095 - logical index), so an integer max picks
  // the largest |v| (to 2^-40 relative) and, among ties, the smallest index;
  // key 0 = no candidate.  (A (double, index) pair reduction costs ~3x more
  // in dependent shuffle/compare rounds: tools/panel_gemv_probe.cu.)
  unsigned long long key = 0;
#pragma unroll
  for (int t = 0; t < kMaxRowsPerThread; ++t) {
    const int P = threadIdx.x + t * kThreads;
    if (P >= n || !s.active[P]) continue;
    double s0 = 0.0, s1 = 0.0;
    int c = 0;
    for (; c + 1 < jj; c += 2) {
      s0 = fma(s.W[c * n + P], s.zs[c], s0);
      s1 = fma(s.W[(c + 1) * n + P], s.zs[c + 1], s1);
    }
    if (c < jj) s0 = fma(s.W[c * n + P], s.zs[c], s0);
    const double v = arow[t] - (s0 + s1);
    out[P] = v;
    if (P != q) {
      const unsigned long long k2 = (static_cast<unsigned long long>(__double_as_longlong(fabs(v))) & ~0xFFFull) |
                                    static_cast<unsigned long long>(0xFFF - s.inv[P]);
      key = k2 > key ? k2 : key;
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long k2 = __shfl_xor_sync(0xffffffffu, key, o);
    key = k2 > key ? k2 : key;
  }
  unsigned long long* kw = reinterpret_cast<unsigned long long*>(rv);  // kWarps slots
  if (lane == 0) kw[warp] = key;
  __syncthreads();
  unsigned long long best = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) best = kw[w] > best ? kw[w] : best;
  __syncthreads();  // kw reusable
  if (best == 0) {
    idx = -1;
    return -1.0;
  }
  idx = 0xFFF - static_cast<int>(best & 0xFFF);
  return fabs(out[s.loc[idx]]);  // the exact value of the winner
}

__global__ void __launch_bounds__(kThreads, 1) bkp_factor_kernel(Params p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ double rv[kWarps];
  __shared__ int ri[kWarps];
  __shared__ double zs[kMaxNb], g0[kMaxNb], g1[kMaxNb];
  __shared__ int pp[kMaxNb];
  __shared__ int s_qmin;
  cg::grid_group grid = cg::this_grid();
  const int n = p.n, nb = p.nb;
  const bool lead = blockIdx.x == 0;

  const int64_t wbytes = 8 * static_cast<int64_t>(nb + 1) * n;
  const int64_t ubytes = 8 * (static_cast<int64_t>(nb) * n + kUpdRows * kMaxNb);
  Panel s;
  s.W = reinterpret_cast<double*>(smem_raw);
  s.zs = zs;
  s.g0 = g0;
  s.g1 = g1;
  s.pp = pp;
  s.loc = reinterpret_cast<int*>(smem_raw + (wbytes > ubytes ? wbytes : ubytes));
  s.inv = s.loc + n;
  s.active = reinterpret_cast<unsigned char*>(s.inv + n);

  long long tacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long tlast = clock64();
  auto mark = [&](int i) {
    if (p.trace && lead && threadIdx.x == 0) {
      const long long t = clock64();
      tacc[i] += t - tlast;
      tlast = t;
    }
  };

  if (lead) {
    for (int i = threadIdx.x; i < n; i += kThreads) {
      s.loc[i] = i;
      s.inv[i] = i;
      s.active[i] = 1;
    }
    if (threadIdx.x == 0) s_qmin = 0;
    __syncthreads();
  }

  for (int k0 = 0; k0 < n;) {
    // ---------------- panel (CTA 0) ----------------
    if (lead) {
      int k = k0, jj = 0;
      double arow[kMaxRowsPerThread], next[kMaxRowsPerThread];
      int q_next = s.loc[k];
      load_row(p, n, q_next, next);  // A changed in the trailing update: fresh row
      while (jj < nb && k < n) {
        mark(7);
        const int q = s.loc[k];
        if (q != q_next) load_row(p, n, q, next);
#pragma unroll
        for (int t = 0; t < kMaxRowsPerThread; ++t) arow[t] = next[t];
        // likely next pivot row: logical k + 1 (unless an interchange moves it)
        const int qn = k + 1 < n && jj + 1 < nb ? s.loc[k + 1] : -1;
        q_next = qn;
        double* wk = s.W + static_cast<int64_t>(jj) * n;
        int r;
        const double lambda = fmax(panel_column(p, s, n, q, jj, arow, qn, next, wk, rv, ri, r), 0.0);
        const double absakk = fabs(wk[q]);
        mark(0);
        int kind = 0;  // 0: 1x1 at k; 1: 1x1 at r (swap k <-> r); 2: 2x2 (k, r) (swap k+1 <-> r)
        // negligible column (linalg.cpp:143-157): exact zero pivot, no interchange
        const bool negl = !(fmax(absakk, lambda) > p.eps);
        if (r >= 0 && !negl && absakk < kAlpha * lambda) {
          const int pr = s.loc[r];
          double* wr = s.W + static_cast<int64_t>(nb) * n;  // scratch row
          double rrow[kMaxRowsPerThread];
          load_row(p, n, pr, rrow);
          int r2;
          const double sigma = fmax(panel_column(p, s, n, pr, jj, rrow, -1, nullptr, wr, rv, ri, r2), 0.0);
          if (absakk * sigma >= kAlpha * lambda * lambda)
            kind = 0;
          else if (fabs(wr[pr]) >= kAlpha * sigma)
            kind = 1;
          else
            kind = 2;
          mark(1);
        }
        if (kind == 2 && jj + 1 >= nb) break;  // no room for the 2x2 block: it opens the next panel
        // interchange (logical labels only), retire the pivot rows, D^{-1}
        const int a_ = kind == 1 ? k : k + 1;
        const int p0 = kind == 1 ? s.loc[r] : s.loc[k];
        const int p1 = kind == 2 ? (a_ != r ? s.loc[r] : s.loc[k + 1]) : -1;
        __syncthreads();  // every thread has read loc and the columns
        if (threadIdx.x == 0) {
          if (kind != 0 && a_ != r) {
            const int pa = s.loc[a_], pb = s.loc[r];
            s.loc[a_] = pb;
            s.loc[r] = pa;
            s.inv[pb] = a_;
            s.inv[pa] = r;
          }
          s.active[p0] = 0;
          if (kind == 2) s.active[p1] = 0;
        }
        const double* scr = s.W + static_cast<int64_t>(nb) * n;
        if (kind == 1)  // the pivot column is column r
          for (int P = threadIdx.x; P < n; P += kThreads) wk[P] = scr[P];
        else if (kind == 2)
          for (int P = threadIdx.x; P < n; P += kThreads) wk[n + P] = scr[P];
        __syncthreads();
        if (threadIdx.x == 0) {
          if (kind != 2) {
            const double dk = negl ? 0.0 : wk[p0];
            s.g0[jj] = fabs(dk) > p.eps ? 1.0 / dk : 0.0;  // |d| <= eps: zero L column (linalg.cpp:226-229)
            s.g1[jj] = 0.0;
            s.pp[jj] = jj;
            p.d[k] = dk;
            p.e[k] = 0.0;
            p.piv[k] = 1;
          } else {
            const double a2 = wk[p0], b2 = wk[p1], c2 = wk[n + p1];
            const double det = a2 * c2 - b2 * b2;
            s.g0[jj] = c2 / det;
            s.g1[jj] = -b2 / det;
            s.pp[jj] = jj + 1;
            s.g0[jj + 1] = a2 / det;
            s.g1[jj + 1] = -b2 / det;
            s.pp[jj + 1] = jj;
            p.d[k] = a2;
            p.d[k + 1] = c2;
            p.e[k] = b2;
            p.e[k + 1] = 0.0;
            p.piv[k] = 2;
            p.piv[k + 1] = -2;
          }
        }
        __syncthreads();
        mark(2);
        const int step = kind == 2 ? 2 : 1;
        k += step;
        jj += step;
      }
      // publish the panel: W columns and D^{-1} for the trailing update,
      // L = W D^{-1} by logical column, qmin and the width
      for (int c = 0; c < jj; ++c) {
        const double gc0 = s.g0[c], gc1 = s.g1[c];
        const double* wc = s.W + static_cast<int64_t>(c) * n;
        const double* wpc = s.W + static_cast<int64_t>(s.pp[c]) * n;
        double* lc = p.lcols + static_cast<int64_t>(k0 + c) * n;
        for (int P = threadIdx.x; P < n; P += kThreads) {
          const double w = wc[P];
          __stcg(p.pan_w + static_cast<int64_t>(c) * n + P, w);
          lc[P] = gc0 * w + gc1 * wpc[P];
        }
      }
      if (static_cast<int>(threadIdx.x) < jj) {
        __stcg(p.pan_g + 3 * threadIdx.x, s.g0[threadIdx.x]);
        __stcg(p.pan_g + 3 * threadIdx.x + 1, s.g1[threadIdx.x]);
        __stcg(p.pan_g + 3 * threadIdx.x + 2, static_cast<double>(s.pp[threadIdx.x]));
      }
      if (threadIdx.x == 0) {
        int qm = s_qmin;
        while (qm < n && !s.active[qm]) ++qm;
        s_qmin = qm;
        p.ctl[0] = qm;
        p.ctl[1] = jj;
      }
      __syncthreads();
      mark(3);
    }
    grid.sync();
    mark(4);
    // ---------------- trailing update (all CTAs) ----------------
    const int qmin = __ldcg(p.ctl + 0), width = __ldcg(p.ctl + 1);
    if (qmin < n && width > 0) {
      // W columns [width][n] in shared memory (CTA 0 has them); per pass up
      // to kUpdRows rows P with their L(P, :) = (D^{-1} W(P, :)) in shared
      // memory; threads sweep Q with the A loads of the pass issued first
      double* ws = reinterpret_cast<double*>(smem_raw);
      if (!lead)
        for (int x = threadIdx.x; x < width * n; x += kThreads) ws[x] = __ldcg(p.pan_w + x);
      double* lrow = ws + static_cast<int64_t>(nb) * n;  // [kUpdRows][kMaxNb]
      __syncthreads();
      const int rows = n - qmin;
      const int per_cta = (rows + static_cast<int>(gridDim.x) - 1) / static_cast<int>(gridDim.x);
      const int r0 = qmin + static_cast<int>(blockIdx.x) * per_cta, r1 = min(n, r0 + per_cta);
      for (int pb = r0; pb < r1; pb += kUpdRows) {
        const int nr = min(kUpdRows, r1 - pb);
        for (int x = threadIdx.x; x < nr * width; x += kThreads) {
          const int rr = x / width, c = x - rr * width;
          const int P = pb + rr;
          const int pc = static_cast<int>(__ldcg(p.pan_g + 3 * c + 2));
          lrow[rr * kMaxNb + c] =
              __ldcg(p.pan_g + 3 * c) * ws[c * n + P] + __ldcg(p.pan_g + 3 * c + 1) * ws[pc * n + P];
        }
        __syncthreads();
        for (int Q = qmin + threadIdx.x; Q < n; Q += kThreads) {
          double v[kUpdRows];
#pragma unroll
          for (int rr = 0; rr < kUpdRows; ++rr)
            v[rr] = rr < nr ? __ldcg(p.a + static_cast<int64_t>(pb + rr) * n + Q) : 0.0;
          for (int c = 0; c < width; ++c) {
            const double wq = ws[c * n + Q];
#pragma unroll
            for (int rr = 0; rr < kUpdRows; ++rr) v[rr] = fma(-lrow[rr * kMaxNb + c], wq, v[rr]);
          }
#pragma unroll
          for (int rr = 0; rr < kUpdRows; ++rr)
            if (rr < nr) __stcg(p.a + static_cast<int64_t>(pb + rr) * n + Q, v[rr]);
        }
        __syncthreads();
      }
    }
    mark(5);
    k0 += width;
    grid.sync();
    mark(6);
  }
  if (p.trace && lead && threadIdx.x == 0)
    for (int i = 0; i < 8; ++i) p.trace[i] = tacc[i];

  // ---------------- outputs: perm, L in logical order ----------------
  if (lead)
    for (int i = threadIdx.x; i < n; i += kThreads) p.perm[i] = s.loc[i];
  grid.sync();
  // L(i, c) = lcols[c][loc[i]] for c < i
  for (int i = blockIdx.x; i < n; i += gridDim.x) {
    const int P = __ldcg(p.perm + i);
    double* dst = p.l + static_cast<int64_t>(i) * p.ldl;
    for (int c = threadIdx.x; c < i; c += kThreads) dst[c] = __ldcg(p.lcols + static_cast<int64_t>(c) * n + P);
  }
}

}  // namespace bkp
}  // namespace gbb

