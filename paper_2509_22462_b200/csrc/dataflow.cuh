// Persistent dataflow kernel: one launch evaluates the forward chain, the
// adjoint chain, the tangent GEMM chain and the Hessian SYRKs of a small
// batch (reference src/nn.cpp:113-292: forward, lagrangian_gradient's
// adjoint, and lagrangian_hessian's tangents + curvature).
//
// Why: launched layer by layer, every tangent GEMM ends in a partial wave
// (c2: 280 tiles on 148 SMs; c5: 896 tiles = 6.05 waves) and every layer
// boundary is a grid-wide barrier.  But the rows of T_l are independent
// tangent directions: row block tm of T_{l+1} needs only row block tm of
// T_l (and sigma'_l), so the layer barrier is artificial.  Here every unit
// of work is an "item" -- one 112 x 128 NT tile over a k-range -- and items
// wait only on the counters of the items they really depend on:
//
//   FWD  z_l = W_l y_{l-1} + b_l (+ sigma, sigma', sigma''; the top layer also
//        seeds gz = lambda .* sigma', d = lambda .* sigma'')   A = Y_{l-1}, B = W_l
//   ADJ  ybar_{l-1} = W_l^T gz_l, gz_{l-1}, d_{l-1}              A = GZ_l,   B = W_l^T
//   GEMM T_{l+1}[tm] = T_l[tm] diag(sigma'_l) W_{l+1}^T          A = T_l,    B = W_{l+1}
//   SYRK H_q += T_l[tm] diag(d_l) T_l[tn]^T over k-piece q       A = B = T_l
//
// The host orders the item list by a list-scheduling simulation (priority =
// longest path to the end), so the list is topological; CTAs claim items in
// list order with one atomicAdd.  A CTA only waits on items claimed before
// its own, by CTAs that are already running, so the kernel cannot deadlock
// whatever the residency.  The producer warp claims the next item when it
// has issued the last TMA load of the current one, waits for that item's
// counters (ld.acquire.gpu), and streams its k-blocks while the consumers
// are still finishing the current tile: tile prologue / epilogue overlap.
//
// Determinism: every item has a fixed k-range and a fixed output; SYRK
// pieces q accumulate into H slot q in layer order (the slot counter orders
// them), and the slots are summed in a fixed order by the symmetrise pass.
#pragma once

#include "kernels.cuh"

namespace gbb {
namespace dev {

enum DfKind : int { kDfFwd = 0, kDfAdj = 1, kDfGemm = 2, kDfSyrk = 3 };

// Stage of the dataflow ring: A box (14 KB) | B box (16 KB) | the item's
// per-k scale for the stage's 16 k (128 B, bulk-copied with the boxes, so the
// consumers hold no scale registers and issue no global loads), padded so
// every stage starts 1024-byte aligned (128B swizzle).
constexpr int kDfScaleOff = kABytes + kBBytes;
constexpr int kDfStageBytes = (kDfScaleOff + kBK * 8 + 1023) / 1024 * 1024;  // 31744
constexpr int kDfSmemBytes = kStages * kDfStageBytes + 1024 /*align slack*/ + 256 /*barriers*/;

// 1-D bulk copy global -> shared, completion counted in bytes on `bar`.
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
constexpr int kDfMaxWait = 5;

struct alignas(16) DfJob {
  int ta, tb;             // A / B operand: indices into DfParams::maps
                          // (A rows: points for FWD/ADJ, tangent rows else)
  const double* scale;    // per-k scale on B (GEMM: sigma'_l, SYRK: d_l), nullable
  int64_t s_stride;
  int64_t a_point_rows, b_point_rows;
  int kind, act;
  int a_bytes;  // bytes of one A box (FWD / ADJ: a box of round_up(points, 8) rows)
  int b_bytes;  // bytes of one B box (kBN rows; square SYRK tiles: kBM rows)
  int b_tile;   // C columns per tile = B row offset per tn (kBN, or kBM for square SYRK tiles)
  int m_valid;  // FWD/ADJ: points; GEMM: n_pad; SYRK: n
  int n_valid;  // valid output columns
  // GEMM: T_{l+1}; SYRK: H slot 0 (slots slot_stride apart)
  double* c;
  int64_t c_point_stride, ldc, slot_stride;
  // FWD: bias, z, y, s1, s2 (pitch ld); top layer: gz/d seeds from lambda
  const double* bias;
  double *z, *y, *s1, *s2;
  int64_t ld;
  const double* lam;
  int64_t ld_lam;
  double *gz_seed, *d_seed;
  // ADJ: ybar, gz, d of layer l-1 and its sigma', sigma'' (pitch ld)
  double *ybar, *gz, *d;
  const double *s1i, *s2i;
  // GEMM: also S_{l+1} = T_{l+1} diag(sigma'_{l+1}) (same layout as c), nullable
  double* c2;
  const double* c2_scale;
  int64_t c2_scale_stride;
};

struct DfItem {
  int job, point, tm, tn, kb0, kb1, slot, sig, nwait, pad;
  int widx[kDfMaxWait], wtgt[kDfMaxWait];
};

// TMA descriptors travel in the kernel parameters (param space, like the
// __grid_constant__ maps of nt_mma_kernel): 192 x 128 B = 24 KB of the 32 KB
// parameter limit.
constexpr int kDfMaxMaps = 192;

struct DfParams {
  CUtensorMap maps[kDfMaxMaps];
  const DfItem* items;
  int n_items;
  const DfJob* jobs;
  int* counters;  // zeroed before the launch; counters[0] is the claim counter
  // optional per-item trace [n_items][4] (globaltimer ns): claimed, dependencies
  // met, consumers start, epilogue done; and trace_sm[n_items] = SM id
  unsigned long long* trace;
  int* trace_sm;
};

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ int sm_id() {
  int r;
  asm volatile("mov.u32 %0, %smid;" : "=r"(r));
  return r;
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// The consumer k-loop over [kb0, kb1).  Full tiles (tangent GEMM): the
// 2 x 4 warp grid of nt_mma_kernel, 7 x 4 DMMA blocks per warp.  Square
// SYRK tiles (112 x 112): SM sub-partition q = warp & 3 owns the 56 x 56
// quadrant q, split between its two warps as 25 + 24 of its 7 x 7 blocks
// (blk_live: both warps keep the pipe busy to the end of each k-step, and
// no warp holds more than 28 accumulator blocks).  Point-row
// tiles (FWD / ADJ, M = points <= 56): every warp takes 16 of the 128
// columns and the MI live 8-row blocks, so no DMMA is issued for empty rows
// (a predicated-off DMMA still occupies the tensor pipe).  The per-k scale
// arrives in the stage (bulk copy by the producer).
constexpr int kAcc = kMI * kNJ;  // 28 DMMA accumulator blocks per warp, in every layout

template <int MI, int NJ, int SET = kBlkAll, bool SCALED = false>
__device__ __forceinline__ void df_mainloop(double (&acc)[kAcc][2], const char* smem, uint64_t* full,
                                            uint64_t* empty, uint32_t& gk, int kb0, int kb1,
                                            int ra, int rb, int t, int lane, int b_off = kABytes) {
  for (int kb = kb0; kb < kb1; ++kb, ++gk) {
    const int s = static_cast<int>(gk % kStages);
    mbar_wait(&full[s], (gk / kStages) & 1);
    const char* sa = smem + s * kDfStageBytes;
    const char* sb = sa + b_off;
    const double* ss = reinterpret_cast<const double*>(sa + kDfScaleOff);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int k = 4 * q + t;
      // the per-k scale (if any) goes on whichever operand has fewer fragments
      constexpr bool kScaleA = SCALED && MI < NJ;
      constexpr bool kScaleB = SCALED && !(MI < NJ);
      const double sc = SCALED ? ss[k] : 1.0;
      double a[MI], b[NJ];
#pragma unroll
      for (int mi = 0; mi < MI; ++mi) a[mi] = kScaleA ? lds_swz(sa, ra + 8 * mi, k) * sc : lds_swz(sa, ra + 8 * mi, k);
#pragma unroll
      for (int nj = 0; nj < NJ; ++nj) b[nj] = kScaleB ? lds_swz(sb, rb + 8 * nj, k) * sc : lds_swz(sb, rb + 8 * nj, k);
#pragma unroll
      for (int mi = 0; mi < MI; ++mi)
#pragma unroll
        for (int nj = 0; nj < NJ; ++nj)
          if (blk_live<SET>(mi, nj)) dmma884(acc[mi * NJ + nj], a[mi], b[nj]);
    }
    stage_release(&empty[s], lane);
  }
}

// Epilogue of one warp's accumulator blocks (layout MI x NJ, the first mi_n
// block rows live): block mi * NJ + nj holds C[rbase + 8 mi][cbase + 8 nj +
// pc0 / pc1].  rmw: accumulate into C (SYRK H slots) with red.add: the slot
// counter lets one item at a time touch a (slot, point, tile), so the
// additions happen in layer order (deterministic).
template <int MI, int NJ, int SET = kBlkAll>
__device__ __forceinline__ void df_store(double (&acc)[kAcc][2], double* raw, int64_t ldr, int rbase, int cbase,
                                         int mi_n, int m_valid, int n_valid, int pc0, int pc1, bool rmw,
                                         double* raw2 = nullptr, const double* s2 = nullptr) {
#pragma unroll
  for (int mi = 0; mi < MI; ++mi) {
    const int r = rbase + 8 * mi;
    if (mi >= mi_n || r >= m_valid) continue;
#pragma unroll
    for (int nj = 0; nj < NJ; ++nj) {
      if (!blk_live<SET>(mi, nj)) continue;
      const int cb = cbase + 8 * nj;
      double* dst = raw + static_cast<int64_t>(r) * ldr + cb;
      if (rmw) {
        if (cb + pc0 < n_valid) red_add_f64(dst + pc0, acc[mi * NJ + nj][0]);
        if (cb + pc1 < n_valid) red_add_f64(dst + pc1, acc[mi * NJ + nj][1]);
      } else {
        if (cb + pc0 < n_valid) dst[pc0] = acc[mi * NJ + nj][0];
        if (cb + pc1 < n_valid) dst[pc1] = acc[mi * NJ + nj][1];
        if (raw2) {  // S_{l+1} = T_{l+1} diag(sigma'_{l+1}) beside T_{l+1}
          double* d2 = raw2 + static_cast<int64_t>(r) * ldr + cb;
          if (cb + pc0 < n_valid) d2[pc0] = acc[mi * NJ + nj][0] * __ldg(s2 + cb + pc0);
          if (cb + pc1 < n_valid) d2[pc1] = acc[mi * NJ + nj][1] * __ldg(s2 + cb + pc1);
        }
      }
    }
  }
}

__global__ void __launch_bounds__(kThreads, 1) df_kernel(const __grid_constant__ DfParams P) {
  extern __shared__ unsigned char smem_raw[];
  char* smem = reinterpret_cast<char*>(smem_raw) + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kDfStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* qfull = empty + kStages;  // item hand-off, 2 slots
  uint64_t* qempty = qfull + 2;
  int* qitem = reinterpret_cast<int*>(qempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&qfull[s], 1);
      mbar_init(&qempty[s], kConsumerWarps);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == kConsumerWarps) {
    // ===== producer: claim, wait for dependencies, stream k-blocks =====
    // (the next item is claimed right after the current one's last load:
    // claiming earlier measured slower -- c3 358 vs 353 ms)
    if (lane == 0) {
      uint32_t gk = 0;
      for (int i = 0;; ++i) {
        const int slot = i & 1;
        if (i >= 2) mbar_wait(&qempty[slot], ((i >> 1) - 1) & 1);
        const int idx = atomicAdd(P.counters, 1);
        if (idx >= P.n_items) {
          qitem[slot] = -1;
          mbar_arrive(&qfull[slot]);
          break;
        }
        const DfItem& it = P.items[idx];
        if (P.trace) {
          P.trace[4 * idx] = global_ns();
          P.trace_sm[idx] = sm_id();
        }
        for (int w = 0; w < it.nwait; ++w) {
          const int* cnt = P.counters + it.widx[w];
          const int tgt = it.wtgt[w];
          if (ld_acquire(cnt) < tgt) {
            int ns = 32;
            while (ld_acquire(cnt) < tgt) {
              __nanosleep(ns);
              ns = ns < 256 ? ns * 2 : 256;
            }
          }
        }
        fence_proxy_async_global();  // generic-proxy results -> TMA reads below
        if (P.trace) P.trace[4 * idx + 1] = global_ns();
        qitem[slot] = idx;
        mbar_arrive(&qfull[slot]);
        const DfJob& J = P.jobs[it.job];
        const int a_row0 = static_cast<int>(J.a_point_rows * it.point) + it.tm * kBM;
        const int b_row0 = static_cast<int>(J.b_point_rows * it.point) + it.tn * J.b_tile;
        // the scale vector has >= 16 * k_blocks entries (zero padded)
        const double* sp = J.scale ? J.scale + J.s_stride * it.point : nullptr;
        // diagonal square SYRK tile: B == A, one box per stage
        const bool diag = J.kind == kDfSyrk && J.b_tile == kBM && it.tm == it.tn;
        for (int kb = it.kb0; kb < it.kb1; ++kb, ++gk) {
          const int s = static_cast<int>(gk % kStages);
          if (gk >= kStages) mbar_wait(&empty[s], ((gk / kStages) - 1) & 1);
          char* sa = smem + s * kDfStageBytes;
          mbar_arrive_expect_tx(&full[s], J.a_bytes + (diag ? 0 : J.b_bytes) + (sp ? kBK * 8 : 0));
          tma_load_2d(sa, &P.maps[J.ta], &full[s], kb * kBK, a_row0);
          if (!diag) tma_load_2d(sa + kABytes, &P.maps[J.tb], &full[s], kb * kBK, b_row0);
          if (sp) bulk_load(sa + kDfScaleOff, sp + kb * kBK, kBK * 8, &full[s]);
        }
      }
      // producer tail: stay until the consumers have released the last
      // stages (no issuing warp exits with bulk copies in flight; see
      // adj_mma_kernel in kernels.cuh)
      for (uint32_t g2 = gk > kStages ? gk - kStages : 0; g2 < gk; ++g2)
        mbar_wait(&empty[g2 % kStages], (g2 / kStages) & 1);
    }
    __syncwarp();
    return;
  }

  // ===== consumers =====
  const int wm = warp >> 2, wn = warp & 3;
  const int g = lane >> 2, t = lane & 3;
  const int ra = wm * kWarpM + row_perm(g);
  const int rb = wn * kWarpN + row_perm(g);
  const int pg = row_perm(g), pc0 = row_perm(2 * t), pc1 = row_perm(2 * t + 1);
  uint32_t gk = 0;
  for (int i = 0;; ++i) {
    const int slot = i & 1;
    mbar_wait(&qfull[slot], (i >> 1) & 1);
    const int idx = qitem[slot];
    __syncwarp();
    if (lane == 0) mbar_arrive(&qempty[slot]);
    if (idx < 0) break;
    if (P.trace && threadIdx.x == 0) P.trace[4 * idx + 2] = global_ns();
    const DfItem& it = P.items[idx];
    const DfJob& J = P.jobs[it.job];
    const int kind = J.kind;
    // FWD / ADJ tiles hold only m_valid (= points) live rows: skip the
    // DMMA blocks past them (uniform per warp)
    const int m_live = kind <= kDfAdj ? J.m_valid : kBM;
    const bool scaled = J.scale != nullptr;

    double acc[kAcc][2];
#pragma unroll
    for (int a = 0; a < kAcc; ++a) acc[a][0] = acc[a][1] = 0.0;

    // warp layout of this item: rows row0 + 8 mi (+ pg), mi < mi_n; columns
    // col0 + 8 nj (+ pc), nj < nj_n; accumulator block mi * nj_n + nj
    int row0, col0, mi_n, nj_n;
    const int sq = kind == kDfSyrk && J.b_tile == kBM;
    // point-row tiles (FWD / ADJ) with few points use the column-split warp layout
    const int small = (kind <= kDfAdj && m_live <= 56) ? (m_live <= 8 ? 1 : m_live <= 16 ? 2 : m_live <= 32 ? 4 : 7) : 0;
    const bool diag = sq && it.tm == it.tn;
    if (diag) {
      row0 = 8 * diag_r0(warp);
      col0 = 0;
      mi_n = diag_r1(warp) - diag_r0(warp);
      nj_n = diag_r1(warp);
#define GBB_DF_DIAG(W)                                                                                    \
  case W:                                                                                                 \
    df_mainloop<diag_r1(W) - diag_r0(W), diag_r1(W), kBlkLower + diag_r0(W), true>(                        \
        acc, smem, full, empty, gk, it.kb0, it.kb1, 8 * diag_r0(W) + row_perm(g), row_perm(g), t, lane, 0); \
    break;
      switch (warp) {
        GBB_DF_DIAG(0)
        GBB_DF_DIAG(1)
        GBB_DF_DIAG(2)
        GBB_DF_DIAG(3)
        GBB_DF_DIAG(4)
        GBB_DF_DIAG(5)
        GBB_DF_DIAG(6)
        GBB_DF_DIAG(7)
        default: break;
      }
#undef GBB_DF_DIAG
    } else if (sq) {
      const int q = warp & 3, h = warp >> 2;
      row0 = (q >> 1) * 56 + h * 24;
      col0 = (q & 1) * 56;
      mi_n = 4;
      nj_n = 7;
      const int ra_q = row0 + row_perm(g), rb_q = col0 + row_perm(g);
      if (h == 0)
        df_mainloop<4, 7, kBlkSqLo, true>(acc, smem, full, empty, gk, it.kb0, it.kb1, ra_q, rb_q, t, lane);
      else
        df_mainloop<4, 7, kBlkSqHi, true>(acc, smem, full, empty, gk, it.kb0, it.kb1, ra_q, rb_q, t, lane);
    } else if (small == 0) {
      row0 = wm * kWarpM;
      col0 = wn * kWarpN;
      mi_n = kMI;
      nj_n = kNJ;
      if (scaled)
        df_mainloop<kMI, kNJ, kBlkAll, true>(acc, smem, full, empty, gk, it.kb0, it.kb1, ra, rb, t, lane);
      else
        df_mainloop<kMI, kNJ, kBlkAll, false>(acc, smem, full, empty, gk, it.kb0, it.kb1, ra, rb, t, lane);
    } else {
      row0 = 0;
      col0 = warp * 16;
      mi_n = small;
      nj_n = 2;
      const int ra_s = row_perm(g), rb_s = warp * 16 + row_perm(g);
      if (small == 1)
        df_mainloop<1, 2>(acc, smem, full, empty, gk, it.kb0, it.kb1, ra_s, rb_s, t, lane);
      else if (small == 2)
        df_mainloop<2, 2>(acc, smem, full, empty, gk, it.kb0, it.kb1, ra_s, rb_s, t, lane);
      else if (small == 4)
        df_mainloop<4, 2>(acc, smem, full, empty, gk, it.kb0, it.kb1, ra_s, rb_s, t, lane);
      else
        df_mainloop<7, 2>(acc, smem, full, empty, gk, it.kb0, it.kb1, ra_s, rb_s, t, lane);
    }

    // ---- epilogue: block e = mi * nj_n + nj holds C[row0+8mi+pg][col0+8nj+pc0 / pc1] ----
    // GEMM: store T; SYRK: accumulate into H slot; FWD / ADJ: raw tile into
    // z / ybar, then one elementwise pass (activation or gz / d) over it.
    double* raw = kind == kDfGemm ? J.c + J.c_point_stride * it.point
                : kind == kDfSyrk ? J.c + J.slot_stride * it.slot + J.c_point_stride * it.point
                : kind == kDfFwd  ? J.z : J.ybar;
    const int64_t ldr = kind >= kDfGemm ? J.ldc : J.ld;
    const int rbase = it.tm * kBM + row0 + pg;
    const int cbase = it.tn * J.b_tile + col0;
    const bool rmw = kind == kDfSyrk;
    if (diag) {
#define GBB_DF_DIAG_ST(W)                                                                                 \
  case W:                                                                                                 \
    df_store<diag_r1(W) - diag_r0(W), diag_r1(W), kBlkLower + diag_r0(W)>(acc, raw, ldr, rbase, cbase,      \
                                                                          mi_n, J.m_valid, J.n_valid, pc0, \
                                                                          pc1, rmw);                       \
    break;
      switch (warp) {
        GBB_DF_DIAG_ST(0)
        GBB_DF_DIAG_ST(1)
        GBB_DF_DIAG_ST(2)
        GBB_DF_DIAG_ST(3)
        GBB_DF_DIAG_ST(4)
        GBB_DF_DIAG_ST(5)
        GBB_DF_DIAG_ST(6)
        GBB_DF_DIAG_ST(7)
        default: break;
      }
#undef GBB_DF_DIAG_ST
    } else if (sq && (warp >> 2) == 0)
      df_store<4, 7, kBlkSqLo>(acc, raw, ldr, rbase, cbase, mi_n, J.m_valid, J.n_valid, pc0, pc1, rmw);
    else if (sq)
      df_store<4, 7, kBlkSqHi>(acc, raw, ldr, rbase, cbase, mi_n, J.m_valid, J.n_valid, pc0, pc1, rmw);
    else if (small == 0)
      df_store<kMI, kNJ>(acc, raw, ldr, rbase, cbase, mi_n, J.m_valid, J.n_valid, pc0, pc1, rmw,
                         J.c2 ? J.c2 + J.c_point_stride * it.point : nullptr,
                         J.c2 ? J.c2_scale + J.c2_scale_stride * it.point : nullptr);
    else
      df_store<7, 2>(acc, raw, ldr, rbase, cbase, mi_n, J.m_valid, J.n_valid, pc0, pc1, rmw);
    if (kind <= kDfAdj) {
      consumer_bar();  // the raw tile is complete (CTA-scope ordering of the stores)
      const int cols = min(kBN, J.n_valid - it.tn * kBN);
      for (int e = threadIdx.x; e < J.m_valid * cols; e += kConsumerWarps * 32) {
        const int r = e / cols, c = it.tn * kBN + e % cols;
        const int64_t o = static_cast<int64_t>(r) * J.ld + c;
        const double v = J.kind == kDfFwd ? J.z[o] : J.ybar[o];
        if (kind == kDfFwd) {  // r = point, c = unit of layer l
          const double zz = v + __ldg(J.bias + c);
          double yy, d1, d2;
          act_eval(J.act, zz, yy, d1, d2);
          J.z[o] = zz;
          J.y[o] = yy;
          J.s1[o] = d1;
          J.s2[o] = d2;
          if (J.lam) {
            const double lv = __ldg(J.lam + static_cast<int64_t>(r) * J.ld_lam + c);
            J.gz_seed[o] = lv * d1;
            J.d_seed[o] = lv * d2;
          }
        } else {  // ADJ: r = point, c = unit of layer l-1
          J.gz[o] = v * __ldcg(J.s1i + o);
          J.d[o] = v * __ldcg(J.s2i + o);
        }
      }
    }
    // ---- publish: stores visible (generic + async proxy) before the count ----
    if (it.sig > 0) {
#ifdef DF_PROXY_FENCE_ALL
      fence_proxy_async_global();
#endif
      consumer_bar();  // CTA-scope: every consumer's stores precede thread 0's release
      if (threadIdx.x == 0) {
        // cumulative gpu-scope fence + generic -> async proxy fence: the
        // tile is visible to later TMA reads of the items that wait on it
        __threadfence();
        fence_proxy_async_global();
        red_release_add(P.counters + it.sig, 1);
      }
    }
    if (P.trace && threadIdx.x == 0) P.trace[4 * idx + 3] = global_ns();
  }
}

// Sum of the SYRK slots' lower triangles, mirrored: H_out[b][r][c] =
// sum_q H_q[b][max(r,c)][min(r,c)] in slot order (exactly symmetric).
__global__ void symmetrize_slots_kernel(const double* __restrict__ hws, int slots, int64_t slot_stride,
                                        int64_t h_point_stride, int64_t ldh, int n, int nb,
                                        double* __restrict__ out) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nn = static_cast<int64_t>(n) * n;
  if (e >= nn * nb) return;
  const int b = static_cast<int>(e / nn);
  const int r = static_cast<int>((e % nn) / n), c = static_cast<int>(e % n);
  const int hi = r > c ? r : c, lo = r > c ? c : r;
  const int64_t o = h_point_stride * b + static_cast<int64_t>(hi) * ldh + lo;
  double v = 0.0;
  for (int q = 0; q < slots; ++q) v += hws[slot_stride * q + o];
  out[e] = v;
}

// Packed lower triangle of H in row order (the reduced-space pattern order,
// formulations.cpp:298-315): out[b][a (a + 1) / 2 + c] = sum_q H_q[b][a][c]
// for c <= a.  Grid (ceil(n / 256), n, nb).
__global__ void pack_lower_kernel(const double* __restrict__ hws, int slots, int64_t slot_stride,
                                  int64_t h_point_stride, int64_t ldh, int n, double* __restrict__ out) {
  const int a = blockIdx.y, b = blockIdx.z;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c > a) return;
  const int64_t o = h_point_stride * b + static_cast<int64_t>(a) * ldh + c;
  double v = 0.0;
  for (int q = 0; q < slots; ++q) v += hws[slot_stride * q + o];
  out[static_cast<int64_t>(b) * n * (n + 1) / 2 + static_cast<int64_t>(a) * (a + 1) / 2 + c] = v;
}

}  // namespace dev
}  // namespace gbb
