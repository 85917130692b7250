// sm_100a kernels of the FP64 gray-box oracle.
//
// The reference computes everything with Eigen on one CPU core
// (reference src/nn.cpp:113-292).  Here the same quantities are produced by:
//
//   fwd_rows_kernel     z_l = W_l y_{l-1} + b_l, epilogue sigma, sigma',
//                       sigma'' (nn.cpp:43-72, 113-146).  HBM-bound GEMV,
//                       one warp per weight row, 16-B coalesced loads.
//   adj_cols_kernel +   ybar_{l-1} = W_l^T (ybar_l .* sigma'_l)
//   adj_reduce_kernel   (nn.cpp:172-196).  HBM-bound column sums with a
//                       deterministic split reduction that also emits the
//                       next layer's gz and d = ybar .* sigma''.
//   nt_mma_kernel       C = A diag(s) B^T on FP64 DMMA.8x8x4 tensor cores:
//                       TMA (cp.async.bulk.tensor, 128B swizzle) -> smem
//                       ring guarded by mbarriers, one producer warp, eight
//                       consumer warps.  Used for the tangent chain
//                       T_{l+1} = T_l diag(sigma'_l) W_{l+1}^T (the forward
//                       tangents of nn.cpp:219-236, transposed) and for the
//                       Hessian SYRK H += T_l diag(ybar_l .* sigma''_l) T_l^T
//                       that replaces the reverse-tangent sweep of
//                       nn.cpp:242-282 (scale applied in registers, the
//                       scaled copy is never materialised).
//   skinny_nt_kernel    the final layer's m <= 16 outputs (tall-skinny).
//   small-K / softmax / symmetrise helpers.
//
// Layout conventions:
//   W_l      row-major [n_l][kp(n_{l-1})], kp(x) = round_up(x, 16)
//   T_l      dz_l/dx transposed: row j = tangent of input direction j,
//            [B * n_pad][kp(n_l)], n_pad = round_up(n, 112)
//   vectors  [B][kp(n_l)], zero padded.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

namespace gbb {
namespace dev {

// ---------------------------------------------------------------------------
// Tiling constants of the DMMA NT kernel.
// ---------------------------------------------------------------------------
constexpr int kBM = 112;              // tile rows  (7 x 16; 784 = 7 x 112)
constexpr int kBN = 128;              // tile cols
constexpr int kBK = 16;               // k per stage = one 128-byte swizzle row
constexpr int kStages = 5;            // smem ring depth (leaves room for a GEMV CTA on the SM)
constexpr int kConsumerWarps = 8;     // 2 (M) x 4 (N)
constexpr int kWarpM = 56;            // 7 DMMA row blocks
constexpr int kWarpN = 32;            // 4 DMMA col blocks
constexpr int kMI = kWarpM / 8;       // 7
constexpr int kNJ = kWarpN / 8;       // 4
constexpr int kThreads = (kConsumerWarps + 1) * 32;
constexpr int kABytes = kBM * kBK * 8;  // 14336 (14 x 1024)
constexpr int kBBytes = kBN * kBK * 8;  // 16384
constexpr int kStageBytes = kABytes + kBBytes;
constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align slack*/ + 256 /*barriers*/;

__host__ __device__ constexpr int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

// ---------------------------------------------------------------------------
// Activations: reference nn.cpp:43-72 (+ softplus, builder extension).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void act_eval(int act, double z, double& y, double& d1, double& d2) {
  switch (act) {
    case 1: {  // tanh
      const double t = tanh(z);
      y = t;
      d1 = 1.0 - t * t;
      d2 = -2.0 * t * (1.0 - t * t);
      return;
    }
    case 2: {  // sigmoid = 0.5 tanh(z/2) + 0.5
      const double s = 0.5 * tanh(0.5 * z) + 0.5;
      const double sp = s * (1.0 - s);
      y = s;
      d1 = sp;
      d2 = sp * (1.0 - 2.0 * s);
      return;
    }
    case 4: {  // softplus (builder extension), stable on both tails
      const double e = exp(-fabs(z));
      const double big = 1.0 / (1.0 + e), small = e / (1.0 + e);
      const double s = z >= 0.0 ? big : small;      // logistic(z)
      const double sm = z >= 0.0 ? small : big;     // logistic(-z) = 1 - s
      y = fmax(z, 0.0) + log1p(e);
      d1 = s;
      d2 = s * sm;
      return;
    }
    default:  // linear (softmax rows are finished by softmax_kernel)
      y = z;
      d1 = 1.0;
      d2 = 0.0;
      return;
  }
}

// ---------------------------------------------------------------------------
// PTX helpers: mbarrier, TMA, DMMA.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// Consumer release of a TMA-filled stage.  The stage was read with generic
// loads (LDS -> registers -> DMMA) and the producer's next TMA load writes it
// through the async proxy: a cross-proxy write-after-read that the mbarrier
// alone does not order.  Each reading thread fences its reads against the
// async proxy, then one lane arrives.  (Without the fence the TMA could land
// before outstanding reads: adj_mma_kernel at 2 CTAs per SM returned wrong
// partials for ~1-4% of its 8-column blocks, tools/adj_mma_conc.cu.)
__device__ __forceinline__ void stage_release(uint64_t* empty, int lane) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(empty)) : "memory");
}
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}
// 2-D tiled TMA load: box lands in smem (128B-swizzled), completion counted
// on `bar` in bytes.
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* m, uint64_t* bar, int c_inner,
                                            int c_outer) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c_inner), "r"(c_outer)
      : "memory");
}
// *p += v at L2 without a return value.  Used where one launch (or one
// dependency-ordered item) is the only writer of an element at a time, so
// the order of the additions is fixed and the result deterministic; it
// replaces a load -> add -> store chain that the compiler serialises per
// element (the store may alias the next load).
__device__ __forceinline__ void red_add_f64(double* p, double v) {
  asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
// D = A(8x4, row) * B(4x8, col) + D on the FP64 tensor pipe (DMMA.8x8x4).
__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}
// Named barrier over the consumer warps only (the producer warp may have exited).
__device__ __forceinline__ void consumer_bar() { asm volatile("bar.sync 1, %0;" ::"n"(kConsumerWarps * 32)); }

// Element (r, k) of a 128B-swizzled [rows][16 doubles] TMA box (TMA's
// SWIZZLE_128B: 16-byte chunk index XOR (row & 7)).  `base` must point into
// shared memory via the __shared__ array so the compiler emits LDS.
__device__ __forceinline__ double lds_swz(const char* base, int r, int k) {
  const int off = r * 128 + ((((k >> 1) ^ (r & 7)) << 4) | ((k & 1) << 3));
  return *reinterpret_cast<const double*>(base + off);
}

// ---------------------------------------------------------------------------
// NT MMA kernel:  C[r][c] (+)= sum_k A[r][k] * s[k] * B[c][k]
// ---------------------------------------------------------------------------
enum NtMode : int { kStore = 0, kAccum = 1, kPartial = 2 };

struct NtParams {
  // Tile enumeration.  For a dense GEMM (tiles == nullptr) the tile id is
  // decoded as (point, tm, tn) with grouped rasterisation over (tm, tn);
  // for the SYRK a host-built list gives (tm, tn) per point.
  const int2* tiles;     // SYRK tile list (tm, tn) or nullptr
  int n_tiles;           // tiles per point in the list
  int tiles_m;           // M tiles per point
  int tiles_n;           // N tiles per point
  int points;            // batch
  int split;             // split-K factor (kPartial when > 1)
  int k_blocks;          // ceil(K / 16)
  // Operand row offsets (rows of the TMA tensors).
  int64_t a_point_rows;  // A row offset per point (0 = broadcast)
  int64_t b_point_rows;  // B row offset per point (0 = shared weights)
  int b_rows_valid;      // rows of B valid per point (cols of C)
  int m_rows_valid;      // rows of C valid per point
  // Per-k scale on B (nullable): s + point * s_stride.
  const double* scale;
  int64_t s_stride;
  // Output.
  double* c;
  int64_t c_point_stride;  // elements
  int64_t ldc;
  int mode;
  double* partial;  // [split][points * n_tiles][kBM][kBN] for kPartial
  int square;       // SYRK on 112 x 112 tiles: B rows tn * kBM, B box kBM rows (see nt_mma_kernel)
  // kStore: also C2 = C diag(c2_scale) (column scale per point), e.g.
  // S_{l+1} = T_{l+1} diag(sigma'_{l+1}) beside T_{l+1}; nullable
  double* c2;
  const double* c2_scale;
  int64_t c2_scale_stride;
  // > 0: number of tiles when the grid is capped below it (persistent CTAs
  // walk tile ids blockIdx.x + j * gridDim.x); 0: one tile per CTA
  int total_tiles;
};

// Grouped rasterisation of a dense tile grid: kGroupM consecutive M tiles
// sweep all N tiles, so CTAs resident together share B (weight) tiles in L2.
__host__ __device__ inline void decode_dense_tile(int local, int tiles_m, int tiles_n, int& tm, int& tn) {
  constexpr int kGroupM = 8;
  const int group = local / (kGroupM * tiles_n);
  const int first_m = group * kGroupM;
  const int gsize = (tiles_m - first_m) < kGroupM ? (tiles_m - first_m) : kGroupM;
  const int in_group = local % (kGroupM * tiles_n);
  tm = first_m + in_group % gsize;
  tn = in_group / gsize;
}

// Row permutation within an 8-row DMMA block: g -> 2(g mod 4) + g/4.
__device__ __forceinline__ int row_perm(int g) { return ((g & 3) << 1) | (g >> 2); }

// Which DMMA blocks (mi, nj) of an MI x NJ warp layout a warp computes.
// kBlkAll: all.  Square SYRK tiles: the two warps of an SM sub-partition
// share a 7 x 7 quadrant as 25 + 24 blocks (kBlkSqLo: block rows 0-2 and
// row 3 columns 0-3; kBlkSqHi, rows 3-6 seen from row 3: row 3 columns 4-6
// and rows 4-6), so both keep the sub-partition's DMMA pipe busy to the end
// of every k-step (a 28 + 21 split leaves the 28-block warp issuing alone).
// kBlkLower + R0: the block lower triangle of a diagonal SYRK tile, for a
// warp whose first block row is R0 (block (mi, nj) is needed iff nj <= R0 + mi).
enum BlkSet : int { kBlkAll = 0, kBlkSqLo = 1, kBlkSqHi = 2, kBlkLower = 16 };
template <int SET>
__host__ __device__ constexpr bool blk_live(int mi, int nj) {
  return SET == kBlkAll    ? true
         : SET == kBlkSqLo ? (mi < 3 || nj < 4)
         : SET == kBlkSqHi ? (mi > 0 || nj >= 4)
                           : nj <= (SET - kBlkLower) + mi;
}

// Diagonal square SYRK tiles (tm == tn) need only the 105 lower blocks of
// the 14 x 14 block grid.  Warp w takes block rows [kDiagR0[w], kDiagR1[w])
// and their columns 0 .. row: per SM sub-partition (warps q, q + 4) that is
// 27 / 26 / 27 / 25 blocks against 49 for a full tile -- the diagonal
// tiles run ~1.8x faster.  (All of these warps keep <= 25 accumulator blocks.)
__host__ __device__ constexpr int diag_r0(int w) {
  return w == 0 ? 0 : w == 1 ? 5 : w == 2 ? 7 : w == 3 ? 10 : w == 4 ? 11 : w == 5 ? 12 : w == 6 ? 9 : 13;
}
__host__ __device__ constexpr int diag_r1(int w) {
  return w == 0 ? 5 : w == 1 ? 7 : w == 2 ? 9 : w == 3 ? 11 : w == 4 ? 12 : w == 5 ? 13 : w == 6 ? 10 : 14;
}

// The consumer k-loop of nt_mma_kernel for an MI x NJ warp layout
// (accumulator block mi * NJ + nj); the per-k scale on B is read one
// k-block ahead through the read-only path (it was written by an earlier
// launch).  SCALED = false: no scale at all -- the tangent GEMMs read the
// pre-scaled S_l = T_l diag(sigma'_l) instead, because the LDS -> DMUL ->
// DMMA chain of a scaled fragment costs ~4% of the tile (measured: c2
// 180.6 -> 187.6 evals/s without the multiplies).
constexpr int kNtAcc = kMI * kNJ;

template <int MI, int NJ, int SET = kBlkAll, bool SCALED = true>
__device__ __forceinline__ void nt_mainloop(double (&acc)[kNtAcc][2], const char* smem, uint64_t* full,
                                            uint64_t* empty, int nkb, int kb_begin, const double* sp, int ra,
                                            int rb, int t, int lane, int b_off, int g0) {
  if (!SCALED) sp = nullptr;
  double sc_next[4];
  if (sp && nkb > 0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) sc_next[q] = __ldg(sp + kb_begin * kBK + 4 * q + t);
  }
  for (int i = 0; i < nkb; ++i) {
    // the smem ring runs on across the tiles of a persistent CTA: stage and
    // phase follow the CTA's global k-block count g0 + i
    const int g = g0 + i;
    const int s = g % kStages;
    double sc[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) sc[q] = sp ? sc_next[q] : 1.0;
    if (sp && i + 1 < nkb) {
#pragma unroll
      for (int q = 0; q < 4; ++q) sc_next[q] = __ldg(sp + (kb_begin + i + 1) * kBK + 4 * q + t);
    }
    mbar_wait(&full[s], (g / kStages) & 1);
    const char* sa = smem + s * kStageBytes;
    const char* sb = sa + b_off;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int k = 4 * q + t;
      double a[MI], b[NJ];
      // the per-k scale goes on whichever operand has fewer fragments
      constexpr bool kScaleA = SCALED && MI < NJ;
      constexpr bool kScaleB = SCALED && !(MI < NJ);
#pragma unroll
      for (int mi = 0; mi < MI; ++mi) a[mi] = kScaleA ? lds_swz(sa, ra + 8 * mi, k) * sc[q] : lds_swz(sa, ra + 8 * mi, k);
#pragma unroll
      for (int nj = 0; nj < NJ; ++nj) b[nj] = kScaleB ? lds_swz(sb, rb + 8 * nj, k) * sc[q] : lds_swz(sb, rb + 8 * nj, k);
#pragma unroll
      for (int mi = 0; mi < MI; ++mi)
#pragma unroll
        for (int nj = 0; nj < NJ; ++nj)
          if (blk_live<SET>(mi, nj)) dmma884(acc[mi * NJ + nj], a[mi], b[nj]);
    }
    stage_release(&empty[s], lane);
  }
}

// Epilogue of one warp's MI x NJ blocks (first mi_n block rows live).
// Tile-relative rows r0 + 8 mi (+ pg), columns c0 + 8 nj (+ pc0 / pc1).
template <int MI, int NJ, int SET = kBlkAll>
__device__ __forceinline__ void nt_store(const double (&acc)[kNtAcc][2], const NtParams& p, int tile, int split_idx,
                                         int point, int tm, int tn, int tile_n, int r0, int c0, int mi_n, int pg,
                                         int pc0, int pc1) {
  if (p.mode == kPartial) {
    double* out = p.partial + ((static_cast<int64_t>(split_idx) * p.points * p.n_tiles +
                                static_cast<int64_t>(tile / p.split)) *
                               kBM * kBN);
#pragma unroll
    for (int mi = 0; mi < MI; ++mi) {
      if (mi >= mi_n) continue;
#pragma unroll
      for (int nj = 0; nj < NJ; ++nj) {
        if (!blk_live<SET>(mi, nj)) continue;
        const int r = r0 + 8 * mi + pg;
        const int cb = c0 + 8 * nj;
        out[r * kBN + cb + pc0] = acc[mi * NJ + nj][0];
        out[r * kBN + cb + pc1] = acc[mi * NJ + nj][1];
      }
    }
    return;
  }
  double* cbase = p.c + p.c_point_stride * point;
  double* c2base = p.c2 ? p.c2 + p.c_point_stride * point : nullptr;
  const double* c2s = p.c2 ? p.c2_scale + p.c2_scale_stride * point : nullptr;
#pragma unroll
  for (int mi = 0; mi < MI; ++mi) {
    const int r = tm * kBM + r0 + 8 * mi + pg;
    if (mi >= mi_n || r >= p.m_rows_valid) continue;
#pragma unroll
    for (int nj = 0; nj < NJ; ++nj) {
      if (!blk_live<SET>(mi, nj)) continue;
      const int cb = tn * tile_n + c0 + 8 * nj;
      double* dst = cbase + static_cast<int64_t>(r) * p.ldc + cb;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = h ? pc1 : pc0;
        if (cb + c < p.b_rows_valid) {
          if (p.mode == kAccum) {
            red_add_f64(dst + c, acc[mi * NJ + nj][h]);
          } else {
            dst[c] = acc[mi * NJ + nj][h];
            if (c2base) c2base[static_cast<int64_t>(r) * p.ldc + cb + c] = acc[mi * NJ + nj][h] * __ldg(c2s + cb + c);
          }
        }
      }
    }
  }
}

// One tile of an nt_mma launch: split-K slice, point, tile coordinates and
// the k-block range (a plain function: a lambda capturing the kernel
// parameters by reference forced them into local memory).
struct NtTile {
  int split_idx, point, tm, tn, kb_begin, nkb, a_row0, b_row0;
  bool diag;
};
__device__ __forceinline__ NtTile nt_decode(const NtParams& p, int tile, bool sq, int tile_n) {
  NtTile T;
  int bid = tile;
  T.split_idx = bid % p.split;
  bid /= p.split;
  if (p.tiles != nullptr) {
    T.point = bid / p.n_tiles;
    const int2 tt = p.tiles[bid % p.n_tiles];
    T.tm = tt.x;
    T.tn = tt.y;
  } else {
    const int per_point = p.tiles_m * p.tiles_n;
    T.point = bid / per_point;
    decode_dense_tile(bid % per_point, p.tiles_m, p.tiles_n, T.tm, T.tn);
  }
  T.kb_begin = static_cast<int>((static_cast<int64_t>(p.k_blocks) * T.split_idx) / p.split);
  const int kb_end = static_cast<int>((static_cast<int64_t>(p.k_blocks) * (T.split_idx + 1)) / p.split);
  T.nkb = kb_end - T.kb_begin;
  T.a_row0 = static_cast<int>(p.a_point_rows * T.point) + T.tm * kBM;
  T.b_row0 = static_cast<int>(p.b_point_rows * T.point) + T.tn * tile_n;
  T.diag = sq && T.tm == T.tn && p.a_point_rows == p.b_point_rows;
  return T;
}

// The consumer side of dense GEMM tiles, looping over this CTA's tiles
// (persistent launches) with the smem ring position carried across tiles.
template <bool kScaled, bool kPersist>
__device__ __forceinline__ void nt_dense_tiles(const NtParams& p, const char* smem, uint64_t* full, uint64_t* empty,
                                               int total, int tile_n, int ra, int rb, int r0, int c0, int pg, int pc0,
                                               int pc1, int t, int lane) {
  if constexpr (!kPersist) {
    // one tile per CTA: straight-line code (the loop below costs registers
    // -- 104 bytes of spills at the 168-register cap -- and 2% on c4)
    const int tile = blockIdx.x;
    const NtTile T = nt_decode(p, tile, false, tile_n);
    double acc[kNtAcc][2];
#pragma unroll
    for (int i = 0; i < kNtAcc; ++i) acc[i][0] = acc[i][1] = 0.0;
    const double* sp = kScaled ? p.scale + p.s_stride * T.point : nullptr;
    nt_mainloop<kMI, kNJ, kBlkAll, kScaled>(acc, smem, full, empty, T.nkb, T.kb_begin, sp, ra, rb, t, lane, kABytes,
                                            0);
    nt_store<kMI, kNJ>(acc, p, tile, T.split_idx, T.point, T.tm, T.tn, tile_n, r0, c0, kMI, pg, pc0, pc1);
    return;
  }
  int gk = 0;  // k-blocks consumed so far by this CTA (ring position)
  for (int tile = blockIdx.x; tile < total; tile += gridDim.x) {
    const NtTile T = nt_decode(p, tile, false, tile_n);
    double acc[kNtAcc][2];
#pragma unroll
    for (int i = 0; i < kNtAcc; ++i) acc[i][0] = acc[i][1] = 0.0;
    const double* sp = kScaled ? p.scale + p.s_stride * T.point : nullptr;
    nt_mainloop<kMI, kNJ, kBlkAll, kScaled>(acc, smem, full, empty, T.nkb, T.kb_begin, sp, ra, rb, t, lane, kABytes,
                                            gk);
    nt_store<kMI, kNJ>(acc, p, tile, T.split_idx, T.point, T.tm, T.tn, tile_n, r0, c0, kMI, pg, pc0, pc1);
    gk += T.nkb;
  }
}

// Square SYRK tiles (p.square): the tile is 112 x 112 (B rows tn * 112, a
// 112-row B box) over the lower triangle -- 87.6% useful work at n = 784
// against 76.7% for 112 x 128 tiles.  SM sub-partition q = warp & 3 owns the
// 56 x 56 quadrant q, split between its two warps as 25 + 24 of its 7 x 7
// blocks (blk_live), so each sub-partition's DMMA pipe gets 49 blocks.
// (168 registers is the real cap: the 9-warp CTA puts 3 warps on one SM
// sub-partition, 3 x 32 x 168 <= 16384 registers; 185 failed to launch)
template <bool kPersist>
__global__ void __launch_bounds__(kThreads, 1)
   
    nt_mma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                  const NtParams p) {
  extern __shared__ unsigned char smem_raw[];
  // 1024-byte alignment for the 128B swizzle, derived from the __shared__
  // array itself so loads stay in the shared window (LDS, not generic LD).
  char* smem = reinterpret_cast<char*>(smem_raw) + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty = full + kStages;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const bool sq = p.square != 0;
  const int tile_n = sq ? kBM : kBN;

  // ---- tile decode: the CTA walks tiles blockIdx.x, + gridDim.x, ... (one
  // tile when the launch has a CTA per tile; persistent when the grid is
  // capped at the SM count, so the producer streams the next tile's k-blocks
  // into the ring while the consumers run the current tile's epilogue) ----
  // persistent launches (total_tiles > 0) are dense GEMMs only; square SYRK
  // launches keep one tile per CTA (their consumers below handle one tile)
  const int total = (kPersist && !sq) ? p.total_tiles : static_cast<int>(gridDim.x);

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == kConsumerWarps) {
    // ===== producer warp: one elected lane issues the TMA ring =====
    if (lane == 0) {
      tma_prefetch_desc(&tmA);
      tma_prefetch_desc(&tmB);
      int gk = 0;  // k-blocks issued so far by this CTA (ring position)
      for (int tile = blockIdx.x; tile < total; tile += gridDim.x) {
        const NtTile T = nt_decode(p, tile, sq, tile_n);
        // diagonal square SYRK tiles: B == A, one box per stage
        const uint32_t bytes = T.diag ? kABytes : kABytes + (sq ? kABytes : kBBytes);
        for (int i = 0; i < T.nkb; ++i, ++gk) {
          const int s = gk % kStages;
          if (gk >= kStages) mbar_wait(&empty[s], ((gk / kStages) - 1) & 1);
          char* sa = smem + s * kStageBytes;
          char* sb = sa + kABytes;
          mbar_arrive_expect_tx(&full[s], bytes);
          const int kc = (T.kb_begin + i) * kBK;
          tma_load_2d(sa, &tmA, &full[s], kc, T.a_row0);
          if (!T.diag) tma_load_2d(sb, &tmB, &full[s], kc, T.b_row0);
        }
      }
      // producer tail: stay until the consumers have released the last
      // stages (see adj_mma_kernel: no issuing warp exits with bulk copies
      // in flight)
      for (int g2 = gk > kStages ? gk - kStages : 0; g2 < gk; ++g2) mbar_wait(&empty[g2 % kStages], (g2 / kStages) & 1);
    }
    __syncwarp();
    return;
  }

  // ===== consumer warps =====
  const int g = lane >> 2;  // DMMA group (row of A / col of B)
  const int t = lane & 3;   // thread in group (k)
  // DMMA group g reads smem row 8*blk + row_perm(g): with the TMA 128B
  // swizzle this makes each half-warp's 16 LDS.64 hit 32 distinct banks
  // (identity order gives 2-way conflicts).  C inherits the permutation.
  const int pg = row_perm(g);
  const int pc0 = row_perm(2 * t), pc1 = row_perm(2 * t + 1);
  if (!sq) {
    // dense GEMM tiles: the persistent loop (one code path per launch, so the
    // accumulators keep one register assignment across the loop)
    const int wm = warp >> 2;  // 0..1
    const int wn = warp & 3;   // 0..3
    const int r0 = wm * kWarpM, c0 = wn * kWarpN;
    if (p.scale)
      nt_dense_tiles<true, kPersist>(p, smem, full, empty, total, tile_n, r0 + pg, c0 + pg, r0, c0, pg, pc0, pc1, t,
                                     lane);
    else
      nt_dense_tiles<false, kPersist>(p, smem, full, empty, total, tile_n, r0 + pg, c0 + pg, r0, c0, pg, pc0, pc1,
                                      t, lane);
    return;
  }
  // square SYRK tiles: one tile per CTA (the host does not cap these grids)
  {
    const int tile = blockIdx.x;
    const int gk = 0;
    const NtTile T = nt_decode(p, tile, sq, tile_n);
    const int split_idx = T.split_idx, point = T.point, tm = T.tm, tn = T.tn, nkb = T.nkb, kb_begin = T.kb_begin;
    double acc[kNtAcc][2];
#pragma unroll
    for (int i = 0; i < kNtAcc; ++i) acc[i][0] = acc[i][1] = 0.0;
    const double* sp = p.scale ? p.scale + p.s_stride * point : nullptr;
    if (T.diag) {
      // block rows [diag_r0(w), diag_r1(w)), columns 0 .. row (B fragments from the A box)
#define GBB_DIAG_WARP(W)                                                                                     \
  case W: {                                                                                                  \
    constexpr int R0 = diag_r0(W), R1 = diag_r1(W);                                                          \
    nt_mainloop<R1 - R0, R1, kBlkLower + R0>(acc, smem, full, empty, nkb, kb_begin, sp, 8 * R0 + pg, pg, t,    \
                                            lane, 0, gk);                                                    \
    nt_store<R1 - R0, R1, kBlkLower + R0>(acc, p, tile, split_idx, point, tm, tn, tile_n, 8 * R0, 0, R1 - R0, \
                                         pg, pc0, pc1);                                                      \
    break;                                                                                                   \
  }
      switch (warp) {
        GBB_DIAG_WARP(0)
        GBB_DIAG_WARP(1)
        GBB_DIAG_WARP(2)
        GBB_DIAG_WARP(3)
        GBB_DIAG_WARP(4)
        GBB_DIAG_WARP(5)
        GBB_DIAG_WARP(6)
        GBB_DIAG_WARP(7)
        default: break;
      }
#undef GBB_DIAG_WARP
    } else {
      const int q = warp & 3, h = warp >> 2;
      const int r0 = (q >> 1) * 56 + h * 24, c0 = (q & 1) * 56;
      if (h == 0) {
        nt_mainloop<4, 7, kBlkSqLo>(acc, smem, full, empty, nkb, kb_begin, sp, r0 + pg, c0 + pg, t, lane, kABytes,
                                    gk);
        nt_store<4, 7, kBlkSqLo>(acc, p, tile, split_idx, point, tm, tn, tile_n, r0, c0, 4, pg, pc0, pc1);
      } else {
        nt_mainloop<4, 7, kBlkSqHi>(acc, smem, full, empty, nkb, kb_begin, sp, r0 + pg, c0 + pg, t, lane, kABytes,
                                    gk);
        nt_store<4, 7, kBlkSqHi>(acc, p, tile, split_idx, point, tm, tn, tile_n, r0, c0, 4, pg, pc0, pc1);
      }
    }
  }
}

// Sum split-K SYRK partials (fixed order: deterministic) into H_ws.
__global__ void syrk_partial_reduce_kernel(const double* __restrict__ partial, const int2* __restrict__ tiles,
                                           int n_tiles, int points, int split, double* __restrict__ h,
                                           int64_t h_point_stride, int64_t ldh, int n_valid, int tile_n) {
  const int tile_global = blockIdx.y;  // point * n_tiles + tile
  const int point = tile_global / n_tiles;
  const int2 t = tiles[tile_global % n_tiles];
  const int64_t tile_elems = static_cast<int64_t>(kBM) * kBN;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < kBM * kBN; e += gridDim.x * blockDim.x) {
    if (e % kBN >= tile_n) continue;  // square tiles use the first kBM columns of a partial row
    const int r = t.x * kBM + e / kBN;
    const int c = t.y * tile_n + e % kBN;
    if (r >= n_valid || c >= n_valid) continue;
    double sum = 0.0;
    for (int s = 0; s < split; ++s)
      sum += partial[(static_cast<int64_t>(s) * points * n_tiles + tile_global) * tile_elems + e];
    h[h_point_stride * point + static_cast<int64_t>(r) * ldh + c] += sum;
  }
}

// ---------------------------------------------------------------------------
// Batched forward / adjoint as GEMMs (B points >= kBatchGemm):
//   forward  Z_l    = Y_{l-1} W_l^T        (nt_mma, then act epilogue)
//   adjoint  Ybar_l = GZ_{l+1} W_{l+1}     (nt_mma on the W^T copy, then
//                                            gz/d epilogue)
// The epilogue runs either inside the split-K reduction or as a separate
// elementwise pass over the stored GEMM result.
// ---------------------------------------------------------------------------
enum EpiMode : int { kEpiAct = 0, kEpiAdj = 1, kEpiStore = 2 };

struct RowEpi {
  int mode;
  int act;
  const double* bias;                 // act
  double *z, *y, *s1o, *s2o;          // act outputs
  const double *s1i, *s2i;            // adj inputs (sigma', sigma'' of this layer)
  double *ybar, *gz, *d;              // adj outputs (gz, d nullable)
  int64_t ld;
  int s_div;  // adj: rows r share the sigma' / sigma'' row r / s_div (reverse-mode J seeds); 0 == 1
};

__device__ __forceinline__ void apply_row_epi(const RowEpi& e, int r, int c, double v) {
  const int64_t o = static_cast<int64_t>(r) * e.ld + c;
  if (e.mode == kEpiStore) {  // plain store into e.z (pitch e.ld); e.y = e.z diag(e.s1i) when set
    e.z[o] = v;
    if (e.y) e.y[o] = v * e.s1i[c];
    return;
  }
  if (e.mode == kEpiAct) {
    const double zz = v + e.bias[c];
    double yy, d1, d2;
    act_eval(e.act, zz, yy, d1, d2);
    e.z[o] = zz;
    e.y[o] = yy;
    e.s1o[o] = d1;
    e.s2o[o] = d2;
  } else {
    e.ybar[o] = v;
    if (e.gz) {
      const int64_t os = e.s_div > 1 ? static_cast<int64_t>(r / e.s_div) * e.ld + c : o;
      e.gz[o] = v * e.s1i[os];
      if (e.d) e.d[o] = v * e.s2i[os];
    }
  }
}

// Elementwise epilogue over a stored [rows][cols] GEMM result (pitch e.ld).
__global__ void rows_epilogue_kernel(const double* __restrict__ v, int rows, int cols, RowEpi e) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= static_cast<int64_t>(rows) * cols) return;
  const int r = static_cast<int>(i / cols), c = static_cast<int>(i % cols);
  apply_row_epi(e, r, c, v[static_cast<int64_t>(r) * e.ld + c]);
}

// Split-K reduction of a dense nt_mma GEMM (kPartial) in fixed split order,
// fused with the row epilogue.  One block row per tile.
__global__ void gemm_partial_reduce_kernel(const double* __restrict__ partial, int split, int tiles_m, int tiles_n,
                                           int rows_valid, int cols_valid, RowEpi e) {
  const int tile = blockIdx.y;
  int tm, tn;
  decode_dense_tile(tile, tiles_m, tiles_n, tm, tn);
  const int64_t n_t = static_cast<int64_t>(tiles_m) * tiles_n;
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < kBM * kBN; x += gridDim.x * blockDim.x) {
    const int r = tm * kBM + x / kBN, c = tn * kBN + x % kBN;
    if (r >= rows_valid || c >= cols_valid) continue;
    double sum = 0.0;
    for (int s = 0; s < split; ++s) sum += partial[(static_cast<int64_t>(s) * n_t + tile) * kBM * kBN + x];
    apply_row_epi(e, r, c, sum);
  }
}

// out[c][r] = in[r][c] for an [rows][cols] matrix (pitches in doubles).
__global__ void transpose_kernel(const double* __restrict__ in, int64_t ldi, int rows, int cols,
                                 double* __restrict__ out, int64_t ldo) {
  __shared__ double t[32][33];
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const int r = r0 + j, c = c0 + threadIdx.x;
    t[j][threadIdx.x] = (r < rows && c < cols) ? in[static_cast<int64_t>(r) * ldi + c] : 0.0;
  }
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const int c = c0 + j, r = r0 + threadIdx.x;
    if (c < cols && r < rows) out[static_cast<int64_t>(c) * ldo + r] = t[threadIdx.x][j];
  }
}

// ---------------------------------------------------------------------------
// Per-point Hessian over several K segments in ONE diagonal tile (n <= 112,
// e.g. the c4 contingencies: n = 108): H_p = sum_s T_s,p^T diag(D_s,p) T_s,p
// with the hidden layers' K ranges concatenated -- one launch and one store
// of each point's tile instead of one launch per layer accumulating into H
// (and no zeroing pass).  Segment s reads its A boxes from tensor map s at
// row a_point_rows[s] * point (0: the shared T_0 = W_0^T), its per-k scale
// from scale[s] + s_stride[s] * point.  Same consumers as nt_mma_kernel's
// diagonal tiles (the block lower triangle, kBlkLower).
// ---------------------------------------------------------------------------
constexpr int kMaxSegs = 4;
struct SyrkSegs {
  int nseg;
  int nkb[kMaxSegs];
  const double* scale[kMaxSegs];
  int64_t s_stride[kMaxSegs];
  int64_t a_point_rows[kMaxSegs];
};

__global__ void __launch_bounds__(kThreads, 1)
    nt_syrk_segs_kernel(const __grid_constant__ CUtensorMap tm0, const __grid_constant__ CUtensorMap tm1,
                        const __grid_constant__ CUtensorMap tm2, const __grid_constant__ CUtensorMap tm3,
                        const NtParams p, const SyrkSegs sg) {
  extern __shared__ unsigned char smem_raw[];
  char* smem = reinterpret_cast<char*>(smem_raw) + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int point = blockIdx.x;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    fence_barrier_init();
  }
  __syncthreads();
  if (warp == kConsumerWarps) {
    if (lane == 0) {
      int gk = 0;
      for (int sgi = 0; sgi < sg.nseg; ++sgi) {
        const CUtensorMap* tm = sgi == 0 ? &tm0 : sgi == 1 ? &tm1 : sgi == 2 ? &tm2 : &tm3;
        tma_prefetch_desc(tm);
        const int row0 = static_cast<int>(sg.a_point_rows[sgi] * point);
        for (int i = 0; i < sg.nkb[sgi]; ++i, ++gk) {
          const int s = gk % kStages;
          if (gk >= kStages) mbar_wait(&empty[s], ((gk / kStages) - 1) & 1);
          char* sa = smem + s * kStageBytes;
          mbar_arrive_expect_tx(&full[s], kABytes);
          tma_load_2d(sa, tm, &full[s], i * kBK, row0);
        }
      }
      for (int g2 = gk > kStages ? gk - kStages : 0; g2 < gk; ++g2) mbar_wait(&empty[g2 % kStages], (g2 / kStages) & 1);
    }
    __syncwarp();
    return;
  }
  const int g = lane >> 2, t = lane & 3;
  const int pg = row_perm(g);
  const int pc0 = row_perm(2 * t), pc1 = row_perm(2 * t + 1);
  double acc[kNtAcc][2];
#pragma unroll
  for (int i = 0; i < kNtAcc; ++i) acc[i][0] = acc[i][1] = 0.0;
#define GBB_SEG_WARP(W)                                                                                       \
  case W: {                                                                                                   \
    constexpr int R0 = diag_r0(W), R1 = diag_r1(W);                                                           \
    int gk = 0;                                                                                               \
    for (int sgi = 0; sgi < sg.nseg; ++sgi) {                                                                 \
      nt_mainloop<R1 - R0, R1, kBlkLower + R0>(acc, smem, full, empty, sg.nkb[sgi], 0,                        \
                                              sg.scale[sgi] + sg.s_stride[sgi] * point, 8 * R0 + pg, pg, t,   \
                                              lane, 0, gk);                                                   \
      gk += sg.nkb[sgi];                                                                                      \
    }                                                                                                         \
    nt_store<R1 - R0, R1, kBlkLower + R0>(acc, p, point, 0, point, 0, 0, kBM, 8 * R0, 0, R1 - R0, pg, pc0,    \
                                         pc1);                                                                \
    break;                                                                                                    \
  }
  switch (warp) {
    GBB_SEG_WARP(0)
    GBB_SEG_WARP(1)
    GBB_SEG_WARP(2)
    GBB_SEG_WARP(3)
    GBB_SEG_WARP(4)
    GBB_SEG_WARP(5)
    GBB_SEG_WARP(6)
    GBB_SEG_WARP(7)
    default: break;
  }
#undef GBB_SEG_WARP
}

// ---------------------------------------------------------------------------
// Forward GEMV chain: z = W y + b with the activation epilogue.
// One warp per output row; NB points per pass, y chunk staged in smem.
// ---------------------------------------------------------------------------
constexpr int kFwdWarps = 8;

// Single point (the c2 hot case): HBM-streaming GEMV, no shared-memory
// staging and no block barriers in the k loop (y is re-read through L1).
// WPR warps share a row (split K, fixed-order reduction through shared
// memory: deterministic) so layers with few rows still fill the GPU; each
// lane keeps 8 independent 16-byte weight loads in flight.
// Optional extras of a single point's last forward layer (elementwise
// output): the y output copy and the adjoint seed gz = lambda sigma',
// d = lambda sigma'' (adj_seed_kernel) -- two dependent launches fewer.
struct FwdTail {
  double* y;          // nullable: y output
  const double* lam;  // nullable: seed the adjoint
  double* gz;
  double* d;
};

template <int WPR>
__global__ void __launch_bounds__(kFwdWarps * 32)
    fwd_row1_kernel(const double* __restrict__ w, int64_t ldw, const double* __restrict__ bias, int rows, int k_dim,
                    const double* __restrict__ yin, int act, double* __restrict__ z_out, double* __restrict__ y_out,
                    double* __restrict__ s1_out, double* __restrict__ s2_out, FwdTail tail) {
  constexpr int kRowsPerCta = kFwdWarps / WPR;
  __shared__ double part[kFwdWarps];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x * kRowsPerCta + warp / WPR;
  const int part_idx = warp % WPR;
  // this warp's k range: whole 64-double chunks, split WPR ways
  const int chunks = (k_dim + 63) / 64;
  const int c0 = (chunks * part_idx) / WPR, c1 = (chunks * (part_idx + 1)) / WPR;
  double acc0 = 0.0, acc1 = 0.0;
  if (row < rows) {
    const double* wr = w + static_cast<int64_t>(row) * ldw;
    int c = c0;
    // kU chunks (kU x 16 B per lane) per step: loads first, then the FMAs
    constexpr int kU = 8;  // 16 measured slower (3.9 vs 4.6 TB/s)
    for (; c + kU <= c1; c += kU) {
      double2 wv[kU], yv[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int k = (c + u) * 64 + 2 * lane;
        wv[u] = k < k_dim ? __ldcs(reinterpret_cast<const double2*>(wr + k)) : make_double2(0.0, 0.0);
        yv[u] = k < k_dim ? __ldg(reinterpret_cast<const double2*>(yin + k)) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        acc0 = fma(wv[u].x, yv[u].x, acc0);
        acc1 = fma(wv[u].y, yv[u].y, acc1);
      }
    }
    for (; c < c1; ++c) {
      const int k = c * 64 + 2 * lane;
      if (k < k_dim) {
        const double2 wv = __ldcs(reinterpret_cast<const double2*>(wr + k));
        const double2 yv = __ldg(reinterpret_cast<const double2*>(yin + k));
        acc0 = fma(wv.x, yv.x, acc0);
        acc1 = fma(wv.y, yv.y, acc1);
      }
    }
  }
  double v = acc0 + acc1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (WPR > 1) {
    if (lane == 0) part[warp] = v;
    __syncthreads();
    if (part_idx != 0) return;
    v = 0.0;
    for (int i = 0; i < WPR; ++i) v += part[warp + i];  // fixed order
  }
  if (lane == 0 && row < rows) {
    const double zz = v + bias[row];
    double yy, d1, d2;
    act_eval(act, zz, yy, d1, d2);
    z_out[row] = zz;
    y_out[row] = yy;
    s1_out[row] = d1;
    s2_out[row] = d2;
    if (tail.y) tail.y[row] = yy;
    if (tail.lam) {  // adj_seed_kernel's elementwise seed, same products
      tail.gz[row] = tail.lam[row] * d1;
      tail.d[row] = tail.lam[row] * d2;
    }
  }
}

template <int NB>
__global__ void __launch_bounds__(kFwdWarps * 32)
    fwd_rows_kernel(const double* __restrict__ w, int64_t ldw, const double* __restrict__ bias, int rows, int k_dim,
                    const double* __restrict__ yin, int64_t ld_in, int nb, int act, double* __restrict__ z_out,
                    double* __restrict__ y_out, double* __restrict__ s1_out, double* __restrict__ s2_out,
                    int64_t ld_out) {
  // 16 KB of staged inputs: small enough to co-reside with an nt_mma CTA
  // (the forward runs beside the tangent GEMMs on the side stream)
  constexpr int kFwdKChunk = 2048 / NB;
  __shared__ __align__(16) double ys[NB][kFwdKChunk];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x * kFwdWarps + warp;
  const int p0 = blockIdx.y * NB;
  double acc[NB];
#pragma unroll
  for (int b = 0; b < NB; ++b) acc[b] = 0.0;
  const double* wr = w + static_cast<int64_t>(row < rows ? row : 0) * ldw;
  for (int k0 = 0; k0 < k_dim; k0 += kFwdKChunk) {
    const int kc = min(kFwdKChunk, k_dim - k0);
    const int kc2 = (kc + 1) & ~1;
    __syncthreads();
    for (int b = 0; b < NB; ++b) {
      const bool live = (p0 + b) < nb;
      for (int k = threadIdx.x; k < kc2; k += blockDim.x)
        ys[b][k] = (live && k < kc) ? yin[static_cast<int64_t>(p0 + b) * ld_in + k0 + k] : 0.0;
    }
    __syncthreads();
    if (row < rows) {
      // weight rows are padded to a multiple of 16 doubles with zeros, so
      // reading the (kc rounded to 2) tail is safe.
#pragma unroll 4
      for (int k = 2 * lane; k < kc2; k += 64) {
        const double2 wv = __ldg(reinterpret_cast<const double2*>(wr + k0 + k));
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          const double2 yv = *reinterpret_cast<const double2*>(&ys[b][k]);
          acc[b] = fma(wv.x, yv.x, acc[b]);
          acc[b] = fma(wv.y, yv.y, acc[b]);
        }
      }
    }
  }
  if (row >= rows) return;
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    double v = acc[b];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    acc[b] = v;
  }
  if (lane < NB && p0 + lane < nb) {
    double zz = 0.0;
#pragma unroll
    for (int b = 0; b < NB; ++b)
      if (b == lane) zz = acc[b];
    zz += bias[row];
    const int64_t o = static_cast<int64_t>(p0 + lane) * ld_out + row;
    double yy, d1, d2;
    act_eval(act, zz, yy, d1, d2);
    z_out[o] = zz;
    y_out[o] = yy;
    s1_out[o] = d1;
    s2_out[o] = d2;
  }
}

// Softmax over each point's final-layer row: nn.cpp:12-17.
__global__ void softmax_kernel(const double* __restrict__ z, double* __restrict__ y, int m, int64_t ld, int nb) {
  const int pt = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (pt >= nb) return;
  const double* zr = z + ld * pt;
  double mx = -INFINITY;
  for (int i = lane; i < m; i += 32) mx = fmax(mx, zr[i]);
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  double sum = 0.0;
  for (int i = lane; i < m; i += 32) sum += exp(zr[i] - mx);
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  // deterministic: each lane recomputes its own entries with the same sum
  for (int i = lane; i < m; i += 32) y[ld * pt + i] = exp(zr[i] - mx) / sum;
}

// ---------------------------------------------------------------------------
// Adjoint seed at the output layer: ybar_L = lambda.
//   elementwise: gz = lambda .* s1, d = lambda .* s2
//   softmax:     gz = y .* lambda - (y^T lambda) y ;  d unused (dense M)
// One warp per point.
// ---------------------------------------------------------------------------
__global__ void adj_seed_kernel(const double* __restrict__ lam, int64_t ld_lam, const double* __restrict__ y,
                                const double* __restrict__ s1, const double* __restrict__ s2, int64_t ld, int m,
                                int nb, int softmax, double* __restrict__ gz, double* __restrict__ d,
                                double* __restrict__ mid, int64_t ld_mid) {
  const int pt = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (pt >= nb) return;
  const double* lr = lam + ld_lam * pt;
  if (!softmax) {
    for (int i = lane; i < m; i += 32) {
      gz[ld * pt + i] = lr[i] * s1[ld * pt + i];
      d[ld * pt + i] = lr[i] * s2[ld * pt + i];
    }
    return;
  }
  const double* yr = y + ld * pt;
  double s = 0.0;
  for (int i = lane; i < m; i += 32) s += yr[i] * lr[i];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  for (int i = lane; i < m; i += 32) gz[ld * pt + i] = yr[i] * lr[i] - s * yr[i];
  // M = sum_i lambda_i Hess(softmax_i):
  //   M_jk = delta_jk y_j (lambda_j - s) - y_j y_k (lambda_j + lambda_k - 2 s)
  double* mr = mid + ld_mid * pt;
  for (int e = lane; e < m * m; e += 32) {
    const int j = e / m, k = e % m;
    double v = -yr[j] * yr[k] * (lr[j] + lr[k] - 2.0 * s);
    if (j == k) v += yr[j] * (lr[j] - s);
    mr[e] = v;
  }
}

// ---------------------------------------------------------------------------
// Adjoint GEMV^T: partial[c][b][k] = sum_{i in chunk c} W[i][k] gz[b][i].
// Threads own two adjacent k (16-B loads, coalesced along the row).
// ---------------------------------------------------------------------------
constexpr int kAdjThreads = 256;
constexpr int kAdjRows = 128;

// The chunk reduction of adj_reduce_kernel folded into the column sweep
// (counters != nullptr): the last chunk CTA of each column block to finish
// (a self-resetting arrival counter per column block) sums that block's
// partials over the chunks in ascending order -- the same order and the
// same values as adj_reduce_kernel, so bit-identical -- and emits ybar / gz /
// d.  Saves one dependent launch per layer of the adjoint chain.
struct AdjFuse {
  unsigned* counters;  // [gridDim.x], zero between launches
  int chunks;
  const double* s1;
  const double* s2;
  int64_t ld;
  double* ybar;
  double* gz;
  double* d;
  int s_div;
};

// KW adjacent k per thread (2: one 16-B load per row; 4: two), so a row's
// NB shared-memory gz values are reused over KW columns -- the multi-vector
// sweeps (reverse-mode J: NB = 12 / 16) are otherwise bound by those loads.
template <int NB, int KW>
__device__ __forceinline__ void adj_cols_sweep(const double* __restrict__ w, int64_t ldw,
                                               const double (&gs)[NB][kAdjRows], int k, int k_dim, int r0, int nr,
                                               int nb, int p0, double* __restrict__ partial, int64_t ld_part) {
  double a[NB][KW];
#pragma unroll
  for (int b = 0; b < NB; ++b)
#pragma unroll
    for (int c = 0; c < KW; ++c) a[b][c] = 0.0;
  const double* wp = w + static_cast<int64_t>(r0) * ldw + k;
  // kRB rows' weights in flight before their FMAs: the multi-vector sweeps
  // were latency-bound with the loads interleaved (ncu: 2 CTAs per SM, DFMA
  // stalled on the loads, 3.0 TB/s).  Each accumulator still takes the rows
  // in ascending order, so the sums are bit-identical.
  // (measured, c2: single-vector adjoint 39-47 -> 35-41 us per 5120^2 layer,
  // 12-vector reverse-mode J 72 -> 60-66 us; 4 rows for NB >= 8 was between)
  constexpr int kRB = KW == 2 ? 8 : 4;
  int i = 0;
  for (; i + kRB <= nr; i += kRB) {
    double wv[kRB][KW];
#pragma unroll
    for (int r = 0; r < kRB; ++r) {
      const double2 w01 = __ldg(reinterpret_cast<const double2*>(wp + static_cast<int64_t>(i + r) * ldw));
      wv[r][0] = w01.x;
      wv[r][1] = w01.y;
      if constexpr (KW == 4) {
        // k + 2 < ldw always (ldw is a multiple of 16 and k a multiple of 4);
        // columns past k_dim are the zero padding
        const double2 w23 = __ldg(reinterpret_cast<const double2*>(wp + static_cast<int64_t>(i + r) * ldw + 2));
        wv[r][2] = w23.x;
        wv[r][3] = w23.y;
      }
    }
#pragma unroll
    for (int r = 0; r < kRB; ++r)
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const double g = gs[b][i + r];
#pragma unroll
        for (int c = 0; c < KW; ++c) a[b][c] = fma(wv[r][c], g, a[b][c]);
      }
  }
  for (; i < nr; ++i) {
    double wv[KW];
    const double2 w01 = __ldg(reinterpret_cast<const double2*>(wp + static_cast<int64_t>(i) * ldw));
    wv[0] = w01.x;
    wv[1] = w01.y;
    if constexpr (KW == 4) {
      const double2 w23 = __ldg(reinterpret_cast<const double2*>(wp + static_cast<int64_t>(i) * ldw + 2));
      wv[2] = w23.x;
      wv[3] = w23.y;
    }
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const double g = gs[b][i];
#pragma unroll
      for (int c = 0; c < KW; ++c) a[b][c] = fma(wv[c], g, a[b][c]);
    }
  }
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    if (p0 + b >= nb) break;
    double* o = partial + (static_cast<int64_t>(blockIdx.y) * nb + p0 + b) * ld_part + k;
#pragma unroll
    for (int c = 0; c < KW; ++c)
      if (k + c < k_dim) o[c] = a[b][c];
  }
}

template <int NB, int KW = 2>
__global__ void __launch_bounds__(kAdjThreads, NB * KW <= 32 ? 2 : 1)
    adj_cols_kernel(const double* __restrict__ w, int64_t ldw, int rows, int k_dim, const double* __restrict__ gz,
                    int64_t ld_gz, int nb, int p0, double* __restrict__ partial, int64_t ld_part, int crows,
                    AdjFuse f) {
  static_assert(KW == 2 || KW == 4, "KW");
  __shared__ double gs[NB][kAdjRows];
  __shared__ int last;
  const int k = KW * (blockIdx.x * kAdjThreads + threadIdx.x);
  const int r0 = blockIdx.y * crows;  // crows <= kAdjRows rows per chunk
  const int nr = min(crows, rows - r0);
  for (int e = threadIdx.x; e < NB * kAdjRows; e += kAdjThreads) {
    const int b = e / kAdjRows, i = e % kAdjRows;
    gs[b][i] = (p0 + b < nb && i < nr) ? gz[static_cast<int64_t>(p0 + b) * ld_gz + r0 + i] : 0.0;
  }
  __syncthreads();
  if (k < k_dim) adj_cols_sweep<NB, KW>(w, ldw, gs, k, k_dim, r0, nr, nb, p0, partial, ld_part);
  if (f.counters == nullptr) return;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    last = atomicAdd(&f.counters[blockIdx.x], 1u) == gridDim.y - 1;
    if (last) f.counters[blockIdx.x] = 0;  // the next launch (stream-ordered) starts from zero
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
#pragma unroll 1
  for (int b = p0; b < p0 + NB && b < nb; ++b)
#pragma unroll
    for (int c = 0; c < KW; ++c) {
      const int kc = k + c;
      if (kc >= k_dim) break;
      double sum = 0.0;
      for (int q = 0; q < f.chunks; ++q) sum += __ldcg(partial + (static_cast<int64_t>(q) * nb + b) * ld_part + kc);
      const int64_t o = static_cast<int64_t>(b) * f.ld + kc;
      const int64_t os = static_cast<int64_t>(b / f.s_div) * f.ld + kc;
      f.ybar[o] = sum;
      if (f.s1) {
        f.gz[o] = sum * f.s1[os];
        if (f.d) f.d[o] = sum * f.s2[os];
      }
    }
}

// ---------------------------------------------------------------------------
// Multi-vector adjoint on the FP64 tensor cores (2 <= nv <= 16 vectors, e.g.
// the m = 10 reverse-mode Jacobian seeds of nn.cpp:148-170):
//   partial[c][v][k] = sum_{i in row chunk c} gz[v][i] W[i][k]
// as skinny DMMA GEMMs, M = 16 vectors (two 8-row blocks), N = 128 columns of
// W per CTA, K = the chunk's rows.  W streams through TMA (8 boxes of 16 x 16
// doubles, 128B-swizzled, per 16-row stage) into a 4-stage mbarrier ring; the
// chunk's gz values sit in shared memory.  Each consumer warp owns one 16-
// column box: per 4-row k-step 2 A fragments (gz), 2 B fragments (W) and 4
// DMMA.8x8x4.  The CUDA-core version does one shared-memory broadcast and
// one DFMA per vector per weight pair and is issue-bound at ~3.3 TB/s; here
// the weight stream is the limit.  The split reduction over chunks is
// adj_reduce_kernel's, in fixed order.
// Two CTAs per SM.  The consumers read W from shared memory with generic
// loads; releasing a stage back to the producer's next TMA write therefore
// needs the async-proxy fence in stage_release -- without it this kernel
// returned wrong partials for ~1-4% of its 8-column blocks (cold launches,
// overlapping handles; tools/adj_mma_conc.cu, profiles/r02_notes.md).
// ---------------------------------------------------------------------------
constexpr int kAmStages = 4;
constexpr int kAmRows = 256;                 // rows per chunk (K of one CTA)
constexpr int kAmStageBytes = 8 * 16 * 16 * 8;  // 8 boxes of 16 x 16 doubles = 16 KB
constexpr int kAmGzPitch = 20;               // gz row pitch (doubles): 2 wavefronts per fragment load
constexpr int kAmSmem = kAmStages * kAmStageBytes + kAmRows * kAmGzPitch * 8 + 1024 + 2 * kAmStages * 8;

__global__ void __launch_bounds__(288, 2)
    adj_mma_kernel(const __grid_constant__ CUtensorMap tmW, int rows, int k_dim, const double* __restrict__ gz,
                   int64_t ld_gz, int nb, int p0, double* __restrict__ partial, int64_t ld_part, int crows) {
  extern __shared__ unsigned char am_raw[];
  char* smem = reinterpret_cast<char*>(am_raw) + ((1024u - (smem_u32(am_raw) & 1023u)) & 1023u);
  double* gzs = reinterpret_cast<double*>(smem + kAmStages * kAmStageBytes);  // [kAmRows][pitch]
  uint64_t* full = reinterpret_cast<uint64_t*>(gzs + kAmRows * kAmGzPitch);
  uint64_t* empty = full + kAmStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * 128;
  const int r0 = blockIdx.y * crows;  // crows <= kAmRows, a multiple of 16
  const int nr = min(crows, rows - r0);
  const int steps = (nr + 15) / 16;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kAmStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 8);
    }
    fence_barrier_init();
  }
  __syncthreads();
  if (warp < 8) {
    // the chunk's gz values, gzs[i][v] (zero past nr or past the vectors),
    // staged by the consumers while the producer's first TMA loads fly; every
    // load of a thread in flight before its stores (a load -> store chain per
    // element made the staging cost more than the chunk's weight stream)
    constexpr int kPer = kAmRows * 16 / 256;
    double v8[kPer];
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int e = u * 256 + threadIdx.x;
      const int i = e >> 4, v = e & 15;
      v8[u] = (i < nr && p0 + v < nb) ? __ldcg(gz + static_cast<int64_t>(p0 + v) * ld_gz + r0 + i) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int e = u * 256 + threadIdx.x;
      gzs[(e >> 4) * kAmGzPitch + (e & 15)] = v8[u];
    }
    asm volatile("bar.sync 1, 256;" ::: "memory");
  }
  if (warp == 8) {
    if (lane == 0) {
      tma_prefetch_desc(&tmW);
      for (int st = 0; st < steps; ++st) {
        const int s = st % kAmStages;
        if (st >= kAmStages) mbar_wait(&empty[s], ((st / kAmStages) - 1) & 1);
        char* dst = smem + s * kAmStageBytes;
        mbar_arrive_expect_tx(&full[s], kAmStageBytes);
#pragma unroll
        for (int b = 0; b < 8; ++b) tma_load_2d(dst + b * 2048, &tmW, &full[s], n0 + 16 * b, r0 + 16 * st);
      }
      // producer tail: stay until the consumers have released every stage,
      // i.e. until every load issued here has landed and been read
      for (int st = (steps > kAmStages ? steps - kAmStages : 0); st < steps; ++st)
        mbar_wait(&empty[st % kAmStages], (st / kAmStages) & 1);
    }
    __syncwarp();
    return;
  }
  const int g = lane >> 2, t = lane & 3;
  double acc[2][2][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  for (int st = 0; st < steps; ++st) {
    const int s = st % kAmStages;
    mbar_wait(&full[s], (st / kAmStages) & 1);
    const char* box = smem + s * kAmStageBytes + warp * 2048;  // this warp's 16 columns
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int il = 4 * q + t;  // row within the stage (k of the DMMA)
      const double* gr = gzs + (16 * st + il) * kAmGzPitch;
      const double a0 = gr[g], a1 = gr[8 + g];
      const double b0 = lds_swz(box, il, g), b1 = lds_swz(box, il, 8 + g);
      dmma884(acc[0][0], a0, b0);
      dmma884(acc[0][1], a0, b1);
      dmma884(acc[1][0], a1, b0);
      dmma884(acc[1][1], a1, b1);
    }
    stage_release(&empty[s], lane);
  }
  // C fragment: thread (g, t) holds C[g][2t], C[g][2t + 1] of each 8 x 8 block
#pragma unroll
  for (int mb = 0; mb < 2; ++mb) {
    const int v = p0 + 8 * mb + g;
    if (v >= nb) continue;
    double* o = partial + (static_cast<int64_t>(blockIdx.y) * nb + v) * ld_part;
#pragma unroll
    for (int nbk = 0; nbk < 2; ++nbk) {
      const int k = n0 + 16 * warp + 8 * nbk + 2 * t;
      if (k < k_dim) o[k] = acc[mb][nbk][0];
      if (k + 1 < k_dim) o[k + 1] = acc[mb][nbk][1];
    }
  }
}

// ybar[b][k] = sum_c partial[c][b][k] (fixed order), then
// gz = ybar .* s1 and d = ybar .* s2 for the layer below (nn.cpp:188-193).
// When s1 == nullptr only ybar is written (the input-gradient).
__global__ void adj_reduce_kernel(const double* __restrict__ partial, int chunks, int64_t ld_part, int k_dim, int nb,
                                  const double* __restrict__ s1, const double* __restrict__ s2, int64_t ld,
                                  double* __restrict__ ybar, double* __restrict__ gz, double* __restrict__ d,
                                  int s_div) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= static_cast<int64_t>(nb) * k_dim) return;
  const int b = static_cast<int>(e / k_dim), k = static_cast<int>(e % k_dim);
  double sum = 0.0;
  for (int c = 0; c < chunks; ++c) sum += partial[(static_cast<int64_t>(c) * nb + b) * ld_part + k];
  const int64_t o = static_cast<int64_t>(b) * ld + k;
  // s_div > 1: b indexes reverse-mode seed vectors, s_div per point
  const int64_t os = static_cast<int64_t>(b / s_div) * ld + k;
  ybar[o] = sum;
  if (s1) {
    gz[o] = sum * s1[os];
    if (d) d[o] = sum * s2[os];
  }
}

// Reverse-mode Jacobian seeds (nn.cpp:148-170): for point p and output i,
// seed vector v = p*m + i is row i of d y_L / d z_L:
//   elementwise: e_i * sigma'_L ;  softmax: y_i (e_i - y)
// written as gz_L[v] (the adjoint chain then yields row i of J at layer 0).
__global__ void jac_seed_kernel(const double* __restrict__ y, const double* __restrict__ s1, int64_t ld, int m,
                                int nb, int softmax, double* __restrict__ gz) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= static_cast<int64_t>(nb) * m * m) return;
  const int p = static_cast<int>(e / (static_cast<int64_t>(m) * m));
  const int i = static_cast<int>((e / m) % m), k = static_cast<int>(e % m);
  double v;
  if (softmax) {
    const double yi = y[ld * p + i];
    v = yi * ((i == k ? 1.0 : 0.0) - y[ld * p + k]);
  } else {
    v = i == k ? s1[ld * p + k] : 0.0;
  }
  gz[(static_cast<int64_t>(p) * m + i) * ld + k] = v;
}

// ---------------------------------------------------------------------------
// Final layer with m <= 16 outputs (tall-skinny NT product):
//   partial[c][b][j][i] = sum_{k in chunk c} A[b][j][k] s[b][k] W[i][k]
// A rows j < n_valid of each point; W is the last layer (m x K, row-major).
// ---------------------------------------------------------------------------
constexpr int kSkMB = 16;      // output slots per row in partial / U
constexpr int kSkRows = 16;    // rows j per CTA (2 per warp)
// K chunk per CTA for MB outputs: 32 KB of staged (scaled) weights at most.
__host__ __device__ constexpr int skinny_kchunk(int mb) { return mb <= 1 ? 1024 : (mb <= 4 ? 512 : 256); }

template <int MB>
__global__ void __launch_bounds__(256)
    skinny_nt_kernel(const double* __restrict__ a, int64_t lda, int64_t a_point_rows, int n_valid,
                     const double* __restrict__ scale, int64_t s_stride, const double* __restrict__ w, int64_t ldw,
                     int m, int k_dim, double* __restrict__ partial) {
  constexpr int kSkKChunk = skinny_kchunk(MB);
  __shared__ __align__(16) double ws[MB][kSkKChunk];
  const int point = blockIdx.z;
  const int chunk = blockIdx.y;
  const int k0 = chunk * kSkKChunk;
  const int kc = min(kSkKChunk, k_dim - k0);
  const double* sp = scale ? scale + s_stride * point : nullptr;
  for (int e = threadIdx.x; e < MB * kSkKChunk; e += blockDim.x) {
    const int i = e / kSkKChunk, k = e % kSkKChunk;
    double v = 0.0;
    if (i < m && k < kc) {
      v = w[static_cast<int64_t>(i) * ldw + k0 + k];
      if (sp) v *= sp[k0 + k];
    }
    ws[i][k] = v;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j0 = blockIdx.x * kSkRows + warp * 2;
  double acc[2][MB];
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int i = 0; i < MB; ++i) acc[r][i] = 0.0;
  const double* a0 = a + (a_point_rows * point + j0) * lda + k0;
  const bool live0 = j0 < n_valid, live1 = j0 + 1 < n_valid;
  for (int k = 2 * lane; k < kc; k += 64) {
    const double2 x0 = live0 ? *reinterpret_cast<const double2*>(a0 + k) : make_double2(0.0, 0.0);
    const double2 x1 = live1 ? *reinterpret_cast<const double2*>(a0 + lda + k) : make_double2(0.0, 0.0);
#pragma unroll
    for (int i = 0; i < MB; ++i) {
      const double2 wv = *reinterpret_cast<const double2*>(&ws[i][k]);
      acc[0][i] = fma(x0.x, wv.x, fma(x0.y, wv.y, acc[0][i]));
      acc[1][i] = fma(x1.x, wv.x, fma(x1.y, wv.y, acc[1][i]));
    }
  }
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int i = 0; i < MB; ++i) {
      double v = acc[r][i];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      acc[r][i] = v;
    }
  // lane i writes output i of both rows: partial layout [chunk][point][rows_pad][16]
  const int64_t rows_pad = static_cast<int64_t>(gridDim.x) * kSkRows;
  const int64_t base = (static_cast<int64_t>(chunk) * gridDim.z + point) * rows_pad;
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    double v = 0.0;
#pragma unroll
    for (int i = 0; i < MB; ++i)
      if (i == lane) v = acc[r][i];
    if (lane < MB) partial[(base + j0 + r) * kSkMB + lane] = v;
  }
}

// U[b][j][i] = sum_c partial[c][b][j][i]   (deterministic order)
// jac != nullptr (elementwise final activation): also J[b][i][j] = s1_i U_ji,
// jacobian_out_kernel's product, folded in (one launch less on the J path).
__global__ void skinny_reduce_kernel(const double* __restrict__ partial, int chunks, int nb, int rows_pad, int m,
                                     double* __restrict__ u, double* __restrict__ jac, const double* __restrict__ s1,
                                     int64_t ld, int n) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t per_point = static_cast<int64_t>(rows_pad) * kSkMB;
  if (e >= per_point * nb) return;
  double sum = 0.0;
  for (int c = 0; c < chunks; ++c) sum += partial[static_cast<int64_t>(c) * nb * per_point + e];
  u[e] = sum;
  if (jac) {
    const int b = static_cast<int>(e / per_point);
    const int j = static_cast<int>((e % per_point) / kSkMB), i = static_cast<int>(e % kSkMB);
    if (i < m && j < n) jac[(static_cast<int64_t>(b) * m + i) * n + j] = s1[ld * b + i] * sum;
  }
}

// J[b][i][j] from U = dz_L/dx^T (rows j, cols i, pitch ldu):
//   elementwise final: J_ij = s1_i U_ji
//   softmax final:     J_ij = y_i U_ji - y_i sum_k y_k U_jk
__global__ void jacobian_out_kernel(const double* __restrict__ u, int64_t ldu, int64_t u_point_rows,
                                    const double* __restrict__ s1, const double* __restrict__ y, int64_t ld, int n,
                                    int m, int nb, int softmax, double* __restrict__ jac) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= static_cast<int64_t>(nb) * n) return;
  const int b = static_cast<int>(e / n), j = static_cast<int>(e % n);
  const double* ur = u + (u_point_rows * b + j) * ldu;
  double* jb = jac + static_cast<int64_t>(b) * m * n;
  if (!softmax) {
    for (int i = 0; i < m; ++i) jb[static_cast<int64_t>(i) * n + j] = s1[ld * b + i] * ur[i];
  } else {
    const double* yr = y + ld * b;
    double dot = 0.0;
    for (int k = 0; k < m; ++k) dot += yr[k] * ur[k];
    for (int i = 0; i < m; ++i) jb[static_cast<int64_t>(i) * n + j] = yr[i] * ur[i] - yr[i] * dot;
  }
}

// Final-layer curvature with a small K = m:
//   H[b][r][c] += sum_{i,k} U[r][i] M[i][k] U[c][k]
// with M = diag(d) (elementwise) or the dense softmax middle.  Only the
// lower triangle (c <= r) is needed; the symmetrise pass mirrors it.
__global__ void small_k_syrk_kernel(const double* __restrict__ u, int64_t ldu, int64_t u_point_rows,
                                    const double* __restrict__ dvec, int64_t ld, const double* __restrict__ mid,
                                    int64_t ld_mid, int n, int m, int nb, double* __restrict__ h,
                                    int64_t h_point_stride, int64_t ldh) {
  const int b = blockIdx.z;
  const int r = blockIdx.y * blockDim.y + threadIdx.y;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n || c >= n || c > r || b >= nb) return;
  const double* ur = u + (u_point_rows * b + r) * ldu;
  const double* uc = u + (u_point_rows * b + c) * ldu;
  double sum = 0.0;
  if (mid == nullptr) {
    const double* dv = dvec + ld * b;
    for (int i = 0; i < m; ++i) sum += ur[i] * dv[i] * uc[i];
  } else {
    const double* mm = mid + ld_mid * b;
    for (int i = 0; i < m; ++i) {
      double t = 0.0;
      for (int k = 0; k < m; ++k) t += mm[i * m + k] * uc[k];
      sum += ur[i] * t;
    }
  }
  h[h_point_stride * b + static_cast<int64_t>(r) * ldh + c] += sum;
}

// H_out[b][r][c] = sum_i H_i[b][max(r,c)][min(r,c)] over the (up to three)
// lower-triangle accumulators, in a fixed order: exactly symmetric output.
__global__ void symmetrize_out_kernel(const double* __restrict__ hws, const double* __restrict__ h1,
                                      const double* __restrict__ h2, int64_t h_point_stride, int64_t ldh, int n,
                                      int nb, double* __restrict__ out) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nn = static_cast<int64_t>(n) * n;
  if (e >= nn * nb) return;
  const int b = static_cast<int>(e / nn);
  const int r = static_cast<int>((e % nn) / n), c = static_cast<int>(e % n);
  const int hi = r > c ? r : c, lo = r > c ? c : r;
  const int64_t o = h_point_stride * b + static_cast<int64_t>(hi) * ldh + lo;
  double v = hws[o];
  if (h1) v += h1[o];
  if (h2) v += h2[o];
  out[e] = v;
}

// Small batches (points x square tiles < SMs: every layer's SYRK is split
// over k) keep each layer's split partials in its own buffer instead of
// reducing them into H per layer; this kernel sums them once -- layers in
// order, each layer's slices in ascending order first, then the direct
// final-layer term hws (nullable), i.e. the additions of the per-layer
// reduce + symmetrise path in the same order, bit-identical -- and writes
// the symmetric H (or its packed lower rows).  Two layers' SYRKs can then
// run concurrently on different streams, and the per-layer reduce launches
// leave the critical path.  Block (bx <= by) of 32 x 8 threads: the 32 x 32
// lower block (by, bx) and, through shared memory, its mirror.
constexpr int kMaxGather = 8;
struct SyrkGather {
  const double* part[kMaxGather];  // [split][points][n_tiles][kBM][kBN] per layer
  int split[kMaxGather];
  int nseg;
  int n_tiles;  // square lower tiles per point (tile id tm (tm + 1) / 2 + tn)
  int points;
};
__global__ void __launch_bounds__(256) syrk_gather_out_kernel(SyrkGather g, const double* __restrict__ hws,
                                                              int64_t h_point_stride, int64_t ldh, int n, int packed,
                                                              double* __restrict__ out) {
  const int bx = blockIdx.x, by = blockIdx.y, b = blockIdx.z;
  if (bx > by) return;
  __shared__ double tile[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t nn = static_cast<int64_t>(n) * n;
  const int64_t slice = static_cast<int64_t>(g.points) * g.n_tiles * (kBM * kBN);
  // this thread's four elements (rows ty, ty + 8, ...): all loads of a
  // split chunk for the four rows in flight before their adds (each
  // element's additions keep the ascending layer / slice order)
  int64_t off[4];
  bool live[4];
  double v[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = by * 32 + ty + 8 * i, c = bx * 32 + tx;
    live[i] = r < n && c <= r;
    const int tm = live[i] ? r / kBM : 0, tn = live[i] ? c / kBM : 0;
    off[i] = live[i] ? (static_cast<int64_t>(b) * g.n_tiles + tm * (tm + 1) / 2 + tn) * (kBM * kBN) +
                           (r % kBM) * kBN + (c % kBM)
                     : 0;
    v[i] = 0.0;
  }
  for (int q = 0; q < g.nseg; ++q) {
    const double* base = g.part[q];
    const int sp = g.split[q];
    double t[4] = {0.0, 0.0, 0.0, 0.0};
    int s = 0;
    for (; s + 4 <= sp; s += 4) {
      double a[4][4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int i = 0; i < 4; ++i) a[u][i] = live[i] ? __ldcg(base + slice * (s + u) + off[i]) : 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int i = 0; i < 4; ++i) t[i] += a[u][i];
    }
    for (; s < sp; ++s)
#pragma unroll
      for (int i = 0; i < 4; ++i) t[i] += live[i] ? __ldcg(base + slice * s + off[i]) : 0.0;
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] += t[i];
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int ry = ty + 8 * i, r = by * 32 + ry, c = bx * 32 + tx;
    if (live[i]) {
      if (hws) v[i] += hws[h_point_stride * b + static_cast<int64_t>(r) * ldh + c];
      if (packed)
        out[static_cast<int64_t>(b) * n * (n + 1) / 2 + static_cast<int64_t>(r) * (r + 1) / 2 + c] = v[i];
      else
        out[nn * b + static_cast<int64_t>(r) * n + c] = v[i];
    }
    tile[ry][tx] = v[i];
  }
  if (packed) return;
  __syncthreads();
  for (int ry = ty; ry < 32; ry += 8) {
    const int r = bx * 32 + ry, c = by * 32 + tx;  // strict upper element (r, c) = H(c, r)
    if (c < n && c > r) out[nn * b + static_cast<int64_t>(r) * n + c] = tile[tx][ry];
  }
}

// dst[b][r][c] = src[b * src_point_rows + r][c] * scale[b * s_stride + c]
// for b < nb, r < rows, c < cols (S_0 = T_0 diag(sigma'_0) per point).
// Grid: x over columns, y strides over b * rows + r (gridDim.y <= 65535).
__global__ void scale_cols_kernel(const double* __restrict__ src, int64_t lds, int64_t src_point_rows, int rows,
                                  int cols, const double* __restrict__ scale, int64_t s_stride,
                                  double* __restrict__ dst, int64_t ldd, int64_t dst_point_rows, int nb) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  for (int64_t y = blockIdx.y; y < static_cast<int64_t>(nb) * rows; y += gridDim.y) {
    const int b = static_cast<int>(y / rows), r = static_cast<int>(y % rows);
    dst[(dst_point_rows * b + r) * ldd + c] = src[(src_point_rows * b + r) * lds + c] * scale[s_stride * b + c];
  }
}

// Strided copy of a [rows][cols] block (pitch src -> pitch dst).
__global__ void copy_rows_kernel(const double* __restrict__ src, int64_t lds, double* __restrict__ dst, int64_t ldd,
                                 int rows, int cols) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= static_cast<int64_t>(rows) * cols) return;
  const int r = static_cast<int>(e / cols), c = static_cast<int>(e % cols);
  dst[static_cast<int64_t>(r) * ldd + c] = src[static_cast<int64_t>(r) * lds + c];
}

}  // namespace dev
}  // namespace gbb
