// OPT-IN (GBOPT_FWD_STREAM=1), not the default: measured slower than the
// per-layer GEMV launches of the CUDA graph on every BASELINE shape (device
// time, CUDA events: c2 165 vs 155 us, c5 130 vs 80 us, c1 ~45 vs ~35 us;
// profiles/r02_fwd_stream.md).  The inter-layer barrier (CTA barrier,
// release/acquire round trip, epilogue) costs ~2.4 us per layer, more than the
// graph's kernel boundaries, and one CTA per SM with a 5-stage TMA ring reads
// no faster than 8 warps of 16-byte loads per row.  Kept as a measured
// alternative.
//
// Forward pass of one point through the whole network in ONE persistent
// launch (the line-search residual and forward_trace, reference
// nn.cpp:113-146 / ipm.cpp:342-343): every layer is an HBM-bound GEMV, so
// the launch is built to keep the weight stream running end to end.
//
//  * one CTA per SM (cooperative launch), 1 producer warp + 8 consumer warps;
//  * layer l's rows are split into contiguous ranges, one per CTA, so a
//    CTA's weights of a layer are ONE contiguous byte range (row-major W,
//    pitch ldw): the producer streams it with 1-D TMA bulk copies
//    (cp.async.bulk, 40 KB chunks = whole rows, or row segments for rows
//    wider than a chunk) into a 5-stage shared-memory ring guarded by
//    full / empty mbarriers;
//  * the producer never waits on the layer dependency: it runs straight on
//    into the next layer's rows while the consumers finish the current
//    layer and wait at the inter-layer barrier, so the HBM stream does not
//    drain at layer boundaries (no launch gaps, no ramp-up per layer);
//  * consumers: warp w takes a fixed 1/8 k-slice of every row in a chunk
//    and accumulates its partial dot product in shared memory; at the end
//    of the layer the 8 partials of each row are summed in warp order
//    (deterministic), the bias and the activation with sigma', sigma'' are
//    applied (the same epilogue as fwd_row1_kernel), and z, y, s1, s2 go to
//    the workspace;
//  * inter-layer barrier among the consumer warps only (one arrival counter
//    per layer, release/acquire at gpu scope); each warp then loads its
//    k-slice of y_l into registers for layer l + 1 (whole-row chunks), so the
//    ring gets all of shared memory (5 x 40 KB) to keep loads in flight
//    across the barrier.
#pragma once

#include <cstdint>

namespace gbb {
namespace dev {

constexpr int kFsConsumerWarps = 8;
constexpr int kFsThreads = (kFsConsumerWarps + 1) * 32;
constexpr int kFsStages = 5;
constexpr int kFsYRegs = 16;  // double2 per lane: a warp's input slice up to 16 x 64 doubles
constexpr int kFsStageBytes = 40960;  // one 5120-wide FP64 row
constexpr int kFsMaxLayers = 48;

struct FsLayer {
  const double* w;  // [rows][ldw], row-major, zero-padded columns
  const double* b;
  double *z, *y, *s1, *s2;
  int rows, cols, ldw, act;
};

struct FsParams {
  FsLayer L[kFsMaxLayers];
  const double* x;     // layer 0's input
  unsigned* arrive;    // [nl] per-layer arrival counters, never reset: launch number
                       // `gen` (1, 2, ...) waits for gen * gridDim.x arrivals
  unsigned gen;
  int nl;
  int max_cta_rows;    // partial-sum rows per CTA
  int ycap;            // y staging capacity (doubles, even)
};

// chunk geometry of (layer, CTA): rows [r0, r1); a chunk holds `spr` whole
// rows, or (spr == 0) one segment of `seg` doubles of a row
struct FsGeom {
  int r0, r1, spr, seg, nseg, nchunks;
};

__device__ __forceinline__ FsGeom fs_geom(const FsLayer& L, int cta, int ncta) {
  FsGeom g;
  g.r0 = static_cast<int>(static_cast<int64_t>(L.rows) * cta / ncta);
  g.r1 = static_cast<int>(static_cast<int64_t>(L.rows) * (cta + 1) / ncta);
  const int rowbytes = L.ldw * 8;
  const int n = g.r1 - g.r0;
  if (rowbytes <= kFsStageBytes) {
    g.spr = kFsStageBytes / rowbytes;
    g.seg = L.ldw;
    g.nseg = 1;
    g.nchunks = (n + g.spr - 1) / g.spr;
  } else {
    g.spr = 0;
    g.seg = kFsStageBytes / 8;
    g.nseg = (L.ldw + g.seg - 1) / g.seg;
    g.nchunks = n * g.nseg;
  }
  return g;
}

__device__ __forceinline__ void fs_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "FSW_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra FSW_%=;\n}" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(bar))),
      "r"(parity)
      : "memory");
}

__global__ void __launch_bounds__(kFsThreads, 1) fwd_stream_kernel(const __grid_constant__ FsParams p) {
  extern __shared__ __align__(128) unsigned char fs_smem[];
  double* stage = reinterpret_cast<double*>(fs_smem);
  double* part = reinterpret_cast<double*>(fs_smem + kFsStages * kFsStageBytes);  // [max_cta_rows][warps]
  uint64_t* full = reinterpret_cast<uint64_t*>(part + static_cast<int64_t>(p.max_cta_rows) * kFsConsumerWarps);
  uint64_t* empty = full + kFsStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cta = blockIdx.x, ncta = gridDim.x;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kFsStages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(full + s))));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(empty + s))),
                   "r"(kFsConsumerWarps));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kFsConsumerWarps) {
    // ---- producer: every layer's weight range of this CTA, chunk by chunk
    if (lane == 0) {
      int g = 0;  // global chunk counter (ring position)
      for (int l = 0; l < p.nl; ++l) {
        const FsLayer& L = p.L[l];
        const FsGeom G = fs_geom(L, cta, ncta);
        const char* base = reinterpret_cast<const char*>(L.w) + static_cast<int64_t>(G.r0) * L.ldw * 8;
        for (int q = 0; q < G.nchunks; ++q, ++g) {
          const int s = g % kFsStages;
          if (g >= kFsStages) fs_wait(empty + s, ((g / kFsStages) - 1) & 1);
          int64_t off;
          uint32_t bytes;
          if (G.spr > 0) {
            const int rr = q * G.spr;
            const int nr = min(G.spr, G.r1 - G.r0 - rr);
            off = static_cast<int64_t>(rr) * L.ldw * 8;
            bytes = static_cast<uint32_t>(nr) * L.ldw * 8;
          } else {
            const int rr = q / G.nseg, sg = q % G.nseg;
            const int k0 = sg * G.seg;
            off = (static_cast<int64_t>(rr) * L.ldw + k0) * 8;
            bytes = static_cast<uint32_t>(min(G.seg, L.ldw - k0)) * 8;
          }
          const uint32_t fb = static_cast<uint32_t>(__cvta_generic_to_shared(full + s));
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "r"(bytes) : "memory");
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  static_cast<uint32_t>(__cvta_generic_to_shared(reinterpret_cast<char*>(stage) + s * kFsStageBytes))),
              "l"(base + off), "r"(bytes), "r"(fb)
              : "memory");
        }
      }
      // producer tail: stay until the consumers have released the last
      // stages (no issuing thread exits with bulk copies in flight)
      for (int g2 = g > kFsStages ? g - kFsStages : 0; g2 < g; ++g2)
        fs_wait(empty + g2 % kFsStages, (g2 / kFsStages) & 1);
    }
    __syncwarp();
    return;
  }

  // ---- consumers (256 threads) ----
  const int ct = threadIdx.x;  // 0..255
  int g = 0;
  for (int l = 0; l < p.nl; ++l) {
    const FsLayer& L = p.L[l];
    const FsGeom G = fs_geom(L, cta, ncta);
    const int nrows = G.r1 - G.r0;
    const double* yin = l == 0 ? p.x : p.L[l - 1].y;
    // this warp's partial column of the layer's rows starts at 0 (only warp
    // w ever touches column w: no CTA barrier needed)
    for (int i = lane; i < nrows; i += 32) part[i * kFsConsumerWarps + warp] = 0.0;
    // Whole-row chunks: the warp's k-slice is the same for every row, so its
    // slice of the input vector lives in registers, loaded once per layer
    // straight from L2 with every load in flight (the previous layer's y was
    // written by other CTAs: ld.cg after the barrier's acquire).
    const int steps_row = (L.ldw + 63) / 64;
    const int wst0 = steps_row * warp / kFsConsumerWarps, wst1 = steps_row * (warp + 1) / kFsConsumerWarps;
    const bool yreg = G.spr > 0 && wst1 - wst0 <= kFsYRegs;
    double2 yr[kFsYRegs];
#pragma unroll
    for (int u = 0; u < kFsYRegs; ++u) {
      const int k = (wst0 + u) * 64 + 2 * lane;
      yr[u] = make_double2(0.0, 0.0);
      if (yreg && wst0 + u < wst1) {
        if (k < L.cols) yr[u].x = __ldcg(yin + k);
        if (k + 1 < L.cols) yr[u].y = __ldcg(yin + k + 1);
      }
    }
    __syncwarp();
    for (int q = 0; q < G.nchunks; ++q, ++g) {
      const int s = g % kFsStages;
      fs_wait(full + s, (g / kFsStages) & 1);
      const double* sb = stage + s * (kFsStageBytes / 8);
      if (yreg) {
        const int rr0 = q * G.spr;
        const int nr = min(G.spr, nrows - rr0);
        for (int r = 0; r < nr; ++r) {
          const double* wr = sb + static_cast<int64_t>(r) * L.ldw;
          double a0 = 0.0, a1 = 0.0;
#pragma unroll
          for (int u = 0; u < kFsYRegs; ++u) {
            const int k = (wst0 + u) * 64 + 2 * lane;
            if (wst0 + u < wst1 && k < L.ldw) {
              const double2 wv = *reinterpret_cast<const double2*>(wr + k);
              a0 = fma(wv.x, yr[u].x, a0);
              a1 = fma(wv.y, yr[u].y, a1);
            }
          }
          double v = a0 + a1;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
          if (lane == 0) part[(rr0 + r) * kFsConsumerWarps + warp] += v;
        }
      } else {
        // row segments (rows wider than a chunk) or very wide whole rows:
        // the input slice comes from L2 with the weights
        int rr0, nr, k0, len, pitch;
        if (G.spr > 0) {
          rr0 = q * G.spr;
          nr = min(G.spr, nrows - rr0);
          k0 = 0;
          len = L.ldw;
          pitch = L.ldw;
        } else {
          rr0 = q / G.nseg;
          nr = 1;
          k0 = (q % G.nseg) * G.seg;
          len = min(G.seg, L.ldw - k0);
          pitch = len;
        }
        const int steps = (len + 63) / 64;
        const int st0 = steps * warp / kFsConsumerWarps, st1 = steps * (warp + 1) / kFsConsumerWarps;
        for (int r = 0; r < nr; ++r) {
          const double* wr = sb + static_cast<int64_t>(r) * pitch;
          double a0 = 0.0, a1 = 0.0;
          for (int t = st0; t < st1; ++t) {
            const int k = t * 64 + 2 * lane;
            if (k < len) {
              const double2 wv = *reinterpret_cast<const double2*>(wr + k);
              const int kk = k0 + k;
              const double x0 = kk < L.cols ? __ldcg(yin + kk) : 0.0;
              const double x1 = kk + 1 < L.cols ? __ldcg(yin + kk + 1) : 0.0;
              a0 = fma(wv.x, x0, a0);
              a1 = fma(wv.y, x1, a1);
            }
          }
          double v = a0 + a1;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
          if (lane == 0) part[(rr0 + r) * kFsConsumerWarps + warp] += v;
        }
      }
      stage_release(empty + s, lane);  // cross-proxy WAR fence, then arrive (kernels.cuh)
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kFsConsumerWarps * 32) : "memory");
    // epilogue: fixed-order sum of the 8 partials, bias, activation
    for (int i = ct; i < nrows; i += kFsConsumerWarps * 32) {
      double v = 0.0;
#pragma unroll
      for (int w8 = 0; w8 < kFsConsumerWarps; ++w8) v += part[i * kFsConsumerWarps + w8];
      const int row = G.r0 + i;
      const double zz = v + L.b[row];
      double yy, d1, d2;
      act_eval(L.act, zz, yy, d1, d2);
      L.z[row] = zz;
      L.y[row] = yy;
      L.s1[row] = d1;
      L.s2[row] = d2;
    }
    if (l + 1 < p.nl) {
      // inter-layer barrier over the consumer groups of every CTA: the CTA
      // barrier orders this CTA's y writes before thread 0's release (which
      // is cumulative), the acquire + CTA barrier orders the other CTAs'
      // writes before the next layer's loads
      asm volatile("bar.sync 1, %0;" ::"n"(kFsConsumerWarps * 32) : "memory");
      if (ct == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p.arrive + l) : "memory");
        unsigned seen = 0;
        do {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(p.arrive + l) : "memory");
        } while (seen < p.gen * static_cast<unsigned>(ncta));
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kFsConsumerWarps * 32) : "memory");
    }
  }
}

}  // namespace dev
}  // namespace gbb
