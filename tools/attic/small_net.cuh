// Single-point evaluation of SMALL nets (round 2): the forward chain and the
// lambda-adjoint chain each as ONE launch of one 16-CTA cluster, instead of
// one GEMV launch per layer (forward) and seed + sweep + reduction launches
// per layer (adjoint).  For nets like BASELINE c1 (784-512-512-10, 5.4 MB of
// weights, L2-resident between IPM iterations) the evaluation is a chain of
// ~18 dependent launches of a few microseconds each; the per-layer launches
// of the forward and adjoint were 8 of them.  Same outputs, same buffers as
// fwd_row1_kernel / adj_seed_kernel / adj_cols_kernel + adj_reduce_kernel
// (nn.cpp:113-146 forward and trace, nn.cpp:172-196 adjoint), with fixed
// summation orders (deterministic):
//   forward  z_l = W_l y_{l-1} + b_l, y_l = sigma(z_l), s1 = sigma', s2 = sigma''
//            -- warp per row, rows spread over the cluster's 256 warps, the
//            input vector staged in every CTA's shared memory, one cluster
//            barrier per layer (global writes are visible cluster-wide after
//            barrier.cluster's release / acquire);
//   adjoint  gz_{L-1} = lambda .* s1_{L-1}, d_{L-1} = lambda .* s2_{L-1}, then
//            per layer ybar_{l-1} = W_l^T gz_l: CTA c sums its row chunk for
//            every column into shared memory, one cluster barrier, CTA c adds
//            the 16 partials of its column block over DSMEM in rank order and
//            writes ybar, gz = ybar .* s1, d = ybar .* s2 (or the gradient at
//            layer 0).
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.cuh"

namespace gbb {
namespace dev {

namespace cgs = cooperative_groups;

constexpr int kSnCtas = 16;       // cluster size (non-portable: set the attribute)
constexpr int kSnThreads = 512;
constexpr int kSnWarps = kSnThreads / 32;
constexpr int kSnMaxL = 8;        // layers
constexpr int kSnMaxWidth = 4096; // widest layer input / output

struct SnLayer {
  const double* w;  // [rows][ldw]
  int64_t ldw;
  const double* b;
  int rows, cols, act;
  double *z, *y, *s1, *s2;  // forward outputs [rows]
  double *ybar, *gz, *d;    // adjoint quantities at this layer's output [rows] (ybar, ybar .* s1, ybar .* s2)
};

struct SnParams {
  int L;
  int lstop;  // the adjoint stops after layer lstop (1: no input gradient)
  const double* x;
  const double* lam;
  double* grad;  // the input gradient (lstop == 0)
  SnLayer ly[kSnMaxL];
};

// dynamic shared memory: the staged vector + the column partials
constexpr int kSnSmem = 2 * kSnMaxWidth * 8;

__global__ void __cluster_dims__(kSnCtas, 1, 1) __launch_bounds__(kSnThreads, 1)
    small_fwd_kernel(const __grid_constant__ SnParams p) {
  extern __shared__ __align__(16) double sn_smem[];
  double* vs = sn_smem;  // the layer's input vector
  cgs::cluster_group cluster = cgs::this_cluster();
  const int rank = static_cast<int>(cluster.block_rank());
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = rank * kSnWarps + warp;
  for (int l = 0; l < p.L; ++l) {
    const SnLayer& ly = p.ly[l];
    const double* in = l == 0 ? p.x : p.ly[l - 1].y;
    for (int k = threadIdx.x; k < ly.cols; k += kSnThreads) vs[k] = __ldcg(in + k);
    __syncthreads();
    for (int r = gw; r < ly.rows; r += kSnCtas * kSnWarps) {
      const double* wr = ly.w + static_cast<int64_t>(r) * ly.ldw;
      double a0 = 0.0, a1 = 0.0;
      int k = 2 * lane;
      for (; k + 65 < ly.cols; k += 128) {  // two 16-byte loads per lane in flight
        const double2 w0 = __ldg(reinterpret_cast<const double2*>(wr + k));
        const double2 w1 = __ldg(reinterpret_cast<const double2*>(wr + k + 64));
        a0 = fma(w0.x, vs[k], a0);
        a1 = fma(w0.y, vs[k + 1], a1);
        a0 = fma(w1.x, vs[k + 64], a0);
        a1 = fma(w1.y, vs[k + 65], a1);
      }
      for (; k < ly.cols; k += 64) {
        const double2 w0 = __ldg(reinterpret_cast<const double2*>(wr + k));
        a0 = fma(w0.x, vs[k], a0);
        if (k + 1 < ly.cols) a1 = fma(w0.y, vs[k + 1], a1);
      }
      double v = a0 + a1;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) {
        const double zz = v + ly.b[r];
        double yy, d1, d2;
        act_eval(ly.act, zz, yy, d1, d2);
        ly.z[r] = zz;
        ly.y[r] = yy;
        ly.s1[r] = d1;
        ly.s2[r] = d2;
      }
    }
    cluster.sync();  // y_l complete and visible in every CTA of the cluster
  }
}

__global__ void __cluster_dims__(kSnCtas, 1, 1) __launch_bounds__(kSnThreads, 1)
    small_adj_kernel(const __grid_constant__ SnParams p) {
  extern __shared__ __align__(16) double sn_smem[];
  double* gs = sn_smem;                 // gz of the current layer [rows]
  double* part = sn_smem + kSnMaxWidth;  // this CTA's column partials [cols]
  cgs::cluster_group cluster = cgs::this_cluster();
  const int rank = static_cast<int>(cluster.block_rank());
  const int L = p.L;
  const SnLayer& last = p.ly[L - 1];
  // seed (adj_seed_kernel's elementwise branch), every CTA its own copy
  for (int i = threadIdx.x; i < last.rows; i += kSnThreads) {
    const double g = p.lam[i] * last.s1[i];
    gs[i] = g;
    if (rank == 0) {
      last.gz[i] = g;
      last.d[i] = p.lam[i] * last.s2[i];
    }
  }
  __syncthreads();
  for (int l = L - 1; l >= p.lstop; --l) {
    const SnLayer& ly = p.ly[l];
    const int rows = ly.rows, cols = ly.cols;
    const int chunk = (rows + kSnCtas - 1) / kSnCtas;
    const int r0 = rank * chunk, r1 = min(rows, r0 + chunk);
    // column partials of this CTA's rows: threads own 2 adjacent columns
    for (int k = 2 * static_cast<int>(threadIdx.x); k < cols; k += 2 * kSnThreads) {
      double a0 = 0.0, a1 = 0.0;
      int r = r0;
      for (; r + 1 < r1; r += 2) {
        const double2 w0 = __ldg(reinterpret_cast<const double2*>(ly.w + static_cast<int64_t>(r) * ly.ldw + k));
        const double2 w1 = __ldg(reinterpret_cast<const double2*>(ly.w + static_cast<int64_t>(r + 1) * ly.ldw + k));
        a0 = fma(w0.x, gs[r], a0);
        a1 = fma(w0.y, gs[r], a1);
        a0 = fma(w1.x, gs[r + 1], a0);
        a1 = fma(w1.y, gs[r + 1], a1);
      }
      if (r < r1) {
        const double2 w0 = __ldg(reinterpret_cast<const double2*>(ly.w + static_cast<int64_t>(r) * ly.ldw + k));
        a0 = fma(w0.x, gs[r], a0);
        a1 = fma(w0.y, gs[r], a1);
      }
      part[k] = a0;
      if (k + 1 < cols) part[k + 1] = a1;
    }
    cluster.sync();  // every CTA's partials are complete
    // this CTA's column block: the 16 partials in rank order
    const int cb = (cols + kSnCtas - 1) / kSnCtas;
    const int k0 = rank * cb, k1 = min(cols, k0 + cb);
    const SnLayer* prev = l > 0 ? &p.ly[l - 1] : nullptr;
    for (int k = k0 + static_cast<int>(threadIdx.x); k < k1; k += kSnThreads) {
      double s = 0.0;
#pragma unroll 4
      for (int c = 0; c < kSnCtas; ++c) s += *cluster.map_shared_rank(part + k, c);
      if (prev) {
        prev->ybar[k] = s;
        prev->gz[k] = s * prev->s1[k];
        prev->d[k] = s * prev->s2[k];
      } else {
        p.grad[k] = s;  // layer 0: the input gradient
      }
    }
    cluster.sync();  // gz_{l-1} complete; the partials may be overwritten
    if (l - 1 >= p.lstop) {
      for (int i = threadIdx.x; i < cols; i += kSnThreads) gs[i] = __ldcg(prev->gz + i);
      __syncthreads();
    }
  }
}

}  // namespace dev
}  // namespace gbb
