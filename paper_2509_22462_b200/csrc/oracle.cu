// Device-resident network and the oracle launch sequence.
//
// One oracle evaluation at B points (shared weights) =
//   1. forward chain       z_l, y_l, sigma'_l, sigma''_l        (fwd_rows)
//   2. adjoint chain       ybar_l, gz_l, d_l = ybar_l .* sigma''_l (adj_*)
//   3. tangent chain       T_0 = W_0^T (constant, uploaded once)
//                          T_{l+1} = T_l diag(sigma'_l) W_{l+1}^T (nt_mma)
//      Hessian            H += T_l diag(d_l) T_l^T  per nonlinear layer
//                          (nt_mma in SYRK mode, lower tiles)
//   4. final layer         U = dz_L/dx^T (skinny or nt_mma), J, curvature
//   5. symmetrise          H_out = mirror(lower(H_ws))
//
// This restates the reference's lagrangian_hessian (src/nn.cpp:198-292)
// as H = sum_l (dz_l/dx)^T diag(ybar_l .* sigma''(z_l)) (dz_l/dx) (+ the
// dense softmax middle on a softmax output layer): the same second
// derivative, computed as a SYRK on the forward tangents instead of a
// second (reverse) tangent sweep -- about half the flops, and the
// asymmetry check of nn.cpp:284-290 is satisfied by construction.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <queue>
#include <string>
#include <tuple>
#include <vector>

#include "dataflow.cuh"
#include "device_net.hpp"
#include "multi.hpp"
#include "kernels.cuh"
#include "fwd_stream.cuh"
#include "net.hpp"

namespace gbb {

using dev::kBK;
using dev::kBM;
using dev::kBN;
using dev::round_up;

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw DeviceError(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}
#define CK(x) cuda_check((x), #x)

namespace {

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess || p == nullptr)
      throw DeviceError("cuTensorMapEncodeTiled is unavailable (driver too old?)");
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

// 2-D FP64 tensor [rows][cols] with row pitch `pitch` doubles; box 16 x box_rows,
// 128-byte swizzle, out-of-bounds elements read as zero.
CUtensorMap make_tmap(const double* base, int64_t cols, int64_t rows, int64_t pitch, int box_rows) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(pitch * 8)};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(kBK), static_cast<cuuint32_t>(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box,
                           estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw DeviceError("cuTensorMapEncodeTiled failed: " + std::to_string(static_cast<int>(r)));
  return m;
}

int ceil_div(int64_t a, int64_t b) { return static_cast<int>((a + b - 1) / b); }
// CTAs per tile of the split-K GEMM reduction (single-point GEMMs, c1):
// 14 x 256 threads take 4 of the tile's 14336 elements each
constexpr int kGemmReduceX = 14;

// Several DeviceNets may run on host threads at once (multi-device calls,
// multi.cpp; or a caller's own threads with distinct handles).  Graph
// capture, and the allocation / device-wide synchronisation that first calls
// of a shape do, must not interleave across threads (a cudaMalloc / cudaFree /
// cudaDeviceSynchronize while another thread captures fails that capture), so
// they take this process-wide lock.  Steady-state calls (graph launches) do
// not.
std::recursive_mutex& setup_mutex() {
  static std::recursive_mutex m;
  return m;
}

// From this many points on, the forward and adjoint chains run as DMMA GEMMs
// over the batch instead of GEMV sweeps.
constexpr int kBatchGemm = 32;

}  // namespace

// ---------------------------------------------------------------------------
// DeviceNet: weights in HBM, workspace, launch sequence.
// ---------------------------------------------------------------------------
DeviceNet::DeviceNet(const Net& net, int ordinal) : net_(net), ordinal_(ordinal) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    cudaGetLastError();
    throw DeviceError("no CUDA device available");
  }
  if (ordinal < 0 || ordinal >= count) throw DeviceError("CUDA device ordinal out of range");
  DeviceGuard g(ordinal_);
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, ordinal_));
  if (prop.major != 10) throw DeviceError(std::string("gbopt_b200 needs an sm_100 (B200) device, found ") + prop.name);
  sm_count_ = prop.multiProcessorCount;
  CK(cudaFuncSetAttribute(dev::nt_mma_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, dev::kSmemBytes));
  CK(cudaFuncSetAttribute(dev::nt_mma_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, dev::kSmemBytes));
  CK(cudaFuncSetAttribute(dev::df_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, dev::kDfSmemBytes));
  CK(cudaFuncSetAttribute(dev::adj_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, dev::kAmSmem));
  if (const char* e = std::getenv("GBOPT_ADJ_MMA")) adj_mma_ = e[0] != '0';
  if (const char* e = std::getenv("GBOPT_SYRK_FUSE")) syrk_fuse_ = e[0] != '0';
  if (const char* e = std::getenv("GBOPT_ADJ_FUSE")) adj_fuse_ = e[0] != '0';
  if (const char* e = std::getenv("GBOPT_SYRK_GATHER")) syrk_gather_ = e[0] != '0';
  if (const char* e = std::getenv("GBOPT_S0_PASS")) s0_mode_ = e[0] == '1' ? 1 : 0;
  CK(cudaFuncSetAttribute(dev::nt_syrk_segs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, dev::kSmemBytes));
  if (const char* e = std::getenv("GBOPT_DATAFLOW"))
    dataflow_mode_ = e[0] == '0' ? 0 : (e[0] == '-' && e[1] == '2') ? -2 : 1;
  if (const char* e = std::getenv("GBOPT_DF_GROUP")) df_group_ = std::max(1, std::atoi(e));
  if (const char* e = std::getenv("GBOPT_DF_SQ")) df_square_ = e[0] != '0';
  // (A maximal shared-memory carveout, tried so GEMV CTAs could co-reside with
  // nt_mma, cost 2% on c2 -- 173.4 vs 177.3 evals/s -- and is not set.  A
  // persistent stream-K schedule of the layer steps was also built and
  // measured slower -- 139-158 vs 177 evals/s on c2, profiles/r01_notes.md --
  // and was removed; the dataflow launch (dataflow.cuh) is the persistent
  // schedule.)
  int prio_lo = 0, prio_hi = 0;
  CK(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
  // Which stream gets the SMs first.  A layer's SYRK costs (n+1)/(2 n_{l-1})
  // of its tangent GEMM: when that is small (c2: 0.08) the GEMM chain is the
  // critical path and keeps priority (the SYRKs fill its last waves); when it
  // is large (c5: 0.38) the side stream goes first so the adjoint and SYRKs
  // are not starved into a tail (measured: c2 177 vs 172 evals/s, c5 579 vs
  // 624).  GBOPT_SIDE_HIGH=0/1 overrides.
  double ratio = 0.0;
  {
    const int64_t n = net.input_dim();
    for (int64_t l = 1; l + 1 < net.layer_count(); ++l)
      ratio = std::max(ratio, static_cast<double>(n + 1) / (2.0 * static_cast<double>(net.layer(l).cols)));
  }
  bool side_high = ratio > 0.2;
  if (const char* e = std::getenv("GBOPT_SIDE_HIGH")) side_high = e[0] == '1';
  CK(cudaStreamCreateWithPriority(&stream_, cudaStreamNonBlocking, side_high ? prio_lo : prio_hi));
  CK(cudaStreamCreateWithPriority(&stream2_, cudaStreamNonBlocking, side_high ? prio_hi : prio_lo));
  concurrent_ = std::getenv("GBOPT_SERIAL") == nullptr;  // debugging / A-B switch
  CK(cudaEventCreateWithFlags(&ev_in_, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&ev_out_, cudaEventDisableTiming));
  CK(cudaStreamCreateWithFlags(&copy_stream_, cudaStreamNonBlocking));

  n_ = net.input_dim();
  m_ = net.output_dim();
  L_ = net.layer_count();
  n_pad_ = round_up(n_, kBM);
  const auto& hl = net.layers();
  for (int64_t l = 0; l < L_; ++l) {
    const HostLayer& h = hl[static_cast<size_t>(l)];
    DevLayer d;
    d.rows = h.rows;
    d.cols = h.cols;
    d.act = h.act;
    d.ldw = round_up(h.cols, 16);
    CK(cudaMalloc(&d.w, sizeof(double) * d.rows * d.ldw));
    CK(cudaMemset(d.w, 0, sizeof(double) * d.rows * d.ldw));
    CK(cudaMemcpy2D(d.w, sizeof(double) * d.ldw, h.w.data(), sizeof(double) * h.cols, sizeof(double) * h.cols,
                    d.rows, cudaMemcpyHostToDevice));
    CK(cudaMalloc(&d.b, sizeof(double) * d.rows));
    CK(cudaMemcpy(d.b, h.b.data(), sizeof(double) * d.rows, cudaMemcpyHostToDevice));
    d.tm_w = make_tmap(d.w, d.cols, d.rows, d.ldw, kBN);
    d.tm_wadj = make_tmap(d.w, d.cols, d.rows, d.ldw, 16);
    layers_.push_back(d);
  }
  // T_0 = W_0^T, [n_pad][kp(n_1)], padded rows zero.
  const HostLayer& h0 = hl[0];
  ldt0_ = round_up(h0.rows, 16);
  std::vector<double> t0(static_cast<size_t>(n_pad_ * ldt0_), 0.0);
  for (int64_t i = 0; i < h0.rows; ++i)
    for (int64_t j = 0; j < h0.cols; ++j) t0[static_cast<size_t>(j * ldt0_ + i)] = h0.w[static_cast<size_t>(i * h0.cols + j)];
  CK(cudaMalloc(&t0_, sizeof(double) * t0.size()));
  CK(cudaMemcpy(t0_, t0.data(), sizeof(double) * t0.size(), cudaMemcpyHostToDevice));
  tm_t0_a_ = make_tmap(t0_, h0.rows, n_pad_, ldt0_, kBM);
  tm_t0_b_ = make_tmap(t0_, h0.rows, n_pad_, ldt0_, kBN);
  // Hidden-layer tangent width (pitch of the ping-pong T buffers).
  int64_t wmax = 16;
  for (int64_t l = 0; l < L_; ++l) wmax = std::max(wmax, layers_[static_cast<size_t>(l)].rows);
  ldt_ = round_up(wmax, 16);
  // SYRK tile list over an n x n lower triangle with kBM x kBN tiles.
  std::vector<int2> tiles;
  for (int tm = 0; tm * kBM < n_; ++tm)
    for (int tn = 0; tn * kBN < n_; ++tn)
      if (static_cast<int64_t>(tn) * kBN <= static_cast<int64_t>(tm) * kBM + kBM - 1) tiles.push_back(make_int2(tm, tn));
  n_syrk_tiles_ = static_cast<int>(tiles.size());
  CK(cudaMalloc(&syrk_tiles_, sizeof(int2) * tiles.size()));
  CK(cudaMemcpy(syrk_tiles_, tiles.data(), sizeof(int2) * tiles.size(), cudaMemcpyHostToDevice));
  // square 112 x 112 lower tiles (tn <= tm) for the layer-by-layer SYRKs
  std::vector<int2> sq;
  for (int tm = 0; tm * kBM < n_; ++tm)
    for (int tn = 0; tn <= tm; ++tn) sq.push_back(make_int2(tm, tn));
  n_sq_tiles_ = static_cast<int>(sq.size());
  CK(cudaMalloc(&sq_tiles_, sizeof(int2) * sq.size()));
  CK(cudaMemcpy(sq_tiles_, sq.data(), sizeof(int2) * sq.size(), cudaMemcpyHostToDevice));
  if (const char* e = std::getenv("GBOPT_SQ")) square_syrk_ = e[0] != '0';
  if (const char* e = std::getenv("GBOPT_FWD_STREAM")) fwd_stream_mode_ = e[0] == '1' ? 1 : 0;
}

DeviceNet::~DeviceNet() {
  DeviceGuard g(ordinal_);
  free_workspace();
  if (fs_arrive_) cudaFree(fs_arrive_);
  if (stage_) cudaFreeHost(stage_);
  for (auto& d : layers_) {
    cudaFree(d.w);
    cudaFree(d.b);
    if (d.wt) cudaFree(d.wt);
  }
  cudaFree(t0_);
  cudaFree(syrk_tiles_);
  cudaFree(sq_tiles_);
  if (stream_) cudaStreamDestroy(stream_);
  if (stream2_) cudaStreamDestroy(stream2_);
  for (cudaEvent_t e : evpool_) cudaEventDestroy(e);
  if (ev_in_) cudaEventDestroy(ev_in_);
  if (ev_out_) cudaEventDestroy(ev_out_);
  for (cudaEvent_t e : chunk_ev_) cudaEventDestroy(e);
  if (copy_stream_) cudaStreamDestroy(copy_stream_);
}

void DeviceNet::free_workspace() {
  free_plans();
  for (void* p : ws_allocs_) cudaFree(p);
  ws_allocs_.clear();
  ws_cap_ = 0;
  drop_graphs();
}

void DeviceNet::drop_graphs() {
  for (auto& kv : graphs_) {
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
  }
  graphs_.clear();
}

double* DeviceNet::ws_alloc(size_t n_doubles) {
  void* p = nullptr;
  CK(cudaMalloc(&p, sizeof(double) * std::max<size_t>(n_doubles, 2)));
  CK(cudaMemset(p, 0, sizeof(double) * std::max<size_t>(n_doubles, 2)));
  ws_allocs_.push_back(p);
  return static_cast<double*>(p);
}

// Split-K factor of a layer's SYRK: enough CTAs to cover the SMs twice, at
// least 8 k-blocks (128 of K) per split.
int DeviceNet::syrk_split(int points, int k_blocks) const {
  const int tiles = points * (square_syrk_ ? n_sq_tiles_ : n_syrk_tiles_);
  if (tiles >= sm_count_) return 1;
  // up to two CTAs' worth per SM: the SYRKs run in the tangent GEMMs' idle
  // SMs, and shorter slices fill them more evenly (c2: 5 -> 10 slices, 184.05
  // -> 184.8 evals/s; 15 / 20 slices 184.3 / 180-183, tools/r02_gpu81.sh)
  return std::max(1, std::min(2 * sm_count_ / tiles, k_blocks / 8));
}

// Adjoint sweep layout of a layer: columns per thread (4 for multi-vector
// sweeps of wide layers -- the shared-memory gz values reused over more
// columns -- else 2) and rows per chunk (kAdjRows, halved down to 16 while
// the grid would not cover two waves).
DeviceNet::AdjLayout DeviceNet::adj_layout(const DevLayer& d, bool multi) const {
  AdjLayout a;
  // (tried in round 2: a 10-vector pass for m = 10 instead of 12 with two
  // dead vectors, and 4 columns per thread with 64-row chunks for c2's J --
  // both slower, 72 -> 90 us per 5120^2 layer; profiles/r02_notes.md)
  a.kw = multi && ceil_div(d.cols, 4 * dev::kAdjThreads) * ceil_div(d.rows, dev::kAdjRows) >= 2 * sm_count_ ? 4 : 2;
  a.gx = static_cast<int>(ceil_div(d.cols, a.kw * dev::kAdjThreads));
  a.crows = dev::kAdjRows;
  while (a.crows > 16 && a.gx * ceil_div(d.rows, a.crows) < 2 * sm_count_) a.crows /= 2;
  a.chunks = static_cast<int>(ceil_div(d.rows, a.crows));
  return a;
}

void DeviceNet::ensure_workspace(int batch) {
  if (batch <= ws_cap_) return;
  std::lock_guard<std::recursive_mutex> lock(setup_mutex());
  free_workspace();
  const int cap = batch;
  const int64_t vcap = static_cast<int64_t>(cap) * std::max<int64_t>(m_, 1);
  Workspace& w = ws_;
  const size_t L = static_cast<size_t>(L_);
  w.z.assign(L, nullptr);
  w.y.assign(L, nullptr);
  w.s1.assign(L, nullptr);
  w.s2.assign(L, nullptr);
  w.ybar.assign(L, nullptr);
  w.gz.assign(L, nullptr);
  w.d.assign(L, nullptr);
  w.ld.assign(L, 0);
  for (size_t l = 0; l < L; ++l) {
    const int64_t ld = round_up(layers_[l].rows, 16);
    w.ld[l] = ld;
    w.z[l] = ws_alloc(cap * ld);
    w.y[l] = ws_alloc(cap * ld);
    w.s1[l] = ws_alloc(cap * ld);
    w.s2[l] = ws_alloc(cap * ld);
    w.ybar[l] = ws_alloc(vcap * ld);  // vcap: reverse-mode J runs m vectors per point
    w.gz[l] = ws_alloc(vcap * ld);
    w.d[l] = ws_alloc(cap * ld);
  }
  w.ld_in = round_up(n_, 16);
  w.ld_lam = round_up(m_, 16);
  w.x = ws_alloc(cap * w.ld_in);
  w.lam = ws_alloc(cap * w.ld_lam);
  w.grad = ws_alloc(vcap * w.ld_in);
  w.mid = ws_alloc(layers_[L - 1].act == kSoftmax ? static_cast<size_t>(cap) * m_ * m_ : 1);
  // adjoint partials: [chunks][cap][ldmax]
  int64_t rmax = 1;
  for (auto& d : layers_) rmax = std::max(rmax, d.rows);
  w.adj_chunks_max = 1;
  for (auto& d : layers_)
    for (bool multi : {false, true}) w.adj_chunks_max = std::max(w.adj_chunks_max, adj_layout(d, multi).chunks);
  w.ld_part = ldt_ > w.ld_in ? ldt_ : w.ld_in;
  w.adj_part = ws_alloc(static_cast<size_t>(w.adj_chunks_max) * vcap * w.ld_part);
  {  // arrival counters of the fused chunk reduction, one per column block
    int gx = 1;
    for (auto& d : layers_) gx = std::max(gx, ceil_div(d.cols, 2 * static_cast<int64_t>(dev::kAdjThreads)));
    w.adj_cnt = reinterpret_cast<unsigned*>(ws_alloc(static_cast<size_t>(gx)));
  }
  // tangents (only needed with >= 2 layers)
  // T_l (l >= 1) lives in ring buffer t_buf(l) = (l - 1) % R.  With R >= the
  // number of tangent layers the GEMM chain never waits for a SYRK to free
  // a buffer (and the dataflow path applies); R is capped by a memory
  // budget (32 GB of the 180 GB) and is at least 2.
  if (L_ >= 2) {
    // S_l = T_l diag(sigma'_l) (the pre-scaled A operand of the tangent
    // GEMMs) lives in a second ring with the same indexing
    const size_t tbytes = sizeof(double) * static_cast<size_t>(cap) * n_pad_ * ldt_ * 2;
    const int want = std::max(2, static_cast<int>(L_) - 1);
    const int fit = static_cast<int>(std::max<size_t>(2, (size_t(32) << 30) / std::max<size_t>(tbytes, 1)));
    const int ring = std::min(want, fit);
    w.t.assign(static_cast<size_t>(ring), nullptr);
    for (auto& b : w.t) b = ws_alloc(static_cast<size_t>(cap) * n_pad_ * ldt_);
    w.s.assign(static_cast<size_t>(ring), nullptr);
    for (auto& b : w.s) b = ws_alloc(static_cast<size_t>(cap) * n_pad_ * ldt_);
    w.s0 = ws_alloc(static_cast<size_t>(cap) * n_pad_ * ldt0_);
    w.tm_s0 = make_tmap(w.s0, layers_[0].rows, static_cast<int64_t>(cap) * n_pad_, ldt0_, kBM);
    w.tm_t_a.assign(L, CUtensorMap{});
    w.tm_t_b.assign(L, CUtensorMap{});
    w.tm_s_a.assign(L, CUtensorMap{});
    for (size_t l = 1; l < L; ++l) {
      const double* buf = w.t[(l - 1) % w.t.size()];
      w.tm_t_a[l] = make_tmap(buf, layers_[l].rows, static_cast<int64_t>(cap) * n_pad_, ldt_, kBM);
      w.tm_t_b[l] = make_tmap(buf, layers_[l].rows, static_cast<int64_t>(cap) * n_pad_, ldt_, kBN);
      w.tm_s_a[l] = make_tmap(w.s[(l - 1) % w.s.size()], layers_[l].rows, static_cast<int64_t>(cap) * n_pad_, ldt_, kBM);
    }
  }
  // Hessian accumulator [cap][n_pad][n_pad] and split-K partials
  w.ldh = n_pad_;
  w.h = ws_alloc(static_cast<size_t>(cap) * n_pad_ * n_pad_);
  // split * points * tiles <= max(2 sm_count, tiles) by construction of syrk_split
  w.syrk_part = ws_alloc(static_cast<size_t>(std::max(2 * sm_count_, std::max(n_syrk_tiles_, n_sq_tiles_))) * kBM * kBN);
  w.gemm_part = ws_alloc(static_cast<size_t>(sm_count_) * kBM * kBN);
  // per-layer SYRK partials of the gather path (single points: points x
  // square tiles < SMs), one buffer per curvature layer
  w.syrk_gather.clear();
  if (n_sq_tiles_ < sm_count_) {
    int segs = 0;
    for (auto& d : layers_) segs += d.act != kLinear;
    if (segs <= dev::kMaxGather)
      for (int q = 0; q < segs; ++q) w.syrk_gather.push_back(ws_alloc(static_cast<size_t>(2 * sm_count_) * kBM * kBN));
  }
  // final-layer skinny product: U [cap][n_pad][16], partials [chunks][cap][n_pad][16]
  const int64_t kfin = layers_[L - 1].cols;
  w.sk_chunks = ceil_div(kfin, dev::skinny_kchunk(m_ <= 1 ? 1 : (m_ <= 4 ? 4 : 16)));
  w.u = ws_alloc(static_cast<size_t>(cap) * n_pad_ * dev::kSkMB);
  w.sk_part = ws_alloc(static_cast<size_t>(w.sk_chunks) * cap * n_pad_ * dev::kSkMB);
  // vectors as TMA A operands (batched forward / adjoint GEMMs)
  w.tm_x = make_tmap(w.x, n_, cap, w.ld_in, kBM);
  w.tm_y.assign(L, CUtensorMap{});
  w.tm_gz.assign(L, CUtensorMap{});
  for (size_t l = 0; l < L; ++l) {
    w.tm_y[l] = make_tmap(w.y[l], layers_[l].rows, cap, w.ld[l], kBM);
    w.tm_gz[l] = make_tmap(w.gz[l], layers_[l].rows, vcap, w.ld[l], kBM);
  }
  // device-side outputs for the host API
  w.y_out = ws_alloc(static_cast<size_t>(cap) * m_);
  w.j_out = ws_alloc(static_cast<size_t>(cap) * m_ * n_);
  w.h_out = ws_alloc(static_cast<size_t>(cap) * n_ * n_);
  w.g_out = ws_alloc(static_cast<size_t>(cap) * n_);
  // ws_alloc zero-fills with cudaMemset on the legacy stream, which does not
  // order against the non-blocking compute streams: finish it here.
  CK(cudaDeviceSynchronize());
  ws_cap_ = cap;
}

// W_l^T copies (row-major [n_{l-1}][kp(n_l)]) for the batched adjoint GEMMs;
// made once, on first use, by a device transpose.
void DeviceNet::ensure_transposed() {
  if (transposed_) return;
  std::lock_guard<std::recursive_mutex> lock(setup_mutex());
  for (auto& d : layers_) {
    d.ldwt = round_up(d.rows, 16);
    CK(cudaMalloc(&d.wt, sizeof(double) * d.cols * d.ldwt));
    // on stream_: a legacy-stream memset would not be ordered before the
    // transpose on the non-blocking stream_
    CK(cudaMemsetAsync(d.wt, 0, sizeof(double) * d.cols * d.ldwt, stream_));
    dim3 grid(ceil_div(d.cols, 32), ceil_div(d.rows, 32));
    dev::transpose_kernel<<<grid, dim3(32, 8), 0, stream_>>>(d.w, d.ldw, static_cast<int>(d.rows),
                                                              static_cast<int>(d.cols), d.wt, d.ldwt);
    CK(cudaGetLastError());
    d.tm_wt = make_tmap(d.wt, d.rows, d.cols, d.ldwt, kBN);
  }
  CK(cudaStreamSynchronize(stream_));
  transposed_ = true;
}

// One layer of the batched forward (transposed == false: Z = Y W^T) or
// adjoint (transposed == true: Ybar = GZ W) as an nt_mma GEMM over the nb
// points, split-K when the tile grid is too small to fill the GPU; the row
// epilogue (activation or gz/d) is fused into the split reduction or run as
// an elementwise pass over `store`.
void DeviceNet::batch_gemm(cudaStream_t st, int nb, const CUtensorMap& ta, const DevLayer& d, bool transposed,
                           const void* epi_ptr, double* store) {
  const dev::RowEpi& e = *static_cast<const dev::RowEpi*>(epi_ptr);
  const int64_t N = transposed ? d.cols : d.rows;
  const int64_t K = transposed ? d.rows : d.cols;
  dev::NtParams p{};
  p.tiles = nullptr;
  p.tiles_m = ceil_div(nb, kBM);
  p.tiles_n = ceil_div(N, kBN);
  p.n_tiles = p.tiles_m * p.tiles_n;
  p.points = 1;
  p.k_blocks = ceil_div(K, kBK);
  int split = 1;
  if (p.n_tiles * 2 <= sm_count_) split = std::max(1, std::min(sm_count_ / p.n_tiles, p.k_blocks / 8));
  p.split = split;
  p.a_point_rows = 0;
  p.b_point_rows = 0;
  p.b_rows_valid = static_cast<int>(N);
  p.m_rows_valid = nb;
  p.scale = nullptr;
  p.c = store;
  p.c_point_stride = 0;
  p.ldc = e.ld;
  p.mode = split > 1 ? dev::kPartial : dev::kStore;
  p.partial = ws_.syrk_part;
  prof_begin(st, transposed ? kTagAdjGemm : kTagFwdGemm, 2.0 * nb * N * K, 8.0 * N * K);
  launch_nt(st, ta, transposed ? d.tm_wt : d.tm_w, p, p.n_tiles * split);
  prof_begin(st, kTagRowEpi, 0, 0);
  if (split > 1) {
    dim3 grid(4, p.n_tiles);
    dev::gemm_partial_reduce_kernel<<<grid, 256, 0, st>>>(ws_.syrk_part, split, p.tiles_m, p.tiles_n, nb,
                                                          static_cast<int>(N), e);
  } else {
    const int64_t tot = static_cast<int64_t>(nb) * N;
    dev::rows_epilogue_kernel<<<ceil_div(tot, 256), 256, 0, st>>>(store, nb, static_cast<int>(N), e);
  }
  after_launch(st);
}

// --------------------------------------------------------------------------
// Launch helpers
// --------------------------------------------------------------------------
// nt_mma launches of more tiles than SMs run persistent (GBOPT_NT_PERSIST=1):
// one CTA per SM walks its tiles, so the producer streams the next tile's
// k-blocks while the consumers store the current one.
void DeviceNet::launch_nt(cudaStream_t st, const CUtensorMap& ta, const CUtensorMap& tb, const dev::NtParams& p,
                          int grid) {
  static const int persist = [] {
    const char* e = std::getenv("GBOPT_NT_PERSIST");
    return e ? std::atoi(e) : 0;
  }();
  // (dense GEMM tiles only: the square SYRK consumers handle one tile per CTA)
  if (persist > 0 && grid > sm_count_ && p.square == 0) {
    dev::NtParams q = p;
    q.total_tiles = grid;
    dev::nt_mma_kernel<true><<<sm_count_ * persist, dev::kThreads, dev::kSmemBytes, st>>>(ta, tb, q);
  } else {
    dev::nt_mma_kernel<false><<<grid, dev::kThreads, dev::kSmemBytes, st>>>(ta, tb, p);
  }
  after_launch(st);
}

void DeviceNet::prof_begin(cudaStream_t st, int tag, double flops, double bytes) {
  if (!profiling_) return;
  ProfRec r;
  r.tag = tag;
  r.flops = flops;
  r.bytes = bytes;
  r.stream = st == stream_ ? 0 : 1;
  CK(cudaEventCreate(&r.e0));
  CK(cudaEventCreate(&r.e1));
  CK(cudaEventRecord(r.e0, st));
  prof_.push_back(r);
}

void DeviceNet::after_launch(cudaStream_t st) {
  CK(cudaGetLastError());
  ++launches_;
  if (profiling_) CK(cudaEventRecord(prof_.back().e1, st));
}

void DeviceNet::profile(int nb, const double* dx, const double* dlam, std::vector<ProfResult>* out, bool timeline) {
  DeviceGuard g(ordinal_);
  ensure_workspace(nb);
  Workspace& w = ws_;
  Outputs o;
  // GBOPT_PROFILE_OUTPUTS = "yjh" subset (default all three): which outputs
  // the profiled evaluation computes, e.g. "j" for the reverse-mode Jacobian
  const char* mask = std::getenv("GBOPT_PROFILE_OUTPUTS");
  const std::string ms(mask ? mask : "yjh");
  o.y = ms.find('y') != std::string::npos ? w.y_out : nullptr;
  o.j = ms.find('j') != std::string::npos ? w.j_out : nullptr;
  o.h = ms.find('h') != std::string::npos ? w.h_out : nullptr;
  prepare(nb, o);
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy2DAsync(w.x, sizeof(double) * w.ld_in, dx, sizeof(double) * n_, sizeof(double) * n_, nb,
                       cudaMemcpyDeviceToDevice, stream_));
  if (dlam)
    CK(cudaMemcpy2DAsync(w.lam, sizeof(double) * w.ld_lam, dlam, sizeof(double) * m_, sizeof(double) * m_, nb,
                         cudaMemcpyDeviceToDevice, stream_));
  profiling_ = true;
  prof_timeline_ = timeline;
  prof_.clear();
  launches_ = 0;
  cudaEvent_t base;
  CK(cudaEventCreate(&base));
  CK(cudaEventRecord(base, stream_));
  try {
    enqueue(stream_, nb, o);
  } catch (...) {
    profiling_ = prof_timeline_ = false;
    throw;
  }
  profiling_ = prof_timeline_ = false;
  CK(cudaStreamSynchronize(stream_));
  out->clear();
  for (auto& r : prof_) {
    float ms = 0.f, t0 = 0.f, t1 = 0.f;
    CK(cudaEventElapsedTime(&ms, r.e0, r.e1));
    CK(cudaEventElapsedTime(&t0, base, r.e0));
    CK(cudaEventElapsedTime(&t1, base, r.e1));
    out->push_back(ProfResult{r.tag, ms, r.flops, r.bytes, t0, t1, r.stream});
    cudaEventDestroy(r.e0);
    cudaEventDestroy(r.e1);
  }
  cudaEventDestroy(base);
  prof_.clear();
}

// Final layer with m <= 16 outputs: U = T_l diag(sigma'_l) W_{l+1}^T into
// w.u ([nb][n_pad][16]) by the skinny split-K kernel + fixed-order reduce.
void DeviceNet::launch_skinny(cudaStream_t st, int nb, const double* t, int64_t ldt, int64_t t_point_rows, int l,
                              double* jac) {
  Workspace& w = ws_;
  const DevLayer& df = layers_[static_cast<size_t>(l + 1)];
  dim3 grid(static_cast<unsigned>(n_pad_ / dev::kSkRows), w.sk_chunks, nb);
  prof_begin(st, kTagSkinny, 2.0 * n_ * m_ * df.cols * nb, 0);
  // template on the output count: no work on empty output slots
  if (m_ <= 1)
    dev::skinny_nt_kernel<1><<<grid, 256, 0, st>>>(t, ldt, t_point_rows, static_cast<int>(n_), w.s1[l], w.ld[l], df.w,
                                                   df.ldw, static_cast<int>(m_), static_cast<int>(df.cols), w.sk_part);
  else if (m_ <= 4)
    dev::skinny_nt_kernel<4><<<grid, 256, 0, st>>>(t, ldt, t_point_rows, static_cast<int>(n_), w.s1[l], w.ld[l], df.w,
                                                   df.ldw, static_cast<int>(m_), static_cast<int>(df.cols), w.sk_part);
  else
    dev::skinny_nt_kernel<16><<<grid, 256, 0, st>>>(t, ldt, t_point_rows, static_cast<int>(n_), w.s1[l], w.ld[l],
                                                    df.w, df.ldw, static_cast<int>(m_), static_cast<int>(df.cols),
                                                    w.sk_part);
  after_launch(st);
  const int64_t tot = static_cast<int64_t>(nb) * n_pad_ * dev::kSkMB;
  prof_begin(st, kTagSkinnyReduce, 0, 0);
  dev::skinny_reduce_kernel<<<ceil_div(tot, 256), 256, 0, st>>>(w.sk_part, w.sk_chunks, nb, static_cast<int>(n_pad_),
                                                                static_cast<int>(m_), w.u, jac, w.s1[l + 1], w.ld[l + 1],
                                                                static_cast<int>(n_));
  after_launch(st);
}

// Everything an evaluation needs that cannot be done inside a stream
// capture (allocations, synchronous uploads): W^T copies, dataflow plans.
void DeviceNet::prepare(int nb, const Outputs& o) {
  const bool df = dataflow_ok(nb, o);
  if (df || static_cast<int64_t>(nb) * std::max<int64_t>(m_, 1) >= kBatchGemm) ensure_transposed();
  if (df) dataflow_plan(nb);
}

// The whole evaluation for `nb` points whose x / lambda already sit in the
// workspace.  Outputs go to the given device pointers (nullable).
//
// Two streams: `sa` carries the critical path (forward chain, tangent GEMM
// chain, final layer, J); `sb` the adjoint chain and every Hessian SYRK,
// which only feed H.  SYRK_l waits for GEMM_l (T_l ready) and then runs
// beside GEMM_{l+1}, filling the SMs the GEMM's last wave leaves idle;
// GEMM_{l+1} overwrites T_{l-1}'s buffer, so it waits for SYRK_{l-1}.
// (Profiling runs serialise both onto one stream.)
void DeviceNet::enqueue(cudaStream_t st, int nb, const Outputs& o) {
  if (dataflow_ok(nb, o)) {
    enqueue_dataflow(st, nb, o);
    return;
  }
  Workspace& w = ws_;
  // profiling serialises onto one stream, except the timeline mode
  const bool two = concurrent_ && (!profiling_ || prof_timeline_);
  cudaStream_t sa = st;
  cudaStream_t sb = two ? stream2_ : st;
  int ev_next = 0;
  auto next_event = [&]() -> cudaEvent_t {
    if (ev_next >= static_cast<int>(evpool_.size())) {
      cudaEvent_t e;
      CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      evpool_.push_back(e);
    }
    return evpool_[static_cast<size_t>(ev_next++)];
  };
  // make `to` wait for everything enqueued so far on `from`
  bool sb_forked = false;  // sb joins a capture only through a fork from sa
  auto link = [&](cudaStream_t from, cudaStream_t to) {
    if (from == to) return;
    if (from == sb && !sb_forked) return;  // nothing was enqueued on sb
    if (to == sb) sb_forked = true;
    cudaEvent_t e = next_event();
    CK(cudaEventRecord(e, from));
    CK(cudaStreamWaitEvent(to, e, 0));
  };
  const int L = static_cast<int>(L_);
  const bool softmax_out = layers_[L - 1].act == kSoftmax;
  const bool want_h = o.h != nullptr;
  const bool want_j = o.j != nullptr;
  const bool need_adj = want_h || o.g != nullptr;
  const bool need_tan = want_h || want_j;

  // ---- 1. forward chain --------------------------------------------------
  const double* yin = w.x;
  int64_t ld_in = w.ld_in;
  const bool batched = nb >= kBatchGemm;
  // Layer 0 runs on sa (GEMM_1 needs only sigma'_0); layers >= 1 run on sb,
  // beside the tangent GEMMs, each recording fwd_done[l] for GEMM_{l+1}.
  std::vector<cudaEvent_t> fwd_done(static_cast<size_t>(L), nullptr);
  // a single point with an elementwise output: the last layer's GEMV also
  // writes y out and seeds the adjoint (no copy node, no seed launch)
  const bool tail_fused = nb == 1 && !batched && !softmax_out;
  for (int l = 0; l < L; ++l) {
    const DevLayer& d = layers_[static_cast<size_t>(l)];
    if (l == 1) link(sa, sb);
    // this layer's stream (shadows the outer `sa` inside the loop body)
    cudaStream_t sa = l == 0 ? st : sb;
    if (batched) {
      dev::RowEpi e{};
      e.mode = dev::kEpiAct;
      e.act = d.act == kSoftmax ? kLinear : d.act;
      e.bias = d.b;
      e.z = w.z[l];
      e.y = w.y[l];
      e.s1o = w.s1[l];
      e.s2o = w.s2[l];
      e.ld = w.ld[l];
      batch_gemm(sa, nb, l == 0 ? w.tm_x : w.tm_y[static_cast<size_t>(l - 1)], d, false, &e, w.z[l]);
      if (two && l > 0) {
        fwd_done[static_cast<size_t>(l)] = next_event();
        CK(cudaEventRecord(fwd_done[static_cast<size_t>(l)], sb));
      }
      continue;
    }
    const int nbpass = nb >= 8 ? 8 : (nb >= 4 ? 4 : 1);
    dim3 grid(ceil_div(d.rows, dev::kFwdWarps), ceil_div(nb, nbpass));
    const int act = d.act == kSoftmax ? kLinear : d.act;
    prof_begin(sa, kTagFwd, 2.0 * d.rows * d.cols * nb, 8.0 * d.rows * d.cols * ceil_div(nb, nbpass));
    if (nb == 1) {
      dev::FwdTail tail{};
      if (l == L - 1 && tail_fused) {
        tail.y = o.y;
        if (need_adj) {
          tail.lam = w.lam;
          tail.gz = w.gz[L - 1];
          tail.d = w.d[L - 1];
        }
      }
      // warps per row so that short layers (the 10-row output) still spread
      // over the GPU: aim at >= 16 warps per SM
      const int64_t target = static_cast<int64_t>(sm_count_) * 16;
      const int wpr = d.rows >= target ? 1 : d.rows * 2 >= target ? 2 : d.rows * 4 >= target ? 4 : 8;
      const dim3 g1(ceil_div(d.rows * wpr, dev::kFwdWarps));
      if (wpr == 1)
        dev::fwd_row1_kernel<1><<<g1, dev::kFwdWarps * 32, 0, sa>>>(d.w, d.ldw, d.b, d.rows, d.cols, yin, act,
                                                                    w.z[l], w.y[l], w.s1[l], w.s2[l], tail);
      else if (wpr == 2)
        dev::fwd_row1_kernel<2><<<g1, dev::kFwdWarps * 32, 0, sa>>>(d.w, d.ldw, d.b, d.rows, d.cols, yin, act,
                                                                    w.z[l], w.y[l], w.s1[l], w.s2[l], tail);
      else if (wpr == 4)
        dev::fwd_row1_kernel<4><<<g1, dev::kFwdWarps * 32, 0, sa>>>(d.w, d.ldw, d.b, d.rows, d.cols, yin, act,
                                                                    w.z[l], w.y[l], w.s1[l], w.s2[l], tail);
      else
        dev::fwd_row1_kernel<8><<<g1, dev::kFwdWarps * 32, 0, sa>>>(d.w, d.ldw, d.b, d.rows, d.cols, yin, act,
                                                                    w.z[l], w.y[l], w.s1[l], w.s2[l], tail);
    } else if (nbpass == 8)
      dev::fwd_rows_kernel<8><<<grid, dev::kFwdWarps * 32, 0, sa>>>(d.w, d.ldw, d.b, d.rows, d.cols, yin, ld_in, nb,
                                                                     act, w.z[l], w.y[l], w.s1[l], w.s2[l], w.ld[l]);
    else if (nbpass == 4)
      dev::fwd_rows_kernel<4><<<grid, dev::kFwdWarps * 32, 0, sa>>>(d.w, d.ldw, d.b, d.rows, d.cols, yin, ld_in, nb,
                                                                     act, w.z[l], w.y[l], w.s1[l], w.s2[l], w.ld[l]);
    else
      dev::fwd_rows_kernel<1><<<grid, dev::kFwdWarps * 32, 0, sa>>>(d.w, d.ldw, d.b, d.rows, d.cols, yin, ld_in, nb,
                                                                     act, w.z[l], w.y[l], w.s1[l], w.s2[l], w.ld[l]);
    after_launch(sa);
    if (two && l > 0) {
      fwd_done[static_cast<size_t>(l)] = next_event();
      CK(cudaEventRecord(fwd_done[static_cast<size_t>(l)], sb));
    }
    yin = w.y[l];
    ld_in = w.ld[l];
  }
  // the forward's tail (softmax, y copy) follows its last layer's stream
  cudaStream_t sf = L > 1 ? sb : sa;
  if (softmax_out) {
    prof_begin(sf, kTagSoftmax, 0, 0);
    dev::softmax_kernel<<<ceil_div(nb, 4), 128, 0, sf>>>(w.z[L - 1], w.y[L - 1], static_cast<int>(m_), w.ld[L - 1],
                                                         nb);
    after_launch(sf);
  }
  if (o.y && !tail_fused) {
    CK(cudaMemcpy2DAsync(o.y, sizeof(double) * m_, w.y[L - 1], sizeof(double) * w.ld[L - 1], sizeof(double) * m_, nb,
                         cudaMemcpyDeviceToDevice, sf));
  }
  cudaEvent_t fwd_all = nullptr;  // the whole forward chain (sb), for the final layer on sa
  if (two && L > 1) {
    fwd_all = next_event();
    CK(cudaEventRecord(fwd_all, sb));
  }

  // ---- 2. adjoint chain --------------------------------------------------
  // Reverse sweep from the seeded gz_{L-1} (nv vectors; vector v belongs to
  // point v / s_div) down to layer `lstop`, leaving ybar/gz/d per layer and,
  // for lstop == 0, the input-space result in w.grad (nn.cpp:172-196).
  auto adjoint_chain = [&](int nv, int s_div, int lstop, bool want_d) {
    const bool gemm = nv >= kBatchGemm;
    for (int l = L - 1; l >= lstop; --l) {
      const DevLayer& d = layers_[static_cast<size_t>(l)];
      if (gemm) {
        dev::RowEpi e{};
        e.mode = dev::kEpiAdj;
        e.s_div = s_div;
        if (l > 0) {
          e.s1i = w.s1[l - 1];
          e.s2i = w.s2[l - 1];
          e.ybar = w.ybar[l - 1];
          e.gz = w.gz[l - 1];
          e.d = want_d ? w.d[l - 1] : nullptr;
          e.ld = w.ld[l - 1];
        } else {
          e.ybar = w.grad;
          e.ld = w.ld_in;
        }
        batch_gemm(sb, nv, w.tm_gz[static_cast<size_t>(l)], d, true, &e, e.ybar);
        continue;
      }
      const AdjLayout al = adj_layout(d, nv >= 5);
      const int kw = al.kw, gx = al.gx, crows = al.crows;
      int chunks = al.chunks;
      dim3 grid(gx, chunks);
      // 4+ vectors (reverse-mode J seeds, small batches): the DMMA kernel
      const bool mma = adj_mma_ && nv >= 4 && d.cols >= 128 && d.rows >= 64;
      if (mma) {
        // 256-row chunks (smaller chunks for narrow layers measured slower:
        // c2's 784-column W_1 with 32-row chunks 14.9 -> 18.9 us, its reduce
        // 8.7 -> 27 us over 5x the partials)
        int am_rows = dev::kAmRows;
        while (ceil_div(d.rows, am_rows) > w.adj_chunks_max) am_rows *= 2;  // partial buffer capacity
        chunks = ceil_div(d.rows, am_rows);
        const dim3 ga(ceil_div(d.cols, 128), chunks);
        for (int p0 = 0; p0 < nv; p0 += 16) {
          prof_begin(sb, kTagAdjCols, 2.0 * d.rows * d.cols * std::min(16, nv - p0), 8.0 * d.rows * d.cols);
          dev::adj_mma_kernel<<<ga, 288, dev::kAmSmem, sb>>>(d.tm_wadj, static_cast<int>(d.rows),
                                                              static_cast<int>(d.cols), w.gz[l], w.ld[l], nv, p0,
                                                              w.adj_part, w.ld_part, am_rows);
          after_launch(sb);
        }
      }
      // the chunk reduction rides on the sweep's last CTA per column block
      // (adj_fuse_; bit-identical to adj_reduce_kernel)
      dev::AdjFuse f{};
      const bool fuse = adj_fuse_ && !mma && w.adj_cnt != nullptr;
      if (fuse) {
        f.counters = w.adj_cnt;
        f.chunks = chunks;
        f.s_div = l > 0 ? s_div : 1;
        if (l > 0) {
          f.s1 = w.s1[l - 1];
          f.s2 = w.s2[l - 1];
          f.ld = w.ld[l - 1];
          f.ybar = w.ybar[l - 1];
          f.gz = w.gz[l - 1];
          f.d = want_d ? w.d[l - 1] : nullptr;
        } else {
          f.ld = w.ld_in;
          f.ybar = w.grad;
        }
      }
      for (int p0 = 0; p0 < nv && !mma;) {
        const int left = nv - p0;
        // one weight sweep per up to 16 vectors (reverse-mode J: m <= 16
        // seeds per point)
        const int pass = left >= 13 ? 16 : (left >= 9 ? 12 : (left >= 5 ? 8 : (left >= 2 ? 4 : 1)));
        prof_begin(sb, kTagAdjCols, 2.0 * d.rows * d.cols * std::min(pass, left), 8.0 * d.rows * d.cols);
#define GBB_ADJ(NBV, KWV)                                                                                          \
  dev::adj_cols_kernel<NBV, KWV><<<grid, dev::kAdjThreads, 0, sb>>>(d.w, d.ldw, d.rows, d.cols, w.gz[l], w.ld[l], nv, \
                                                                    p0, w.adj_part, w.ld_part, crows, f)
        if (pass == 16) {
          if (kw == 4) GBB_ADJ(16, 4); else GBB_ADJ(16, 2);
        } else if (pass == 12) {
          if (kw == 4) GBB_ADJ(12, 4); else GBB_ADJ(12, 2);

        } else if (pass == 8) {
          if (kw == 4) GBB_ADJ(8, 4); else GBB_ADJ(8, 2);
        } else if (pass == 4) {
          GBB_ADJ(4, 2);
        } else {
          GBB_ADJ(1, 2);
        }
#undef GBB_ADJ
        p0 += pass;
        after_launch(sb);
      }
      if (fuse) continue;
      const int64_t tot = static_cast<int64_t>(nv) * d.cols;
      prof_begin(sb, kTagAdjReduce, 0, 0);
      if (l > 0) {
        dev::adj_reduce_kernel<<<ceil_div(tot, 256), 256, 0, sb>>>(
            w.adj_part, chunks, w.ld_part, static_cast<int>(d.cols), nv, w.s1[l - 1], w.s2[l - 1], w.ld[l - 1],
            w.ybar[l - 1], w.gz[l - 1], want_d ? w.d[l - 1] : nullptr, s_div);
      } else {
        dev::adj_reduce_kernel<<<ceil_div(tot, 256), 256, 0, sb>>>(w.adj_part, chunks, w.ld_part,
                                                                   static_cast<int>(d.cols), nv, nullptr, nullptr,
                                                                   w.ld_in, w.grad, nullptr, nullptr, 1);
      }
      after_launch(sb);
    }
  };

  cudaEvent_t adj_done = nullptr;  // the adjoint chain (d_l of every layer) on sb
  if (need_adj) {
    link(sa, sb);  // the adjoint needs the forward chain
    if (!tail_fused) {
      prof_begin(sb, kTagAdjSeed, 0, 0);
      dev::adj_seed_kernel<<<ceil_div(nb, 4), 128, 0, sb>>>(
          w.lam, w.ld_lam, w.y[L - 1], w.s1[L - 1], w.s2[L - 1], w.ld[L - 1], static_cast<int>(m_), nb,
          softmax_out ? 1 : 0, w.gz[L - 1], w.d[L - 1], w.mid, m_ * m_);
      after_launch(sb);
    }
    adjoint_chain(nb, 1, o.g ? 0 : 1, true);
    if (two) {
      adj_done = next_event();
      CK(cudaEventRecord(adj_done, sb));
    }
    if (o.g) {
      CK(cudaMemcpy2DAsync(o.g, sizeof(double) * n_, w.grad, sizeof(double) * w.ld_in, sizeof(double) * n_, nb,
                           cudaMemcpyDeviceToDevice, sb));
    }
  }

  // J without H: reverse mode with m seed vectors per point, like the
  // reference jacobian (nn.cpp:148-170) -- m weight sweeps instead of the
  // n-column tangent chain.
  if (want_j && !want_h) {
    link(sa, sb);
    const int nv = nb * static_cast<int>(m_);
    const int64_t tot = static_cast<int64_t>(nb) * m_ * m_;
    prof_begin(sb, kTagAdjSeed, 0, 0);
    dev::jac_seed_kernel<<<ceil_div(tot, 256), 256, 0, sb>>>(w.y[L - 1], w.s1[L - 1], w.ld[L - 1],
                                                             static_cast<int>(m_), nb, softmax_out ? 1 : 0,
                                                             w.gz[L - 1]);
    after_launch(sb);
    adjoint_chain(nv, static_cast<int>(m_), 0, false);
    CK(cudaMemcpy2DAsync(o.j, sizeof(double) * n_, w.grad, sizeof(double) * w.ld_in, sizeof(double) * n_, nv,
                         cudaMemcpyDeviceToDevice, sb));
    link(sb, sa);
    return;
  }

  if (!need_tan) {
    link(sb, sa);
    return;
  }
  // ---- 3. tangent chain + Hessian SYRK ------------------------------------
  // One point tile (n <= 112, e.g. c4's contingencies), a batch that fills
  // the GPU and every tangent resident: all hidden layers' curvature in ONE
  // multi-segment launch after the last tangent GEMM (nt_syrk_segs_kernel),
  // storing each point's tile once instead of zeroing H and accumulating a
  // launch per layer (GBOPT_SYRK_FUSE=0: per layer)
  int nl_hidden = 0;
  for (int l = 0; l + 1 < L; ++l) nl_hidden += layers_[static_cast<size_t>(l)].act != kLinear;
  const bool fuse_syrk = want_h && syrk_fuse_ && square_syrk_ && n_pad_ == kBM && nb >= sm_count_ &&
                         nl_hidden >= 1 && nl_hidden <= dev::kMaxSegs &&
                         static_cast<int>(w.t.size()) >= L - 2;
  const int kfin_layer = L - 1;
  const bool skinny_final = m_ <= dev::kSkMB;
  // T_l lives in: l == 0 -> t0_ (broadcast over points), else ring buffer
  // (l - 1) % R.
  const int ring = static_cast<int>(w.t.size());
  auto t_buf = [&](int l) -> double* { return w.t[static_cast<size_t>((l - 1) % ring)]; };
  auto t_ptr = [&](int l) -> const double* { return l == 0 ? t0_ : t_buf(l); };
  auto t_ld = [&](int l) -> int64_t { return l == 0 ? ldt0_ : ldt_; };
  auto t_point_rows = [&](int l) -> int64_t { return l == 0 ? 0 : n_pad_; };
  auto tmap_a = [&](int l) -> const CUtensorMap& { return l == 0 ? tm_t0_a_ : w.tm_t_a[static_cast<size_t>(l)]; };
  auto tmap_b = [&](int l) -> const CUtensorMap& { return l == 0 ? tm_t0_b_ : w.tm_t_b[static_cast<size_t>(l)]; };

  // Gather path (small batches: every SYRK is split over k): each layer's
  // partials stay in their own buffer, one syrk_gather_out launch sums them
  // into the output; the last hidden layer's SYRK then runs on sa beside the
  // side stream's (GBOPT_SYRK_GATHER=0: reduce per layer into H on sb)
  const bool gather = want_h && !fuse_syrk && syrk_gather_ && square_syrk_ &&
                      static_cast<int64_t>(nb) * n_sq_tiles_ < sm_count_ &&
                      static_cast<int>(w.syrk_gather.size()) >= [&] {
                        int segs = 0;
                        for (int l = 0; l < L; ++l) segs += layers_[static_cast<size_t>(l)].act != kLinear;
                        return segs;
                      }();
  dev::SyrkGather gat{};
  gat.n_tiles = n_sq_tiles_;
  gat.points = nb;
  // the final layer's curvature as a direct update into H (small K)
  const DevLayer& dl = layers_[static_cast<size_t>(L - 1)];
  const bool h_direct = dl.act != kLinear && (softmax_out || m_ <= dev::kSkMB || L == 1);
  if (want_h && !fuse_syrk && (!gather || h_direct))
    CK(cudaMemsetAsync(w.h, 0, sizeof(double) * nb * n_pad_ * n_pad_, sb));
  auto syrk = [&](int l, cudaStream_t ss) {
    const DevLayer& d = layers_[static_cast<size_t>(l)];
    dev::NtParams p{};
    p.tiles = syrk_tiles_;
    p.n_tiles = n_syrk_tiles_;
    p.points = nb;
    p.split = syrk_split(nb, ceil_div(d.rows, kBK));
    p.k_blocks = ceil_div(d.rows, kBK);
    p.a_point_rows = t_point_rows(l);
    p.b_point_rows = t_point_rows(l);
    p.b_rows_valid = static_cast<int>(n_);
    p.m_rows_valid = static_cast<int>(n_);
    p.scale = w.d[l];
    p.s_stride = w.ld[l];
    p.c = w.h;
    p.c_point_stride = n_pad_ * n_pad_;
    p.ldc = n_pad_;
    p.mode = p.split > 1 ? dev::kPartial : dev::kAccum;
    p.partial = w.syrk_part;
    if (square_syrk_) {  // 112 x 112 lower tiles, B through the 112-row box map
      p.tiles = sq_tiles_;
      p.n_tiles = n_sq_tiles_;
      p.square = 1;
    }
    if (gather) {  // this layer's slices into its own buffer (split 1 too: no atomics into a shared H)
      p.mode = dev::kPartial;
      p.partial = w.syrk_gather[static_cast<size_t>(gat.nseg)];
      gat.part[gat.nseg] = p.partial;
      gat.split[gat.nseg++] = p.split;
    }
    prof_begin(ss, kTagSyrk, static_cast<double>(d.rows) * n_ * (n_ + 1) * nb, 0);
    launch_nt(ss, tmap_a(l), square_syrk_ ? tmap_a(l) : tmap_b(l), p, nb * p.n_tiles * p.split);
    if (p.split > 1 && !gather) {
      prof_begin(sb, kTagSyrkReduce, 0, 0);
      dim3 grid(8, nb * p.n_tiles);
      dev::syrk_partial_reduce_kernel<<<grid, 256, 0, ss>>>(w.syrk_part, p.tiles, p.n_tiles, nb, p.split, w.h,
                                                            n_pad_ * n_pad_, n_pad_, static_cast<int>(n_),
                                                            square_syrk_ ? kBM : kBN);
      after_launch(ss);
    }
  };

  // Pre-scaled tangents pay one extra tile store per tile; nets whose
  // single-point GEMMs are split-K (c1: 28 tiles) are launch-latency bound
  // and keep the per-fragment scale.
  bool prescaled = true;
  for (int l = 0; l + 2 < L && prescaled; ++l)
    if (nb == 1 && (n_pad_ / kBM) * ceil_div(layers_[static_cast<size_t>(l + 1)].rows, kBN) * 2 <= sm_count_)
      prescaled = false;
  cudaEvent_t t_last = nullptr;  // gather path: T_{L-2} ready on sa (the final layer then runs on sb)
  bool defer_last = false;        // gather path: SYRK_{L-2} on sa after the final layer
  // syrk_done[l]: event on sb after SYRK_l (nullptr when none ran)
  std::vector<cudaEvent_t> syrk_done(static_cast<size_t>(L), nullptr);
  for (int l = 0; l + 1 < L; ++l) {
    // curvature of hidden layer l, on sb once T_l exists (T_0 is constant)
    // gather path, last hidden layer before a skinny final layer: its SYRK
    // runs on sa (beside the side stream's SYRKs) once its d (sb's adjoint
    // chain) exists.  With one tangent GEMM (L = 3, c1) it runs right after
    // that GEMM and the final layer moves to sb, so the two SYRKs overlap
    // (c1 9.5k -> 10.4k evals/s); with a longer chain the final layer's
    // bandwidth-bound skinny product goes first on sa, alone on the SMs
    // (c2: 183.7 vs 182.8 evals/s the other way round)
    const bool defer = gather && two && l >= 1 && l == L - 2 && l + 1 == kfin_layer && skinny_final &&
                       adj_done != nullptr && layers_[static_cast<size_t>(l)].act != kLinear;
    if (defer && L == 3) {
      t_last = next_event();
      CK(cudaEventRecord(t_last, sa));
      CK(cudaStreamWaitEvent(sa, adj_done, 0));
      syrk(l, sa);
    }
    defer_last = defer && L > 3;
    if (want_h && !fuse_syrk && layers_[static_cast<size_t>(l)].act != kLinear && !defer) {
      if (l > 0) link(sa, sb);
      syrk(l, sb);
      if (two) {
        syrk_done[static_cast<size_t>(l)] = next_event();
        CK(cudaEventRecord(syrk_done[static_cast<size_t>(l)], sb));
      }
    }
    // propagate the tangents to layer l+1 (unless it is a skinny final)
    if (l + 1 == kfin_layer && skinny_final) break;
    // T_{l+1} overwrites T_{l+1-R} in the ring: wait for that layer's SYRK
    const int prev = l + 1 - ring;
    if (prev >= 1 && syrk_done[static_cast<size_t>(prev)])
      CK(cudaStreamWaitEvent(sa, syrk_done[static_cast<size_t>(prev)], 0));
    // ... and needs sigma'_l from the forward chain (sb for l >= 1)
    if (l >= 1 && fwd_done[static_cast<size_t>(l)])
      CK(cudaStreamWaitEvent(sa, fwd_done[static_cast<size_t>(l)], 0));
    const DevLayer& dn = layers_[static_cast<size_t>(l + 1)];
    dev::NtParams p{};
    p.tiles = nullptr;
    p.tiles_m = static_cast<int>(n_pad_ / kBM);
    p.tiles_n = ceil_div(dn.rows, kBN);
    p.n_tiles = p.tiles_m * p.tiles_n;
    p.points = nb;
    p.split = 1;
    p.k_blocks = ceil_div(dn.cols, kBK);
    p.a_point_rows = t_point_rows(l);
    p.b_point_rows = 0;
    p.b_rows_valid = static_cast<int>(dn.rows);
    p.m_rows_valid = static_cast<int>(n_pad_);
    p.scale = w.s1[l];
    p.s_stride = w.ld[l];
    p.c = t_buf(l + 1);
    p.c_point_stride = n_pad_ * ldt_;
    p.ldc = ldt_;
    p.mode = dev::kStore;
    // Pre-scaled A operand: GEMM_{l+1} reads S_l = T_l diag(sigma'_l) (no
    // per-fragment multiply in the k-loop) and writes S_{l+1} beside T_{l+1}
    // when a later GEMM reads it.  S_0 (per point) by one elementwise pass.
    const CUtensorMap* ta = &tmap_a(l);
    if (prescaled) {
      // S_0 (per point) costs one pass writing nb x n_pad x n_1 doubles; it
      // pays for itself when the GEMM it feeds is wide: the saved multiply is
      // ~4% of 2 nb n n_1 n_2 flops against 8 nb n n_1 bytes written, i.e.
      // n_2 >~ 1400 (c2/c3: 5120 yes; c4/c5: 1024 no -- the first GEMM then
      // keeps the per-fragment scale on the shared T_0).
      const bool s0_pass = s0_mode_ >= 0 ? s0_mode_ == 1 : layers_[1].rows >= 2048;
      if (l == 0 && s0_pass) {
        const int cols0 = static_cast<int>(layers_[0].rows);
        prof_begin(sa, kTagRowEpi, 0, 0);
        dev::scale_cols_kernel<<<dim3(ceil_div(cols0, 256), static_cast<unsigned>(std::min<int64_t>(nb * n_pad_, 65535))),
                                 256, 0, sa>>>(
            t0_, ldt0_, 0, static_cast<int>(n_pad_), cols0, w.s1[0], w.ld[0], w.s0, ldt0_, n_pad_, nb);
        after_launch(sa);
        ta = &w.tm_s0;
      } else if (l > 0) {
        ta = &w.tm_s_a[static_cast<size_t>(l)];
      }
      if (l > 0 || s0_pass) {
        p.a_point_rows = n_pad_;
        p.scale = nullptr;
      }
      const bool next_gemm = l + 2 < L && !(l + 2 == kfin_layer && skinny_final);
      if (next_gemm) {
        if (fwd_done[static_cast<size_t>(l + 1)])
          CK(cudaStreamWaitEvent(sa, fwd_done[static_cast<size_t>(l + 1)], 0));  // sigma'_{l+1}
        p.c2 = w.s[static_cast<size_t>(l % ring)];
        p.c2_scale = w.s1[static_cast<size_t>(l + 1)];
        p.c2_scale_stride = w.ld[static_cast<size_t>(l + 1)];
      }
    }
    // a single point with fewer tiles than half the SMs (c1: 28 tiles):
    // split K, then a fixed-order reduction stores T_{l+1}
    if (nb == 1 && p.n_tiles * 2 <= sm_count_) {
      p.split = std::max(1, std::min(sm_count_ / p.n_tiles, p.k_blocks / 8));
      if (p.split > 1) {
        p.mode = dev::kPartial;
        p.partial = w.gemm_part;  // not syrk_part: SYRKs on sb may run concurrently
        prof_begin(sa, kTagGemm, 2.0 * n_ * dn.rows * dn.cols * nb, 0);
        launch_nt(sa, *ta, dn.tm_w, p, p.n_tiles * p.split);
        dev::RowEpi e{};
        e.mode = dev::kEpiStore;
        e.z = p.c;
        e.y = p.c2;  // S_{l+1} (nb == 1: sigma' row of point 0)
        e.s1i = p.c2_scale;
        e.ld = ldt_;
        prof_begin(sa, kTagRowEpi, 0, 0);
        dev::gemm_partial_reduce_kernel<<<dim3(kGemmReduceX, p.n_tiles), 256, 0, sa>>>(
            w.gemm_part, p.split, p.tiles_m, p.tiles_n, static_cast<int>(n_pad_), static_cast<int>(dn.rows), e);
        after_launch(sa);
        continue;
      }
    }
    prof_begin(sa, kTagGemm, 2.0 * n_ * dn.rows * dn.cols * nb, 0);
    launch_nt(sa, *ta, dn.tm_w, p, nb * p.n_tiles);
  }

  if (fuse_syrk) {
    link(sa, sb);  // every tangent T_l exists
    dev::SyrkSegs sg{};
    const CUtensorMap* maps[dev::kMaxSegs] = {};
    double flops = 0.0;
    for (int l = 0; l + 1 < L; ++l) {
      const DevLayer& d = layers_[static_cast<size_t>(l)];
      if (d.act == kLinear) continue;
      const int s_i = sg.nseg++;
      maps[s_i] = &tmap_a(l);
      sg.nkb[s_i] = ceil_div(d.rows, kBK);
      sg.scale[s_i] = w.d[l];
      sg.s_stride[s_i] = w.ld[l];
      sg.a_point_rows[s_i] = t_point_rows(l);
      flops += static_cast<double>(d.rows) * n_ * (n_ + 1) * nb;
    }
    for (int s_i = sg.nseg; s_i < dev::kMaxSegs; ++s_i) maps[s_i] = maps[0];
    dev::NtParams p{};
    p.points = nb;
    p.split = 1;
    p.b_rows_valid = static_cast<int>(n_);
    p.m_rows_valid = static_cast<int>(n_);
    p.c = w.h;
    p.c_point_stride = n_pad_ * n_pad_;
    p.ldc = n_pad_;
    p.mode = dev::kStore;
    prof_begin(sb, kTagSyrk, flops, 0);
    dev::nt_syrk_segs_kernel<<<nb, dev::kThreads, dev::kSmemBytes, sb>>>(*maps[0], *maps[1], *maps[2], *maps[3], p,
                                                                          sg);
    after_launch(sb);
  }

  // ---- 4. final layer -------------------------------------------------------
  cudaStream_t sfin = sa;
  if (t_last) {
    sfin = sb;  // after the forward chain (stream order) and T_{L-2}
    CK(cudaStreamWaitEvent(sb, t_last, 0));
  } else if (fwd_all) {
    CK(cudaStreamWaitEvent(sa, fwd_all, 0));  // sigma'/y of the last layers
  }
  const DevLayer& df = layers_[static_cast<size_t>(kfin_layer)];
  const double* u;
  int64_t ldu, u_point_rows;
  if (kfin_layer == 0) {
    u = t0_;
    ldu = ldt0_;
    u_point_rows = 0;
  } else if (skinny_final) {
    const int l = kfin_layer - 1;
    // elementwise final activation: J written by the skinny reduction
    launch_skinny(sfin, nb, t_ptr(l), t_ld(l), t_point_rows(l), l, want_j && !softmax_out ? o.j : nullptr);
    u = w.u;
    ldu = dev::kSkMB;
    u_point_rows = n_pad_;
  } else {
    u = t_ptr(kfin_layer);
    ldu = ldt_;
    u_point_rows = n_pad_;
  }
  if (want_j && !(skinny_final && kfin_layer > 0 && !softmax_out)) {
    const int64_t tot = static_cast<int64_t>(nb) * n_;
    prof_begin(sfin, kTagJacOut, 0, 0);
    dev::jacobian_out_kernel<<<ceil_div(tot, 128), 128, 0, sfin>>>(u, ldu, u_point_rows, w.s1[kfin_layer],
                                                                   w.y[kfin_layer], w.ld[kfin_layer],
                                                                   static_cast<int>(n_), static_cast<int>(m_), nb,
                                                                   softmax_out ? 1 : 0, o.j);
    after_launch(sfin);
  }
  if (defer_last) {
    CK(cudaStreamWaitEvent(sa, adj_done, 0));
    syrk(L - 2, sa);
  }
  if (want_h) {
    cudaStream_t sh = sb;  // the SYRKs live on sb
    link(sa, sb);          // the final curvature needs U (sa)
    if (df.act != kLinear) {
      if (softmax_out || skinny_final || kfin_layer == 0) {
        // K = m is small: direct lower-triangle update (dense middle for softmax)
        dim3 blk(16, 16);
        dim3 grid(ceil_div(n_, 16), ceil_div(n_, 16), nb);
        prof_begin(sh, kTagSmallSyrk, 0, 0);
        dev::small_k_syrk_kernel<<<grid, blk, 0, sh>>>(u, ldu, u_point_rows, w.d[kfin_layer], w.ld[kfin_layer],
                                                       softmax_out ? w.mid : nullptr, m_ * m_, static_cast<int>(n_),
                                                       static_cast<int>(m_), nb, w.h, n_pad_ * n_pad_, n_pad_);
        after_launch(sh);
      } else {
        syrk(kfin_layer, sh);
      }
    }
    const int64_t tot = static_cast<int64_t>(nb) * n_ * n_;
    prof_begin(sh, kTagSymmetrize, 0, 0);
    if (gather)
      dev::syrk_gather_out_kernel<<<dim3(ceil_div(n_, 32), ceil_div(n_, 32), nb), 256, 0, sh>>>(
          gat, h_direct ? w.h : nullptr, n_pad_ * n_pad_, n_pad_, static_cast<int>(n_), o.h_packed ? 1 : 0, o.h);
    else if (o.h_packed)
      dev::pack_lower_kernel<<<dim3(ceil_div(n_, 256), static_cast<unsigned>(n_), nb), 256, 0, sh>>>(
          w.h, 1, 0, n_pad_ * n_pad_, n_pad_, static_cast<int>(n_), o.h);
    else
      dev::symmetrize_out_kernel<<<ceil_div(tot, 256), 256, 0, sh>>>(w.h, nullptr, nullptr, n_pad_ * n_pad_, n_pad_,
                                                                    static_cast<int>(n_), nb, o.h);
    after_launch(sh);
  }
  link(sb, sa);  // join: the evaluation ends on `st`
}

void DeviceNet::run(cudaStream_t st, int nb, const Outputs& o) {
  const int mode = net_.schedule >= 0 ? net_.schedule : dataflow_mode_;
  if (mode == -2 && dataflow_possible(nb, o) && df_choice_.count(choice_key(nb, o)) == 0) autotune(st, nb, o);
  dispatch(st, nb, o);
}

// Auto schedule (mode -1): a fixed rule on the shape, so every process picks
// the same kernels for the same call and the results are reproducible bit
// for bit.  The dataflow launch removes the per-layer barrier of the
// layer-by-layer graph; that pays when the chain is deep (>= 8 layers) AND
// the tangent GEMM tiles of a layer quantise badly onto the SMs (>= 10% of
// the layer-by-layer waves idle), so the barriers cost whole partial waves.
// Fitted to the measured pairs (layered vs dataflow, round 1): c5 (21
// layers, 896 tiles = 6.05 waves, 13.5% idle) 656 vs 713 evals/s -> dataflow;
// c2 (6 layers, 280 tiles) 180.6 vs 173.8 -> layered; c1 (3 layers) layered.
bool DeviceNet::dataflow_rule(int nb) const {
  if (L_ < 8) return false;
  const int64_t row_blocks = n_pad_ / kBM;
  double waves = 0.0, busy = 0.0;
  for (int64_t l = 1; l + 1 < L_; ++l) {
    const int64_t tiles = nb * row_blocks * ceil_div(layers_[static_cast<size_t>(l)].rows, static_cast<int64_t>(kBN));
    const double w = static_cast<double>(tiles) / sm_count_;
    busy += w;
    waves += std::ceil(w);
  }
  return waves > 0.0 && (waves - busy) / waves >= 0.10;
}

// Opt-in measured schedule (mode -2, GBOPT_DATAFLOW=-2 / set_schedule(-2)):
// the first evaluation of a shape runs both schedules twice (warm, then
// timed with events on `st`) and keeps the faster.  Not the default: two
// processes may time differently and pick different kernels.
void DeviceNet::autotune(cudaStream_t st, int nb, const Outputs& o) {
  ensure_transposed();
  dataflow_plan(nb);
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  float ms[2] = {0.f, 0.f};
  try {
    for (int f = 0; f < 2; ++f) {
      df_force_ = f;
      dispatch(st, nb, o);
      CK(cudaEventRecord(e0, st));
      dispatch(st, nb, o);
      CK(cudaEventRecord(e1, st));
      CK(cudaEventSynchronize(e1));
      CK(cudaEventElapsedTime(&ms[f], e0, e1));
    }
  } catch (...) {
    df_force_ = -1;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    throw;
  }
  df_force_ = -1;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  df_choice_[choice_key(nb, o)] = ms[1] < ms[0];
  df_tuned_ms_[choice_key(nb, o)] = {ms[0], ms[1]};
}

void DeviceNet::dispatch(cudaStream_t st, int nb, const Outputs& o) {
  last_dataflow_ = dataflow_ok(nb, o);
  const GraphKey key{nb, o.y, o.j, o.h, o.g, last_dataflow_, o.h_packed};
  if (!net_.use_graphs) {
    launches_ = 0;
    enqueue(st, nb, o);
    last_launches_ = launches_;
    return;
  }
  auto it = graphs_.find(key);
  if (it == graphs_.end()) {
    std::lock_guard<std::recursive_mutex> lock(setup_mutex());
    launches_ = 0;
    cudaGraph_t graph = nullptr;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    try {
      enqueue(st, nb, o);
    } catch (...) {
      cudaStreamEndCapture(st, &graph);
      if (graph) cudaGraphDestroy(graph);
      throw;
    }
    CK(cudaStreamEndCapture(st, &graph));
    GraphEntry e;
    e.launches = launches_;
    // keep the two streams' priorities inside the graph
    const cudaError_t ie = cudaGraphInstantiate(&e.exec, graph, cudaGraphInstantiateFlagUseNodePriority);
    cudaGraphDestroy(graph);
    CK(ie);
    if (graphs_.size() > 16) drop_graphs();
    it = graphs_.emplace(key, e).first;
  }
  CK(cudaGraphLaunch(it->second.exec, st));
  last_launches_ = it->second.launches;
}

// ---------------------------------------------------------------------------
// Persistent single-point forward (fwd_stream.cuh).
// ---------------------------------------------------------------------------
size_t DeviceNet::fwd_stream_smem() const {
  int64_t ycap = 16, max_rows = 1;
  for (const DevLayer& d : layers_) {
    ycap = std::max(ycap, d.ldw);
    max_rows = std::max<int64_t>(max_rows, (d.rows + sm_count_ - 1) / sm_count_ + 1);
  }
  (void)ycap;
  return static_cast<size_t>(dev::kFsStages) * dev::kFsStageBytes +
         8 * static_cast<size_t>(max_rows) * dev::kFsConsumerWarps + 16 * dev::kFsStages;
}

bool DeviceNet::fwd_stream_ok() const {
  if (fwd_stream_mode_ == 0) return false;
  if (L_ > dev::kFsMaxLayers || profiling_) return false;
  int optin = 0;
  if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ordinal_) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return fwd_stream_smem() <= static_cast<size_t>(optin);
}

// x already in ws_.x (point 0); z, y, s1, s2 of every layer to the workspace.
void DeviceNet::launch_fwd_stream(cudaStream_t st) {
  Workspace& w = ws_;
  if (!fs_arrive_) {
    std::lock_guard<std::recursive_mutex> lock(setup_mutex());
    CK(cudaMalloc(&fs_arrive_, sizeof(unsigned) * dev::kFsMaxLayers));
    CK(cudaMemset(fs_arrive_, 0, sizeof(unsigned) * dev::kFsMaxLayers));
    fs_gen_ = 0;
  }
  static thread_local dev::FsParams p;  // ~3 KB, copied at launch
  p.nl = static_cast<int>(L_);
  p.x = w.x;
  p.arrive = fs_arrive_;
  int64_t ycap = 16, max_rows = 1;
  for (int64_t l = 0; l < L_; ++l) {
    const DevLayer& d = layers_[static_cast<size_t>(l)];
    dev::FsLayer& f = p.L[l];
    f.w = d.w;
    f.b = d.b;
    f.z = w.z[static_cast<size_t>(l)];
    f.y = w.y[static_cast<size_t>(l)];
    f.s1 = w.s1[static_cast<size_t>(l)];
    f.s2 = w.s2[static_cast<size_t>(l)];
    f.rows = static_cast<int>(d.rows);
    f.cols = static_cast<int>(d.cols);
    f.ldw = static_cast<int>(d.ldw);
    f.act = d.act == kSoftmax ? kLinear : d.act;
    ycap = std::max(ycap, d.ldw);
    max_rows = std::max<int64_t>(max_rows, (d.rows + sm_count_ - 1) / sm_count_ + 1);
  }
  p.ycap = static_cast<int>(ycap);
  p.max_cta_rows = static_cast<int>(max_rows);
  const size_t smem = fwd_stream_smem();
  if (!fs_attr_set_) {
    CK(cudaFuncSetAttribute(dev::fwd_stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            static_cast<int>(smem)));
    fs_attr_set_ = true;
  }
  // counters are never reset: this launch waits for gen * grid arrivals per
  // layer (no memset launch per call); restart from zero before they wrap
  if (fs_gen_ >= (0xffffffffu / static_cast<unsigned>(sm_count_)) - 1) {
    CK(cudaMemsetAsync(fs_arrive_, 0, sizeof(unsigned) * dev::kFsMaxLayers, st));
    fs_gen_ = 0;
  }
  p.gen = ++fs_gen_;
  void* args[] = {&p};
  prof_begin(st, kTagFwd, 0.0, 0.0);
  CK(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(dev::fwd_stream_kernel), dim3(sm_count_),
                                 dim3(dev::kFsThreads), args, smem, st));
  after_launch(st);
  if (L_ > 0 && layers_[static_cast<size_t>(L_ - 1)].act == kSoftmax) {
    dev::softmax_kernel<<<1, 128, 0, st>>>(w.z[static_cast<size_t>(L_ - 1)], w.y[static_cast<size_t>(L_ - 1)],
                                            static_cast<int>(m_), w.ld[static_cast<size_t>(L_ - 1)], 1);
    after_launch(st);
  }
}

// Host-buffer entry: copy in, evaluate, copy out, synchronise.
void DeviceNet::evaluate_host(int nb, const double* x, const double* lam, double* y, double* jac, double* hess,
                              double* grad, bool hess_packed) {
  const int64_t n = n_, m = m_, hsz = hess_packed ? n_ * (n_ + 1) / 2 : n_ * n_;
  for (int p0 = 0; p0 < nb || p0 == 0; p0 += kMaxChunk) {
    const int c = std::min(kMaxChunk, nb - p0);
    auto at = [p0](auto* ptr, int64_t per) { return ptr ? ptr + per * p0 : ptr; };
    evaluate_host_chunk(c, at(x, n), at(lam, m), at(y, m), at(jac, m * n), at(hess, hsz), at(grad, n), hess_packed);
    if (nb <= 0) break;
  }
}

void DeviceNet::evaluate_device(int nb, const double* dx, const double* dlam, double* dy, double* dj, double* dh,
                                cudaStream_t user) {
  const int64_t n = n_, m = m_;
  for (int p0 = 0; p0 < nb || p0 == 0; p0 += kMaxChunk) {
    const int c = std::min(kMaxChunk, nb - p0);
    auto at = [p0](auto* ptr, int64_t per) { return ptr ? ptr + per * p0 : ptr; };
    evaluate_device_chunk(c, at(dx, n), at(dlam, m), at(dy, m), at(dj, m * n), at(dh, n * n), user);
    if (nb <= 0) break;
  }
}

void DeviceNet::evaluate_host_chunk(int nb, const double* x, const double* lam, double* y, double* jac, double* hess,
                                    double* grad, bool hess_packed) {
  DeviceGuard g(ordinal_);
  ensure_workspace(nb);
  Workspace& w = ws_;
  // Results go to pinned caller buffers directly; pageable ones through a
  // pinned staging area (a pageable D2H runs at a fraction of the PCIe rate)
  // and are written only after the evaluation has completed.
  const size_t hsz = hess_packed ? static_cast<size_t>(n_ * (n_ + 1) / 2) : static_cast<size_t>(n_ * n_);
  struct Out {
    double* dst;
    double* src;
    size_t per_point;
  };
  const Out outs[4] = {{y, w.y_out, static_cast<size_t>(m_)},
                       {jac, w.j_out, static_cast<size_t>(m_ * n_)},
                       {hess, w.h_out, hsz},
                       {grad, w.g_out, static_cast<size_t>(n_)}};
  size_t staged = 0, out_bytes = 0;
  bool pinned[4] = {false, false, false, false};
  for (int i = 0; i < 4; ++i) {
    if (!outs[i].dst) continue;
    cudaPointerAttributes a;
    pinned[i] = cudaPointerGetAttributes(&a, outs[i].dst) == cudaSuccess && a.type == cudaMemoryTypeHost;
    cudaGetLastError();
    if (!pinned[i]) staged += outs[i].per_point * nb;
    out_bytes += sizeof(double) * outs[i].per_point * nb;
  }
  if (staged > stage_cap_) {
    std::lock_guard<std::recursive_mutex> lock(setup_mutex());  // cudaFreeHost synchronises the device
    if (stage_) cudaFreeHost(stage_);
    stage_ = nullptr;
    stage_cap_ = 0;
    CK(cudaHostAlloc(reinterpret_cast<void**>(&stage_), sizeof(double) * staged, cudaHostAllocDefault));
    stage_cap_ = staged;
  }
  // Batched results whose copy-out is a visible share of the call (c4: 94 KB
  // per point against ~0.5 GFLOP of work, ~12%) leave the GPU in chunks:
  // chunk c's D2H on copy_stream_ overlaps chunk c + 1's evaluation, so only
  // the last chunk's copy is exposed.  At ~37 TFLOP/s against ~50 GB/s of
  // PCIe (740 flop/B break-even) a point below ~25k flops per output byte
  // spends > ~3% of its time in the copy; above that (c3: 36k flop/B) the
  // smaller chunks cost more than they hide.  Measured: c4 (4096 points) 4
  // chunks 56.0k -> 59.6k e2e evals/s (8 chunks: 59.4k); c5 (16 points, 8.8k
  // flop/B) 2 chunks 700 -> 717 (4 chunks: 699).
  // Forward only (the line-search residual, forward_trace), opt-in
  // (GBOPT_FWD_STREAM=1): one persistent launch streams every layer's weights
  // (fwd_stream.cuh).  The default is the per-layer GEMV graph below.
  if (nb == 1 && !jac && !hess && !grad && fwd_stream_ok()) {
    launches_ = 0;
    CK(cudaMemcpyAsync(w.x, x, sizeof(double) * n_, cudaMemcpyHostToDevice, stream_));
    static const bool fwd_events = std::getenv("GBOPT_FWD_EVENTS") != nullptr;  // diagnostics: device time
    cudaEvent_t fe0 = nullptr, fe1 = nullptr;
    if (fwd_events) {
      CK(cudaEventCreate(&fe0));
      CK(cudaEventCreate(&fe1));
      CK(cudaEventRecord(fe0, stream_));
    }
    launch_fwd_stream(stream_);
    if (fwd_events) {
      CK(cudaEventRecord(fe1, stream_));
      CK(cudaEventSynchronize(fe1));
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, fe0, fe1));
      std::fprintf(stderr, "GBOPT_FWD_EVENTS stream %.4f ms\n", ms);
      cudaEventDestroy(fe0);
      cudaEventDestroy(fe1);
    }
    if (y) {
      double* d = pinned[0] ? y : stage_;
      CK(cudaMemcpyAsync(d, w.y[static_cast<size_t>(L_ - 1)], sizeof(double) * m_, cudaMemcpyDeviceToHost, stream_));
    }
    CK(cudaStreamSynchronize(stream_));
    if (y && !pinned[0]) std::memcpy(y, stage_, sizeof(double) * m_);
    last_launches_ = launches_;
    return;
  }
  double flops = 0.0;  // F_jac + F_hess per point
  for (size_t l = 0; l < layers_.size(); ++l) {
    if (l > 0) flops += 2.0 * static_cast<double>(layers_[l].rows * layers_[l].cols * n_);
    if (layers_[l].act != kLinear) flops += static_cast<double>(layers_[l].rows * n_ * (n_ + 1));
  }
  const double bytes_pp = static_cast<double>(out_bytes) / nb;
  int chunks = 1;
  if (out_bytes >= (size_t(64) << 20) && flops < 25000.0 * bytes_pp) chunks = nb >= 128 ? 4 : (nb >= 16 ? 2 : 1);
  if (const char* e = std::getenv("GBOPT_HOST_CHUNKS")) chunks = std::max(1, std::min(nb, std::atoi(e)));
  const int per = (nb + chunks - 1) / chunks;
  while (static_cast<int>(chunk_ev_.size()) < chunks) {
    cudaEvent_t e;
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    chunk_ev_.push_back(e);
  }
  CK(cudaEventRecord(ev_in_, stream_));
  CK(cudaStreamWaitEvent(copy_stream_, ev_in_, 0));  // no copy of this call overtakes earlier work
  int ci = 0;
  for (int c0 = 0; c0 < nb; c0 += per, ++ci) {
    const int nbc = std::min(per, nb - c0);
    Outputs o;
    o.y = y ? w.y_out + static_cast<size_t>(c0) * m_ : nullptr;
    o.j = jac ? w.j_out + static_cast<size_t>(c0) * m_ * n_ : nullptr;
    o.h = hess ? w.h_out + static_cast<size_t>(c0) * hsz : nullptr;
    o.g = grad ? w.g_out + static_cast<size_t>(c0) * n_ : nullptr;
    o.h_packed = hess_packed;
    prepare(nbc, o);
    CK(cudaMemcpy2DAsync(w.x, sizeof(double) * w.ld_in, x + static_cast<size_t>(c0) * n_, sizeof(double) * n_,
                         sizeof(double) * n_, nbc, cudaMemcpyHostToDevice, stream_));
    if (lam)
      CK(cudaMemcpy2DAsync(w.lam, sizeof(double) * w.ld_lam, lam + static_cast<size_t>(c0) * m_, sizeof(double) * m_,
                           sizeof(double) * m_, nbc, cudaMemcpyHostToDevice, stream_));
    static const bool fwd_events = std::getenv("GBOPT_FWD_EVENTS") != nullptr;  // diagnostics: device time
    cudaEvent_t fe0 = nullptr, fe1 = nullptr;
    if (fwd_events) {
      CK(cudaEventCreate(&fe0));
      CK(cudaEventCreate(&fe1));
      CK(cudaEventRecord(fe0, stream_));
    }
    run(stream_, nbc, o);
    if (fwd_events) {
      CK(cudaEventRecord(fe1, stream_));
      CK(cudaEventSynchronize(fe1));
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, fe0, fe1));
      std::fprintf(stderr, "GBOPT_FWD_EVENTS run %.4f ms\n", ms);
      cudaEventDestroy(fe0);
      cudaEventDestroy(fe1);
    }
    cudaStream_t cs = chunks > 1 ? copy_stream_ : stream_;
    if (chunks > 1) {
      CK(cudaEventRecord(chunk_ev_[static_cast<size_t>(ci)], stream_));
      CK(cudaStreamWaitEvent(copy_stream_, chunk_ev_[static_cast<size_t>(ci)], 0));
    }
    size_t off = 0;
    for (int i = 0; i < 4; ++i) {
      if (!outs[i].dst) continue;
      const size_t pp = outs[i].per_point;
      double* d = pinned[i] ? outs[i].dst + static_cast<size_t>(c0) * pp : stage_ + off + static_cast<size_t>(c0) * pp;
      CK(cudaMemcpyAsync(d, outs[i].src + static_cast<size_t>(c0) * pp, sizeof(double) * pp * nbc,
                         cudaMemcpyDeviceToHost, cs));
      if (!pinned[i]) off += pp * nb;
    }
  }
  CK(cudaStreamSynchronize(stream_));
  if (chunks > 1) CK(cudaStreamSynchronize(copy_stream_));
  size_t off = 0;
  for (int i = 0; i < 4; ++i) {
    if (!outs[i].dst || pinned[i]) continue;
    std::memcpy(outs[i].dst, stage_ + off, sizeof(double) * outs[i].per_point * nb);
    off += outs[i].per_point * nb;
  }
}

// Device-buffer entry: ordered after / before `user` stream, no host sync.
void DeviceNet::evaluate_device_chunk(int nb, const double* dx, const double* dlam, double* dy, double* dj,
                                      double* dh, cudaStream_t user) {
  DeviceGuard g(ordinal_);
  ensure_workspace(nb);
  Workspace& w = ws_;
  {
    Outputs po;
    po.y = dy;
    po.j = dj;
    po.h = dh;
    prepare(nb, po);
  }
  CK(cudaEventRecord(ev_in_, user));
  CK(cudaStreamWaitEvent(stream_, ev_in_, 0));
  CK(cudaMemcpy2DAsync(w.x, sizeof(double) * w.ld_in, dx, sizeof(double) * n_, sizeof(double) * n_, nb,
                       cudaMemcpyDeviceToDevice, stream_));
  if (dlam)
    CK(cudaMemcpy2DAsync(w.lam, sizeof(double) * w.ld_lam, dlam, sizeof(double) * m_, sizeof(double) * m_, nb,
                         cudaMemcpyDeviceToDevice, stream_));
  Outputs o;
  o.y = dy;
  o.j = dj;
  o.h = dh;
  o.g = nullptr;
  run(stream_, nb, o);
  CK(cudaEventRecord(ev_out_, stream_));
  CK(cudaStreamWaitEvent(user, ev_out_, 0));
}

void DeviceNet::copy_intermediate(const char* name, int layer, int nb, double* out) {
  DeviceGuard g(ordinal_);
  if (layer < 0 || layer >= L_) throw StructuralError("copy_intermediate: layer out of range");
  if (nb <= 0 || nb > ws_cap_) throw StructuralError("copy_intermediate: batch exceeds the last evaluation");
  const std::string s(name);
  const size_t l = static_cast<size_t>(layer);
  double* src = s == "z" ? ws_.z[l] : s == "y" ? ws_.y[l] : s == "s1" ? ws_.s1[l] : s == "s2" ? ws_.s2[l]
              : s == "ybar" ? ws_.ybar[l] : s == "gz" ? ws_.gz[l] : s == "d" ? ws_.d[l] : nullptr;
  if (!src) throw StructuralError("copy_intermediate: unknown buffer " + s);
  CK(cudaStreamSynchronize(stream_));
  CK(cudaMemcpy2D(out, sizeof(double) * layers_[l].rows, src, sizeof(double) * ws_.ld[l],
                  sizeof(double) * layers_[l].rows, nb, cudaMemcpyDeviceToHost));
}

// ---------------------------------------------------------------------------
// Persistent dataflow path (dataflow.cuh): plan construction and launch.
// ---------------------------------------------------------------------------
// Shapes the dataflow launch can run (independent of the schedule mode).
bool DeviceNet::dataflow_possible(int nb, const Outputs& o) const {
  if (!concurrent_) return false;
  if (o.h == nullptr || o.g != nullptr) return false;  // the full (y, J, H) oracle only
  if (L_ < 2 || m_ > dev::kSkMB || layers_[static_cast<size_t>(L_ - 1)].act == kSoftmax) return false;
  if (6 * L_ + 1 > dev::kDfMaxMaps) return false;  // TMA descriptors in the kernel parameters
  if (nb < 1 || nb > kBM) return false;  // FWD / ADJ items hold all points in one M tile
  if (L_ >= 3 && static_cast<int64_t>(ws_.t.size()) < L_ - 2) return false;  // one T buffer per tangent layer
  return true;
}

bool DeviceNet::dataflow_ok(int nb, const Outputs& o) const {
  int mode = net_.schedule >= 0 ? net_.schedule : dataflow_mode_;
  if (df_force_ >= 0) mode = df_force_;
  if (mode == 0 || !dataflow_possible(nb, o)) return false;
  if (mode == 1) return true;
  if (mode == -2) {  // measured: what the first evaluation of this shape timed (autotune in run())
    const auto c = df_choice_.find(choice_key(nb, o));
    return c != df_choice_.end() && c->second;
  }
  return dataflow_rule(nb);  // auto: the shape rule
}

// One eager dataflow evaluation with the per-item trace on: rows of
// {kind, job, point, tm, tn, kb0, kb1, sm, t_claim, t_ready, t_begin, t_end}
// (times in us from the earliest claim), in claim order.
std::vector<double> DeviceNet::dataflow_trace(int nb, const double* dx, const double* dlam) {
  DeviceGuard g(ordinal_);
  ensure_workspace(nb);
  Workspace& w = ws_;
  Outputs o;
  o.y = w.y_out;
  o.j = w.j_out;
  o.h = w.h_out;
  if (!dataflow_ok(nb, o)) throw StructuralError("dataflow_trace: the dataflow schedule does not apply");
  prepare(nb, o);
  DfPlan& P = df_plans_.at(nb);
  CK(cudaDeviceSynchronize());
  CK(cudaMalloc(&df_trace_, sizeof(unsigned long long) * 4 * P.n_items));
  CK(cudaMalloc(&df_trace_sm_, sizeof(int) * P.n_items));
  CK(cudaMemcpy2D(w.x, sizeof(double) * w.ld_in, dx, sizeof(double) * n_, sizeof(double) * n_, nb,
                  cudaMemcpyDeviceToDevice));
  CK(cudaMemcpy2D(w.lam, sizeof(double) * w.ld_lam, dlam, sizeof(double) * m_, sizeof(double) * m_, nb,
                  cudaMemcpyDeviceToDevice));
  std::vector<unsigned long long> tr(static_cast<size_t>(4) * P.n_items);
  std::vector<int> sm(static_cast<size_t>(P.n_items));
  std::vector<dev::DfItem> items(static_cast<size_t>(P.n_items));
  std::vector<dev::DfJob> jobs;
  try {
    enqueue_dataflow(stream_, nb, o);
    CK(cudaStreamSynchronize(stream_));
    CK(cudaMemcpy(tr.data(), df_trace_, sizeof(unsigned long long) * tr.size(), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(sm.data(), df_trace_sm_, sizeof(int) * sm.size(), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(items.data(), P.items, sizeof(dev::DfItem) * items.size(), cudaMemcpyDeviceToHost));
    int nj = 0;
    for (const auto& it : items) nj = std::max(nj, it.job + 1);
    jobs.resize(static_cast<size_t>(nj));
    CK(cudaMemcpy(jobs.data(), P.jobs, sizeof(dev::DfJob) * jobs.size(), cudaMemcpyDeviceToHost));
  } catch (...) {
    cudaFree(df_trace_);
    cudaFree(df_trace_sm_);
    df_trace_ = nullptr;
    df_trace_sm_ = nullptr;
    throw;
  }
  cudaFree(df_trace_);
  cudaFree(df_trace_sm_);
  df_trace_ = nullptr;
  df_trace_sm_ = nullptr;
  unsigned long long t0 = ~0ull;
  for (int i = 0; i < P.n_items; ++i) t0 = std::min(t0, tr[static_cast<size_t>(4 * i)]);
  std::vector<double> out;
  out.reserve(static_cast<size_t>(12) * P.n_items);
  for (int i = 0; i < P.n_items; ++i) {
    const dev::DfItem& it = items[static_cast<size_t>(i)];
    out.push_back(jobs[static_cast<size_t>(it.job)].kind);
    out.push_back(it.job);
    out.push_back(it.point);
    out.push_back(it.tm);
    out.push_back(it.tn);
    out.push_back(it.kb0);
    out.push_back(it.kb1);
    out.push_back(sm[static_cast<size_t>(i)]);
    for (int k = 0; k < 4; ++k) out.push_back(1e-3 * static_cast<double>(tr[static_cast<size_t>(4 * i + k)] - t0));
  }
  return out;
}

void DeviceNet::free_plans() {
  for (auto& kv : df_plans_) {
    DfPlan& p = kv.second;
    cudaFree(p.items);
    cudaFree(p.jobs);
    cudaFree(p.counters);
    cudaFree(p.hslots);
  }
  df_plans_.clear();
}

// The item list of one dataflow launch, ordered by a list-scheduling
// simulation of the GPU (sm_count workers, priority = longest remaining
// path), so the order is topological and claims the critical path first.
DfPlan& DeviceNet::dataflow_plan(int nb) {
  auto found = df_plans_.find(nb);
  if (found != df_plans_.end()) return found->second;
  std::lock_guard<std::recursive_mutex> lock(setup_mutex());
  Workspace& w = ws_;
  const int L = static_cast<int>(L_);
  const int tiles_m = static_cast<int>(n_pad_ / kBM);
  auto rows = [&](int l) { return layers_[static_cast<size_t>(l)].rows; };
  auto kbs = [&](int64_t k) { return ceil_div(k, kBK); };
  const int ring = static_cast<int>(w.t.size());
  auto t_buf = [&](int l) -> double* { return w.t[static_cast<size_t>((l - 1) % ring)]; };
  auto t_point_rows = [&](int l) -> int64_t { return l == 0 ? 0 : n_pad_; };

  // ---- TMA descriptors (copied to device memory; jobs point at them) ----
  std::vector<CUtensorMap> maps;
  auto map_id = [&](const CUtensorMap& m) {
    for (size_t i = 0; i < maps.size(); ++i)
      if (std::memcmp(&maps[i], &m, sizeof(CUtensorMap)) == 0) return static_cast<int>(i);
    if (maps.size() >= static_cast<size_t>(dev::kDfMaxMaps)) throw StructuralError("dataflow: too many TMA descriptors");
    maps.push_back(m);
    return static_cast<int>(maps.size()) - 1;
  };
  std::vector<dev::DfJob> jobs;
  std::vector<std::pair<int, int>> job_maps;
  auto add_job = [&](const dev::DfJob& j, int ma, int mb) {
    jobs.push_back(j);
    job_maps.emplace_back(ma, mb);
    return static_cast<int>(jobs.size()) - 1;
  };

  // ---- counters ----
  int nc = 1;  // [0] = claim counter
  std::vector<int> fwd_cnt(static_cast<size_t>(L)), adj_cnt(static_cast<size_t>(L), 0), row_base(static_cast<size_t>(L), 0);
  for (int l = 0; l < L; ++l) fwd_cnt[static_cast<size_t>(l)] = nc++;
  for (int l = 1; l < L; ++l) adj_cnt[static_cast<size_t>(l)] = nc++;
  for (int l = 1; l + 1 < L; ++l) {
    row_base[static_cast<size_t>(l)] = nc;
    nc += nb * tiles_m;
  }
  // SYRK tiles over the lower triangle: square 112 x 112 blocks (tn <= tm;
  // 87.6% useful work at n = 784 against 76.7% for 112 x 128 tiles), or
  // 112 x 128 tiles with GBOPT_DF_SQ=0
  const bool sq = df_square_;
  const int stn = sq ? kBM : kBN;
  std::vector<int2> stiles;
  for (int tm = 0; tm * kBM < n_; ++tm)
    for (int tn = 0; tn * stn < n_; ++tn)
      if (static_cast<int64_t>(tn) * stn <= static_cast<int64_t>(tm) * kBM + kBM - 1) stiles.push_back(make_int2(tm, tn));
  const int n_st = static_cast<int>(stiles.size());
  std::vector<int> syrk_layers, pieces;
  int slots = 1;
  for (int l = 0; l + 1 < L; ++l) {
    if (layers_[static_cast<size_t>(l)].act == kLinear) continue;
    syrk_layers.push_back(l);
    const int p = std::max(1, std::min(8, static_cast<int>(std::lround(kbs(rows(l)) / 64.0))));
    pieces.push_back(p);
    slots = std::max(slots, p);
  }
  const int hcnt_base = nc;
  nc += slots * nb * n_st;
  auto hcnt = [&](int q, int p, int t) { return hcnt_base + (q * nb + p) * n_st + t; };

  // ---- items (created in a topological order) ----
  const double sm_rate = 35.0e12 / 148.0;                     // FP64 flop/s per SM (DMMA)
  const double t_kb = 2.0 * kBM * kBN * kBK / sm_rate * 1e3;   // ms per full k-block
  const double t_kb_mem = 16384.0 / 60.0e9 * 1e3;             // ms per streamed 16 KB B box
  const double t_item = 2.0e-3;                                // ms per item (epilogue, hand-off)
  struct Node {
    dev::DfItem it;
    double cost;
  };
  std::vector<Node> nodes;
  auto add_item = [&](int job, int point, int tm, int tn, int kb0, int kb1, int slot, int sig,
                      std::initializer_list<std::pair<int, int>> waits, double cost) {
    Node nd{};
    nd.it.job = job;
    nd.it.point = point;
    nd.it.tm = tm;
    nd.it.tn = tn;
    nd.it.kb0 = kb0;
    nd.it.kb1 = kb1;
    nd.it.slot = slot;
    nd.it.sig = sig;
    for (const auto& wt : waits) {
      if (wt.second <= 0) continue;
      bool dup = false;
      for (int i = 0; i < nd.it.nwait; ++i) dup = dup || (nd.it.widx[i] == wt.first && nd.it.wtgt[i] >= wt.second);
      if (dup) continue;
      if (nd.it.nwait >= dev::kDfMaxWait) throw StructuralError("dataflow: too many dependencies");
      nd.it.widx[nd.it.nwait] = wt.first;
      nd.it.wtgt[nd.it.nwait] = wt.second;
      ++nd.it.nwait;
    }
    nd.cost = cost;
    nodes.push_back(nd);
  };
  // FWD / ADJ A operands (points x K): a box of round_up(nb, 8) rows, not 112
  const int a_rows = static_cast<int>(std::min<int64_t>(kBM, round_up(nb, 8)));
  const int a_bytes_small = a_rows * kBK * 8;
  const int tm_x = map_id(make_tmap(w.x, n_, ws_cap_, w.ld_in, a_rows));
  std::vector<int> nfwd(static_cast<size_t>(L)), nadj(static_cast<size_t>(L), 0);
  const double gemv_mma = std::min(1.0, ceil_div(nb, 8) / 14.0) * t_kb;
  double flops = 0, bytes = 0;
  // forward chain (+ the adjoint seed in the top layer's epilogue)
  for (int l = 0; l < L; ++l) {
    const DevLayer& d = layers_[static_cast<size_t>(l)];
    dev::DfJob j{};
    j.kind = dev::kDfFwd;
    j.act = d.act;
    j.m_valid = nb;
    j.n_valid = static_cast<int>(d.rows);
    j.bias = d.b;
    j.z = w.z[static_cast<size_t>(l)];
    j.y = w.y[static_cast<size_t>(l)];
    j.s1 = w.s1[static_cast<size_t>(l)];
    j.s2 = w.s2[static_cast<size_t>(l)];
    j.ld = w.ld[static_cast<size_t>(l)];
    if (l == L - 1) {
      j.lam = w.lam;
      j.ld_lam = w.ld_lam;
      j.gz_seed = w.gz[static_cast<size_t>(l)];
      j.d_seed = w.d[static_cast<size_t>(l)];
    }
    j.a_bytes = a_bytes_small;
    j.b_bytes = dev::kBBytes;
    j.b_tile = kBN;
    const int job = add_job(j, l == 0 ? tm_x : map_id(make_tmap(w.y[static_cast<size_t>(l - 1)], rows(l - 1), ws_cap_,
                                                                  w.ld[static_cast<size_t>(l - 1)], a_rows)),
                            map_id(d.tm_w));
    nfwd[static_cast<size_t>(l)] = ceil_div(d.rows, kBN);
    const int kb = kbs(d.cols);
    for (int tn = 0; tn < nfwd[static_cast<size_t>(l)]; ++tn)
      add_item(job, 0, 0, tn, 0, kb, 0, fwd_cnt[static_cast<size_t>(l)],
               {{l > 0 ? fwd_cnt[static_cast<size_t>(l - 1)] : 0, l > 0 ? nfwd[static_cast<size_t>(l - 1)] : 0}},
               kb * std::max(t_kb_mem, gemv_mma) + t_item);
    flops += 2.0 * d.rows * d.cols * nb;
    bytes += 8.0 * d.rows * d.cols;
  }
  // adjoint chain down to ybar_0 / d_0 (layer 0's input gradient is not needed)
  for (int l = L - 1; l >= 1; --l) {
    const DevLayer& d = layers_[static_cast<size_t>(l)];
    dev::DfJob j{};
    j.kind = dev::kDfAdj;
    j.m_valid = nb;
    j.n_valid = static_cast<int>(d.cols);
    j.ybar = w.ybar[static_cast<size_t>(l - 1)];
    j.gz = w.gz[static_cast<size_t>(l - 1)];
    j.d = w.d[static_cast<size_t>(l - 1)];
    j.s1i = w.s1[static_cast<size_t>(l - 1)];
    j.s2i = w.s2[static_cast<size_t>(l - 1)];
    j.ld = w.ld[static_cast<size_t>(l - 1)];
    j.a_bytes = a_bytes_small;
    j.b_bytes = dev::kBBytes;
    j.b_tile = kBN;
    const int job = add_job(j, map_id(make_tmap(w.gz[static_cast<size_t>(l)], rows(l), ws_cap_ * std::max<int64_t>(m_, 1),
                                                w.ld[static_cast<size_t>(l)], a_rows)),
                            map_id(d.tm_wt));
    nadj[static_cast<size_t>(l)] = ceil_div(d.cols, kBN);
    const int kb = kbs(d.rows);
    const std::pair<int, int> dep = l == L - 1 ? std::make_pair(fwd_cnt[static_cast<size_t>(L - 1)], nfwd[static_cast<size_t>(L - 1)])
                                               : std::make_pair(adj_cnt[static_cast<size_t>(l + 1)], nadj[static_cast<size_t>(l + 1)]);
    for (int tn = 0; tn < nadj[static_cast<size_t>(l)]; ++tn)
      add_item(job, 0, 0, tn, 0, kb, 0, adj_cnt[static_cast<size_t>(l)], {dep},
               kb * std::max(t_kb_mem, gemv_mma) + t_item);
    flops += 2.0 * d.rows * d.cols * nb;
    bytes += 8.0 * d.rows * d.cols;
  }
  // tangent GEMMs T_{l+1} = T_l diag(sigma'_l) W_{l+1}^T, l + 1 <= L - 2, and
  // the SYRK pieces of layer l once T_l exists
  std::vector<int> ntiles_n(static_cast<size_t>(L), 0);
  size_t si = 0;
  for (int l = 0; l + 1 < L; ++l) {
    if (l + 2 < L) {
      const DevLayer& dn = layers_[static_cast<size_t>(l + 1)];
      dev::DfJob j{};
      j.kind = dev::kDfGemm;
      j.a_bytes = dev::kABytes;
      j.b_bytes = dev::kBBytes;
      j.b_tile = kBN;
      // l >= 1: the pre-scaled S_l = T_l diag(sigma'_l) as A (no multiply in
      // the k-loop); l == 0: T_0 = W_0^T with sigma'_0 applied per fragment
      j.scale = l == 0 ? w.s1[0] : nullptr;
      j.s_stride = w.ld[static_cast<size_t>(l)];
      j.a_point_rows = t_point_rows(l);
      const bool next_gemm = l + 3 < L;  // a GEMM (l+1 -> l+2) reads S_{l+1}
      if (next_gemm) {
        j.c2 = w.s[static_cast<size_t>(l % ring)];
        j.c2_scale = w.s1[static_cast<size_t>(l + 1)];
        j.c2_scale_stride = w.ld[static_cast<size_t>(l + 1)];
      }
      j.m_valid = static_cast<int>(n_pad_);
      j.n_valid = static_cast<int>(dn.rows);
      j.c = t_buf(l + 1);
      j.c_point_stride = n_pad_ * ldt_;
      j.ldc = ldt_;
      const int ma = l == 0 ? map_id(tm_t0_a_) : map_id(w.tm_s_a[static_cast<size_t>(l)]);
      const int job = add_job(j, ma, map_id(dn.tm_w));
      const int tn_n = ceil_div(dn.rows, kBN);
      ntiles_n[static_cast<size_t>(l + 1)] = tn_n;
      const int kb = kbs(dn.cols);
      // groups of df_group_ row blocks sweep the N tiles together: the
      // W_{l+1} tile of one tn is read by the group's CTAs at about the same
      // time (L2 reuse), and a group's rows complete after group * tn_n
      // tiles, so the next layer can start on them early
      for (int p = 0; p < nb; ++p)
        for (int g0 = 0; g0 < tiles_m; g0 += df_group_)
          for (int tn = 0; tn < tn_n; ++tn)
            for (int tm = g0; tm < std::min(tiles_m, g0 + df_group_); ++tm)
            add_item(job, p, tm, tn, 0, kb, 0, row_base[static_cast<size_t>(l + 1)] + p * tiles_m + tm,
                     {{fwd_cnt[static_cast<size_t>(l)], nfwd[static_cast<size_t>(l)]},
                      {l >= 1 ? row_base[static_cast<size_t>(l)] + p * tiles_m + tm : 0,
                       l >= 1 ? ntiles_n[static_cast<size_t>(l)] : 0},
                      {next_gemm ? fwd_cnt[static_cast<size_t>(l + 1)] : 0,
                       next_gemm ? nfwd[static_cast<size_t>(l + 1)] : 0}},
                     kb * t_kb + t_item);
      flops += 2.0 * n_ * dn.rows * dn.cols * nb;
    }
    if (si < syrk_layers.size() && syrk_layers[si] == l) {
      const DevLayer& d = layers_[static_cast<size_t>(l)];
      dev::DfJob j{};
      j.kind = dev::kDfSyrk;
      j.a_bytes = dev::kABytes;
      j.b_bytes = sq ? dev::kABytes : dev::kBBytes;
      j.b_tile = stn;
      j.scale = w.d[static_cast<size_t>(l)];
      j.s_stride = w.ld[static_cast<size_t>(l)];
      j.a_point_rows = t_point_rows(l);
      j.b_point_rows = t_point_rows(l);
      j.m_valid = static_cast<int>(n_);
      j.n_valid = static_cast<int>(n_);
      j.c = nullptr;  // patched: the plan's H slots
      j.c_point_stride = n_pad_ * n_pad_;
      j.ldc = n_pad_;
      const int ma = l == 0 ? map_id(tm_t0_a_) : map_id(w.tm_t_a[static_cast<size_t>(l)]);
      const int mb = sq ? ma : l == 0 ? map_id(tm_t0_b_) : map_id(w.tm_t_b[static_cast<size_t>(l)]);
      const int job = add_job(j, ma, mb);
      const int kb = kbs(d.rows);
      const int np = pieces[si];
      // d_l comes from ADJ(l+1) (its epilogue), T_l rows from GEMM(l-1)
      const std::pair<int, int> ddep{adj_cnt[static_cast<size_t>(l + 1)], nadj[static_cast<size_t>(l + 1)]};
      for (int p = 0; p < nb; ++p)
        for (int t = 0; t < n_st; ++t) {
          const int ti = stiles[static_cast<size_t>(t)].x, tj = stiles[static_cast<size_t>(t)].y;
          const int b0 = std::min(tiles_m - 1, tj * stn / kBM), b1 = std::min(tiles_m - 1, (tj * stn + stn - 1) / kBM);
          auto rdep = [&](int blk) -> std::pair<int, int> {
            if (l == 0) return {0, 0};
            return {row_base[static_cast<size_t>(l)] + p * tiles_m + blk, ntiles_n[static_cast<size_t>(l)]};
          };
          for (int q = 0; q < np; ++q) {
            // ordinal of layer l among the SYRK layers that use slot q
            int ord = 0;
            for (size_t u = 0; u < si; ++u) ord += pieces[u] > q ? 1 : 0;
            const int k0 = static_cast<int>(static_cast<int64_t>(kb) * q / np);
            const int k1 = static_cast<int>(static_cast<int64_t>(kb) * (q + 1) / np);
            add_item(job, p, ti, tj, k0, k1, q, hcnt(q, p, t),
                     {ddep, rdep(ti), rdep(b0), rdep(b1), {hcnt(q, p, t), ord}}, (k1 - k0) * t_kb + t_item);
          }
        }
      flops += static_cast<double>(d.rows) * n_ * (n_ + 1) * nb;
      ++si;
    }
  }

  // ---- list-scheduling simulation -> claim order ----
  const size_t N = nodes.size();
  std::vector<double> rank(N, 0.0), cmax(static_cast<size_t>(nc), 0.0);
  for (size_t i = N; i-- > 0;) {
    rank[i] = nodes[i].cost + cmax[static_cast<size_t>(nodes[i].it.sig)];
    for (int k = 0; k < nodes[i].it.nwait; ++k) {
      double& c = cmax[static_cast<size_t>(nodes[i].it.widx[k])];
      c = std::max(c, rank[i]);
    }
  }
  std::vector<std::vector<std::pair<int, int>>> waiters(static_cast<size_t>(nc));
  std::vector<int> pending(N, 0), count(static_cast<size_t>(nc), 0);
  for (size_t i = 0; i < N; ++i) {
    pending[i] = nodes[i].it.nwait;
    for (int k = 0; k < nodes[i].it.nwait; ++k)
      waiters[static_cast<size_t>(nodes[i].it.widx[k])].emplace_back(static_cast<int>(i), nodes[i].it.wtgt[k]);
  }
  auto by_rank = [&](int a, int b) { return rank[static_cast<size_t>(a)] < rank[static_cast<size_t>(b)] ||
                                            (rank[static_cast<size_t>(a)] == rank[static_cast<size_t>(b)] && a > b); };
  std::priority_queue<int, std::vector<int>, decltype(by_rank)> ready(by_rank);
  using Ev = std::pair<double, int>;
  std::priority_queue<Ev, std::vector<Ev>, std::greater<Ev>> events;
  for (size_t i = 0; i < N; ++i)
    if (pending[i] == 0) ready.push(static_cast<int>(i));
  std::vector<int> order;
  order.reserve(N);
  int free_w = sm_count_;
  double now = 0.0;
  while (order.size() < N) {
    while (free_w > 0 && !ready.empty()) {
      const int i = ready.top();
      ready.pop();
      order.push_back(i);
      events.emplace(now + nodes[static_cast<size_t>(i)].cost, i);
      --free_w;
    }
    if (events.empty()) throw StructuralError("dataflow: dependency cycle in the item list");
    const Ev e = events.top();
    events.pop();
    now = e.first;
    ++free_w;
    const int sig = nodes[static_cast<size_t>(e.second)].it.sig;
    const int c = ++count[static_cast<size_t>(sig)];
    for (const auto& wt : waiters[static_cast<size_t>(sig)])
      if (wt.second == c && --pending[static_cast<size_t>(wt.first)] == 0) ready.push(wt.first);
  }
  while (!events.empty()) {
    now = events.top().first;
    events.pop();
  }

  // ---- self-check of the claim order (the kernel's deadlock freedom rests
  // on it): every wait must be satisfiable by items claimed before the
  // waiting one, and every counter must reach its largest target ----
  {
    std::vector<int> seen(static_cast<size_t>(nc), 0), total(static_cast<size_t>(nc), 0);
    for (size_t i = 0; i < N; ++i) ++total[static_cast<size_t>(nodes[i].it.sig)];
    for (size_t i = 0; i < N; ++i) {
      const dev::DfItem& it = nodes[static_cast<size_t>(order[i])].it;
      for (int k = 0; k < it.nwait; ++k)
        if (seen[static_cast<size_t>(it.widx[k])] < it.wtgt[k])
          throw StructuralError("dataflow: claim order violates a dependency (internal error)");
      if (it.sig <= 0 || it.sig >= nc) throw StructuralError("dataflow: item without a valid signal counter");
      ++seen[static_cast<size_t>(it.sig)];
    }
  }

  // ---- upload ----
  DfPlan plan;
  plan.nb = nb;
  plan.n_items = static_cast<int>(N);
  plan.n_counters = nc;
  plan.slots = slots;
  plan.slot_stride = static_cast<int64_t>(nb) * n_pad_ * n_pad_;
  plan.flops = flops;
  plan.bytes = bytes;
  plan.sim_ms = now;
  plan.maps = maps;
  CK(cudaMalloc(&plan.hslots, sizeof(double) * static_cast<size_t>(plan.slot_stride) * slots));
  for (size_t i = 0; i < jobs.size(); ++i) {
    jobs[i].ta = job_maps[i].first;
    jobs[i].tb = job_maps[i].second;
    if (jobs[i].kind == dev::kDfSyrk) {
      jobs[i].c = plan.hslots;
      jobs[i].slot_stride = plan.slot_stride;
    }
  }
  CK(cudaMalloc(&plan.jobs, sizeof(dev::DfJob) * jobs.size()));
  CK(cudaMemcpy(plan.jobs, jobs.data(), sizeof(dev::DfJob) * jobs.size(), cudaMemcpyHostToDevice));
  std::vector<dev::DfItem> items(N);
  for (size_t i = 0; i < N; ++i) items[i] = nodes[static_cast<size_t>(order[i])].it;
  CK(cudaMalloc(&plan.items, sizeof(dev::DfItem) * N));
  CK(cudaMemcpy(plan.items, items.data(), sizeof(dev::DfItem) * N, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&plan.counters, sizeof(int) * static_cast<size_t>(nc)));
  return df_plans_.emplace(nb, plan).first->second;
}

// One evaluation on the dataflow path: counters/H slots reset, the
// persistent launch, then the final layer (U, J, output curvature) and the
// symmetrise pass.
void DeviceNet::enqueue_dataflow(cudaStream_t st, int nb, const Outputs& o) {
  auto found = df_plans_.find(nb);
  if (found == df_plans_.end()) throw StructuralError("dataflow plan missing (prepare() not called)");
  DfPlan& P = found->second;
  Workspace& w = ws_;
  const int L = static_cast<int>(L_);
  CK(cudaMemsetAsync(P.counters, 0, sizeof(int) * static_cast<size_t>(P.n_counters), st));
  CK(cudaMemsetAsync(P.hslots, 0, sizeof(double) * static_cast<size_t>(P.slot_stride) * P.slots, st));
  thread_local dev::DfParams prm;  // 24 KB: not on the stack (copied at launch)
  std::memset(&prm, 0, sizeof(prm));
  std::copy(P.maps.begin(), P.maps.end(), prm.maps);
  prm.items = P.items;
  prm.n_items = P.n_items;
  prm.jobs = P.jobs;
  prm.counters = P.counters;
  prm.trace = df_trace_;
  prm.trace_sm = df_trace_sm_;
  prof_begin(st, kTagDataflow, P.flops, P.bytes);
  const int grid = std::min(sm_count_, P.n_items);
  dev::df_kernel<<<grid, dev::kThreads, dev::kDfSmemBytes, st>>>(prm);
  after_launch(st);
  if (o.y)
    CK(cudaMemcpy2DAsync(o.y, sizeof(double) * m_, w.y[static_cast<size_t>(L - 1)],
                         sizeof(double) * w.ld[static_cast<size_t>(L - 1)], sizeof(double) * m_, nb,
                         cudaMemcpyDeviceToDevice, st));
  // final layer: U = T_{L-2} diag(sigma'_{L-2}) W_{L-1}^T (m <= 16 outputs)
  const int l = L - 2;
  const double* tl = l == 0 ? t0_ : w.t[static_cast<size_t>((l - 1) % static_cast<int>(w.t.size()))];
  launch_skinny(st, nb, tl, l == 0 ? ldt0_ : ldt_, l == 0 ? 0 : n_pad_, l);
  const DevLayer& df = layers_[static_cast<size_t>(L - 1)];
  if (o.j) {
    const int64_t tot = static_cast<int64_t>(nb) * n_;
    prof_begin(st, kTagJacOut, 0, 0);
    dev::jacobian_out_kernel<<<ceil_div(tot, 128), 128, 0, st>>>(w.u, dev::kSkMB, n_pad_, w.s1[static_cast<size_t>(L - 1)],
                                                                 w.y[static_cast<size_t>(L - 1)],
                                                                 w.ld[static_cast<size_t>(L - 1)], static_cast<int>(n_),
                                                                 static_cast<int>(m_), nb, 0, o.j);
    after_launch(st);
  }
  if (df.act != kLinear) {  // output-layer curvature, K = m: into slot 0
    dim3 blk(16, 16);
    dim3 grid2(ceil_div(n_, 16), ceil_div(n_, 16), nb);
    prof_begin(st, kTagSmallSyrk, 0, 0);
    dev::small_k_syrk_kernel<<<grid2, blk, 0, st>>>(w.u, dev::kSkMB, n_pad_, w.d[static_cast<size_t>(L - 1)],
                                                    w.ld[static_cast<size_t>(L - 1)], nullptr, 0, static_cast<int>(n_),
                                                    static_cast<int>(m_), nb, P.hslots, n_pad_ * n_pad_, n_pad_);
    after_launch(st);
  }
  const int64_t tot = static_cast<int64_t>(nb) * n_ * n_;
  prof_begin(st, kTagSymmetrize, 0, 0);
  if (o.h_packed)
    dev::pack_lower_kernel<<<dim3(ceil_div(n_, 256), static_cast<unsigned>(n_), nb), 256, 0, st>>>(
        P.hslots, P.slots, P.slot_stride, n_pad_ * n_pad_, n_pad_, static_cast<int>(n_), o.h);
  else
  dev::symmetrize_slots_kernel<<<ceil_div(tot, 256), 256, 0, st>>>(P.hslots, P.slots, P.slot_stride, n_pad_ * n_pad_,
                                                                   n_pad_, static_cast<int>(n_), nb, o.h);
  after_launch(st);
}

// ---------------------------------------------------------------------------
// Net <-> DeviceNet glue.
// ---------------------------------------------------------------------------
Net::~Net() = default;

DeviceNet& Net::device(int ordinal) {
  if (dev_) {
    if (ordinal >= 0 && ordinal != dev_->ordinal())
      throw StructuralError("network is already bound to CUDA device " + std::to_string(dev_->ordinal()));
    return *dev_;
  }
  if (ordinal < 0) {
    int cur = 0;
    if (cudaGetDevice(&cur) != cudaSuccess) {
      cudaGetLastError();
      throw DeviceError("no CUDA device available");
    }
    ordinal = cur;
  }
  dev_ = std::make_unique<DeviceNet>(*this, ordinal);
  return *dev_;
}

int Net::bound_ordinal() const { return dev_ ? dev_->ordinal() : -1; }

MultiPool& Net::multi() {
  if (!multi_) multi_ = std::make_unique<MultiPool>(*this);
  return *multi_;
}

const char* kernel_tag_name(int tag) {
  static const char* names[kTagCount] = {"fwd_rows",     "softmax",       "adj_seed",     "adj_cols",
                                         "adj_reduce",   "nt_mma.gemm",   "nt_mma.syrk",  "syrk_reduce",
                                         "skinny_nt",    "skinny_reduce", "jacobian_out", "small_k_syrk",
                                         "symmetrize",   "nt_mma.fwd",    "nt_mma.adj",   "row_epilogue",
                                         "nt_mma.step",  "dataflow"};
  return (tag >= 0 && tag < kTagCount) ? names[tag] : "unknown";
}

int device_count() {
  int c = 0;
  if (cudaGetDeviceCount(&c) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return c;
}

}  // namespace gbb
