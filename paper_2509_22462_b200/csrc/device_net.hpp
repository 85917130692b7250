// Device-resident network (weights in HBM in kernel layout), its workspace
// and the oracle launch sequence.  See oracle.cu and DESIGN.md.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <tuple>
#include <vector>

#include "net.hpp"

namespace gbb {
namespace dev {
struct NtParams;
struct DfItem;
struct DfJob;
}

void cuda_check(cudaError_t e, const char* what);
int device_count();

// Restores the caller's current device on scope exit.
class DeviceGuard {
 public:
  explicit DeviceGuard(int ordinal) {
    if (cudaGetDevice(&prev_) != cudaSuccess) prev_ = -1;
    cuda_check(cudaSetDevice(ordinal), "cudaSetDevice");
  }
  ~DeviceGuard() {
    if (prev_ >= 0) cudaSetDevice(prev_);
  }

 private:
  int prev_ = -1;
};

struct DevLayer {
  int64_t rows = 0, cols = 0, ldw = 0;
  int act = 0;
  double* w = nullptr;  // [rows][ldw]
  double* b = nullptr;  // [rows]
  CUtensorMap tm_w;     // TMA view of w, box 16 x kBN (B operand)
  CUtensorMap tm_wadj;  // TMA view of w, 16 x 16 boxes (multi-vector adjoint, adj_mma_kernel)
  double* wt = nullptr;  // W^T [cols][ldwt] (created for batched adjoints)
  int64_t ldwt = 0;
  CUtensorMap tm_wt;
};

struct Workspace {
  std::vector<double*> z, y, s1, s2, ybar, gz, d;  // per layer [cap][ld[l]]
  std::vector<int64_t> ld;
  int64_t ld_in = 0, ld_lam = 0;
  double *x = nullptr, *lam = nullptr, *grad = nullptr, *mid = nullptr;
  int adj_chunks_max = 0;
  int64_t ld_part = 0;
  double* adj_part = nullptr;
  unsigned* adj_cnt = nullptr;  // arrival counters of the fused adjoint chunk reduction
  std::vector<double*> t;                   // ring of tangent buffers
  std::vector<double*> s;                   // ring of pre-scaled tangents S_l = T_l diag(sigma'_l)
  double* s0 = nullptr;                     // S_0 = W_0^T diag(sigma'_0) per point [cap][n_pad][ldt0]
  CUtensorMap tm_s0;
  std::vector<CUtensorMap> tm_s_a;          // S_l as the A operand (l >= 1)
  std::vector<CUtensorMap> tm_t_a, tm_t_b;  // per layer l >= 1 (buffer (l-1) % ring)
  int64_t ldh = 0;
  double* h = nullptr;             // H accumulator [cap][n_pad][n_pad], lower triangle
  double* syrk_part = nullptr;  // split-K partials (SYRK and batched GEMMs; side stream)
  double* gemm_part = nullptr;
  std::vector<double*> syrk_gather;  // per-layer SYRK partials of the gather path  // split-K partials of single-point tangent GEMMs (main stream)
  CUtensorMap tm_x;                   // x as an A operand [cap][n]
  std::vector<CUtensorMap> tm_y, tm_gz;  // y_l / gz_l as A operands [cap][n_l]
  int sk_chunks = 0;
  double *u = nullptr, *sk_part = nullptr;
  double *y_out = nullptr, *j_out = nullptr, *h_out = nullptr, *g_out = nullptr;
};

enum KernelTag : int {
  kTagFwd = 0, kTagSoftmax, kTagAdjSeed, kTagAdjCols, kTagAdjReduce, kTagGemm, kTagSyrk, kTagSyrkReduce,
  kTagSkinny, kTagSkinnyReduce, kTagJacOut, kTagSmallSyrk, kTagSymmetrize, kTagFwdGemm, kTagAdjGemm, kTagRowEpi,
  kTagStep, kTagDataflow,
  kTagCount
};
const char* kernel_tag_name(int tag);

struct ProfResult {
  int tag;
  float ms;
  double flops;  // algorithmic FP64 flops of this launch
  double bytes;  // algorithmic HBM bytes (weight streams) of this launch
  float t0, t1;  // start / end relative to the evaluation start (ms)
  int stream;    // 0 critical-path stream, 1 side stream
};

struct Outputs {
  double* y = nullptr;  // [nb][m]
  double* j = nullptr;  // [nb][m][n]
  double* h = nullptr;  // [nb][n][n], or [nb][n (n + 1) / 2] packed lower rows when h_packed
  double* g = nullptr;  // [nb][n]
  bool h_packed = false;
};

// One persistent dataflow launch (dataflow.cuh) for a batch size: the
// ordered item list, the jobs, their TMA descriptors and the counters, all
// in device memory.  Built on first use, dropped with the workspace.
struct DfPlan {
  int nb = 0;
  int n_items = 0, n_counters = 0, slots = 0;
  int64_t slot_stride = 0;  // doubles between H slots
  dev::DfItem* items = nullptr;
  dev::DfJob* jobs = nullptr;
  std::vector<CUtensorMap> maps;  // TMA descriptors (kernel parameters)
  int* counters = nullptr;
  double* hslots = nullptr;  // [slots][nb][n_pad][n_pad]
  double flops = 0, bytes = 0;  // algorithmic work of the launch
  double sim_ms = 0;            // list-scheduling estimate of the launch
};

class DeviceNet {
 public:
  DeviceNet(const Net& net, int ordinal);
  ~DeviceNet();
  DeviceNet(const DeviceNet&) = delete;
  DeviceNet& operator=(const DeviceNet&) = delete;

  int ordinal() const { return ordinal_; }
  int64_t last_launches() const { return last_launches_; }
  bool last_dataflow() const { return last_dataflow_; }

  // Host buffers in/out (synchronous).  Any output may be null.
  void evaluate_host(int nb, const double* x, const double* lam, double* y, double* jac, double* hess, double* grad,
                     bool hess_packed = false);
  // Copies an intermediate per-layer vector of the most recent evaluation
  // ("z", "y", "s1", "s2", "ybar", "gz", "d") for `nb` points into out
  // (nb x rows(l), row-major).  Synchronous; for white-box tests.
  void copy_intermediate(const char* name, int layer, int nb, double* out);
  struct AdjLayout {
    int kw = 2, gx = 1, crows = 128, chunks = 1;
  };
  AdjLayout adj_layout(const DevLayer& d, bool multi) const;
  // Eager run with CUDA events around every launch (on the launching stream).
  void profile(int nb, const double* dx, const double* dlam, std::vector<ProfResult>* out, bool timeline = false);
  // Device buffers, ordered on `user` stream, asynchronous.
  void evaluate_device(int nb, const double* dx, const double* dlam, double* dy, double* dj, double* dh,
                       cudaStream_t user);
  // Batches above kMaxChunk points run as consecutive sub-batches (grid
  // dimensions y / z of the per-point launches stay <= 65535).
  static constexpr int kMaxChunk = 32768;

 private:
  void evaluate_host_chunk(int nb, const double* x, const double* lam, double* y, double* jac, double* hess,
                           double* grad, bool hess_packed);
  void evaluate_device_chunk(int nb, const double* dx, const double* dlam, double* dy, double* dj, double* dh,
                             cudaStream_t user);
  using GraphKey = std::tuple<int, double*, double*, double*, double*, bool, bool>;
  struct GraphEntry {
    cudaGraphExec_t exec = nullptr;
    int64_t launches = 0;
  };

  void ensure_workspace(int batch);
  void free_workspace();
  void drop_graphs();
  double* ws_alloc(size_t n_doubles);
  int syrk_split(int points, int k_blocks) const;
  void ensure_transposed();
  void prepare(int nb, const Outputs& o);
  void launch_skinny(cudaStream_t st, int nb, const double* t, int64_t ldt, int64_t t_point_rows, int l,
                     double* jac = nullptr);
  void batch_gemm(cudaStream_t st, int nb, const CUtensorMap& ta, const DevLayer& d, bool transposed,
                  const void* epi, double* store);
  void launch_nt(cudaStream_t st, const CUtensorMap& ta, const CUtensorMap& tb, const dev::NtParams& p, int grid);
  void enqueue(cudaStream_t st, int nb, const Outputs& o);
  // Persistent dataflow path (y, J, H at small batch): oracle.cu.
  bool dataflow_ok(int nb, const Outputs& o) const;
  bool dataflow_possible(int nb, const Outputs& o) const;
  using ChoiceKey = std::tuple<int, bool, bool, bool>;
  static ChoiceKey choice_key(int nb, const Outputs& o) { return ChoiceKey{nb, o.y != nullptr, o.j != nullptr, o.h != nullptr}; }
  std::map<ChoiceKey, bool> df_choice_;                     // auto schedule: dataflow measured faster
  std::map<ChoiceKey, std::pair<float, float>> df_tuned_ms_;  // (layered, dataflow) ms of the autotune
  int df_force_ = -1;  // autotune override of the schedule mode
  void autotune(cudaStream_t st, int nb, const Outputs& o);
  bool dataflow_rule(int nb) const;
  void dispatch(cudaStream_t st, int nb, const Outputs& o);
  DfPlan& dataflow_plan(int nb);
  void enqueue_dataflow(cudaStream_t st, int nb, const Outputs& o);
  void free_plans();
  unsigned long long* df_trace_ = nullptr;
  int* df_trace_sm_ = nullptr;

 public:
  std::vector<double> dataflow_trace(int nb, const double* dx, const double* dlam);

 private:
  int dataflow_mode_ = -1;  // GBOPT_DATAFLOW: -1 auto, 0 off, 1 whenever the shape allows
  std::map<int, DfPlan> df_plans_;
  bool df_square_ = true;  // square 112 x 112 SYRK tiles in the dataflow launch (GBOPT_DF_SQ)
  int df_group_ = 4;  // row blocks per raster group of the tangent GEMM items (GBOPT_DF_GROUP)
  void prof_begin(cudaStream_t st, int tag, double flops, double bytes);
  void after_launch(cudaStream_t st);
  struct ProfRec {
    int tag;
    double flops, bytes;
    cudaEvent_t e0, e1;
    int stream;
  };
  bool profiling_ = false, prof_timeline_ = false;
  std::vector<ProfRec> prof_;
  void run(cudaStream_t st, int nb, const Outputs& o);

  const Net& net_;
  int ordinal_ = 0;
  int sm_count_ = 148;
  cudaStream_t stream_ = nullptr;   // high priority: critical path
  cudaStream_t stream2_ = nullptr;  // low priority: adjoint + SYRKs
  bool concurrent_ = true;
  std::vector<cudaEvent_t> evpool_;
  cudaEvent_t ev_in_ = nullptr, ev_out_ = nullptr;
  cudaStream_t copy_stream_ = nullptr;  // host-buffer calls: D2H of finished chunks
  std::vector<cudaEvent_t> chunk_ev_;
  int64_t n_ = 0, m_ = 0, L_ = 0, n_pad_ = 0;
  std::vector<DevLayer> layers_;
  double* t0_ = nullptr;  // W_0^T [n_pad][ldt0_]
  int64_t ldt0_ = 0, ldt_ = 0;
  CUtensorMap tm_t0_a_, tm_t0_b_;
  int2* syrk_tiles_ = nullptr;
  int n_syrk_tiles_ = 0;
  int2* sq_tiles_ = nullptr;  // square 112 x 112 lower tiles (layer-by-layer SYRKs)
  int n_sq_tiles_ = 0;
  bool square_syrk_ = true;   // GBOPT_SQ=0: 112 x 128 SYRK tiles
  Workspace ws_;
  int ws_cap_ = 0;
  bool transposed_ = false;
  std::vector<void*> ws_allocs_;
  std::map<GraphKey, GraphEntry> graphs_;
  int64_t launches_ = 0, last_launches_ = 0;
  double* stage_ = nullptr;  // pinned staging for results bound for pageable host buffers
  size_t stage_cap_ = 0;
  bool last_dataflow_ = false;
  // persistent single-point forward (fwd_stream.cuh)
  bool fwd_stream_ok() const;
  size_t fwd_stream_smem() const;
  void launch_fwd_stream(cudaStream_t st);
  unsigned* fs_arrive_ = nullptr;
  unsigned fs_gen_ = 0;
  bool fs_attr_set_ = false;
  // GBOPT_FWD_STREAM=1 opts in; off by default: measured slower than the
  // per-layer GEMV graph (c2 165 vs 155 us device time, c5 130 vs 80 us;
  // profiles/r02_fwd_stream.md)
  int fwd_stream_mode_ = 0;
  bool adj_mma_ = true;  // multi-vector adjoints on DMMA (GBOPT_ADJ_MMA=0: CUDA-core sweeps)
  bool adj_fuse_ = true;  // chunk reduction in the adjoint sweep's last CTA (GBOPT_ADJ_FUSE=0: separate launch)
  bool syrk_fuse_ = true;
  int s0_mode_ = -1;  // S_0 = T_0 diag(sigma'_0) materialised: -1 by the rule, 0 / 1 forced (GBOPT_S0_PASS)
  bool syrk_gather_ = true;  // small batches: per-layer SYRK partials, one gather (GBOPT_SYRK_GATHER=0: per-layer reduce)  // one-tile points: all layers' curvature in one launch (GBOPT_SYRK_FUSE=0: per layer)
};

}  // namespace gbb
