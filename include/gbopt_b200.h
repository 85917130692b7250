/* gbopt_b200 -- B200-native (sm_100a) FP64 gray-box NN oracle, C ABI.
 *
 * Drop-in for the reference's network C interface (reference
 * proj/include/gbopt.h:1-81, proj/src/capi.cpp:31-178) with the same
 * conventions:
 *   - every fallible call returns a gbopt_status (0 = OK);
 *   - on failure the thread-local message from gbopt_last_error() says why;
 *   - out-pointers / out-buffers are written only on GBOPT_OK;
 *   - opaque handles are released by their _free function;
 *   - caller-owned buffers carry explicit lengths; a null pointer or a
 *     length that does not match the network is GBOPT_ERR_ARGUMENT;
 *   - exceptions never cross this boundary;
 *   - a handle is not thread-safe by itself; distinct handles may be used
 *     from distinct threads.
 *
 * Layouts chosen by this ABI (the reference returns Eigen column-major):
 *   J (m x n) is ROW-major: J[i*n + j] = dNN_i/dx_j (the order the
 *   reduced-space callback writes, reference formulations.cpp:320-331);
 *   H (n x n) is the full symmetric matrix, row-major;
 *   weights passed to gbopt_net_from_layers are row-major (GBNN order).
 *
 * Activation codes follow GBNN v1 (reference nn_io.cpp:184, nn.hpp:12-17):
 *   0 linear, 1 tanh, 2 sigmoid, 3 softmax (final layer only),
 *   4 softplus (extension of this build; the reference rejects code 4).
 *
 * Compute entry points (forward ... oracle_batched) run on the GPU the
 * handle is bound to; there is no CPU fallback.  Without a usable CUDA
 * device they return GBOPT_ERR_DEVICE.  Loading, saving, generation and
 * the accessors are host-side and work without a GPU.
 */
#ifndef GBOPT_B200_H
#define GBOPT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Same values as the reference gbopt_status (gbopt.h:19-31) plus
 * GBOPT_ERR_DEVICE for CUDA failures / no device. */
typedef enum gbopt_status {
  GBOPT_OK = 0,
  GBOPT_ERR_STRUCTURAL = 1,
  GBOPT_ERR_NUMERIC = 2,
  GBOPT_ERR_SINGULAR = 3,
  GBOPT_ERR_IO = 4,
  GBOPT_ERR_FORMAT = 5,
  GBOPT_ERR_DIMENSION = 6,
  GBOPT_ERR_TRUNCATED = 7,
  GBOPT_ERR_RANGE = 8,
  GBOPT_ERR_ARGUMENT = 9,
  GBOPT_ERR_INTERNAL = 10,
  GBOPT_ERR_DEVICE = 11
} gbopt_status;

typedef enum gbopt_activation {
  GBOPT_ACT_LINEAR = 0,
  GBOPT_ACT_TANH = 1,
  GBOPT_ACT_SIGMOID = 2,
  GBOPT_ACT_SOFTMAX = 3,
  GBOPT_ACT_SOFTPLUS = 4
} gbopt_activation;

/* Weight initialisers for gbopt_net_random_ex.  UNIFORM_FANIN is the
 * reference random_net (nn.cpp:336-367): W and b ~ U(+-1/sqrt(fan_in)). */
typedef enum gbopt_init {
  GBOPT_INIT_UNIFORM_FANIN = 0,
  GBOPT_INIT_XAVIER_UNIFORM = 1, /* U(+-sqrt(6/(fan_in+fan_out))) */
  GBOPT_INIT_XAVIER_NORMAL = 2,  /* N(0, 2/(fan_in+fan_out)) */
  GBOPT_INIT_NORMAL_FANIN = 3    /* N(0, 1/fan_in) */
} gbopt_init;

typedef struct gbopt_net gbopt_net;
typedef struct gbopt_prng gbopt_prng;

/* Thread-local message of the most recent failed call on this thread; never
 * NULL; empty after a successful call.  (reference gbopt.h:50-53) */
const char* gbopt_last_error(void);

/* Library version string, e.g. "gbopt_b200 1.0 sm_100a". */
const char* gbopt_version(void);

/* ---- devices ------------------------------------------------------------ */

/* Number of CUDA devices visible (0 when none / no driver). */
int gbopt_device_count(void);

/* ---- seeded generation (reference prng.hpp:11-23) ------------------------
 * mt19937_64; uniform01 = (raw >> 11) * 2^-53.  Normals are Box-Muller on
 * two uniforms (u1 mapped to (0,1]), both values of each pair used. */
gbopt_status gbopt_prng_new(uint64_t seed, gbopt_prng** out);
void gbopt_prng_free(gbopt_prng* rng);
gbopt_status gbopt_prng_raw(gbopt_prng* rng, uint64_t* buf, size_t n);
gbopt_status gbopt_prng_uniform(gbopt_prng* rng, double lo, double hi,
                                double* buf, size_t n);
gbopt_status gbopt_prng_normal(gbopt_prng* rng, double mean, double stddev,
                               double* buf, size_t n);

/* ---- networks (reference gbopt.h:59-81) --------------------------------- */

/* GBNN v1 binary, or the JSON mirror when the path ends in ".json"
 * (reference nn_io.cpp:144-247). */
gbopt_status gbopt_net_load(const char* path, gbopt_net** out);
gbopt_status gbopt_net_save(const gbopt_net* net, const char* path);

/* Reference random_net (nn.cpp:336-367); activations by name: linear,
 * tanh, sigmoid, softmax, softplus. */
gbopt_status gbopt_net_random(const int64_t* widths, size_t n_widths,
                              const char* hidden_activation,
                              const char* final_activation, uint64_t seed,
                              gbopt_net** out);

/* Seeded net drawn from an existing generator stream: for each layer in
 * order, W row-major then b (the draw order of nn.cpp:354-362).  Biases
 * are U(bias_lo, bias_hi); bias_lo == bias_hi gives constant biases and
 * draws nothing.  For GBOPT_INIT_UNIFORM_FANIN the biases use the fan-in
 * bound exactly as random_net and bias_lo/hi are ignored. */
gbopt_status gbopt_net_random_ex(gbopt_prng* rng, const int64_t* widths,
                                 size_t n_widths, int hidden_activation,
                                 int final_activation, int init,
                                 double bias_lo, double bias_hi,
                                 gbopt_net** out);

/* "Load MLP weights and activations" from memory: n_layers layers, widths
 * has n_layers+1 entries, weights[l] is row-major widths[l+1] x widths[l],
 * biases[l] has widths[l+1] entries.  Validates like the reference
 * NeuralNet constructor (nn.cpp:74-103). */
gbopt_status gbopt_net_from_layers(size_t n_layers, const int64_t* widths,
                                   const int32_t* activations,
                                   const double* const* weights,
                                   const double* const* biases,
                                   gbopt_net** out);

void gbopt_net_free(gbopt_net* net);

int64_t gbopt_net_input_dim(const gbopt_net* net);
int64_t gbopt_net_output_dim(const gbopt_net* net);
int64_t gbopt_net_param_count(const gbopt_net* net);
int64_t gbopt_net_layer_count(const gbopt_net* net);

/* Shape/activation of layer l and a row-major copy of its parameters
 * (w: rows*cols, b: rows; either may be NULL when not wanted). */
gbopt_status gbopt_net_layer_info(const gbopt_net* net, int64_t l,
                                  int64_t* rows, int64_t* cols,
                                  int32_t* activation);
gbopt_status gbopt_net_layer_copy(const gbopt_net* net, int64_t l, double* w,
                                  size_t w_len, double* b, size_t b_len);

/* Binds the handle to CUDA device `ordinal` and uploads the weights into
 * HBM in kernel layout (idempotent).  Compute calls on an unbound handle
 * bind it to the calling thread's current CUDA device. */
gbopt_status gbopt_net_bind_device(gbopt_net* net, int ordinal);
/* Device the handle is bound to, or -1. */
int gbopt_net_device(const gbopt_net* net);

/* ---- oracle calls (reference nn.hpp:58-74) -------------------------------
 * All synchronous: results are in the caller's host buffers on return. */

/* y = NN(x).  (reference gbopt.h:78-81, nn.cpp:113-125) */
gbopt_status gbopt_net_forward(const gbopt_net* net, const double* x,
                               size_t n, double* y, size_t m);

/* Per-layer values of one forward pass (reference ForwardTrace,
 * nn.hpp:31-36, NeuralNet::forward_trace, nn.cpp:127-146):
 * z_l = W_l y_{l-1} + b_l and y_l = sigma_l(z_l), layers concatenated
 * (z = [z_0 | z_1 | ...], same for y); len == sum of the layers' output
 * widths for both buffers. */
gbopt_status gbopt_net_forward_trace(const gbopt_net* net, const double* x,
                                     size_t n, double* z, double* y,
                                     size_t len);

/* J = dy/dx, m x n row-major, jac_len == m*n.  (nn.cpp:148-170) */
gbopt_status gbopt_net_jacobian(const gbopt_net* net, const double* x,
                                size_t n, double* jac, size_t jac_len);

/* g = grad_x(lambda^T NN(x)), length n.  (nn.cpp:172-196) */
gbopt_status gbopt_net_lagrangian_gradient(const gbopt_net* net,
                                           const double* x, size_t n,
                                           const double* lambda, size_t m,
                                           double* g, size_t g_len);

/* H = sum_i lambda_i Hess NN_i(x), n x n symmetric, hess_len == n*n.
 * (nn.cpp:198-292) */
gbopt_status gbopt_net_lagrangian_hessian(const gbopt_net* net,
                                          const double* x, size_t n,
                                          const double* lambda, size_t m,
                                          double* hess, size_t hess_len);

/* Fused evaluation at one point: y (m), J (m*n), H (n*n) from one forward
 * pass.  Any of y / jac / hess may be NULL when not wanted (its length is
 * then ignored).  lambda may be NULL only when hess is NULL. */
gbopt_status gbopt_net_oracle(const gbopt_net* net, const double* x,
                              size_t n, const double* lambda, size_t m,
                              double* y, double* jac, double* hess);

/* Batched fused evaluation of B independent points with the shared
 * weights: X is B x n, Lambda is B x m (row-major), outputs Y (B x m),
 * J (B x m x n), H (B x n x n).  Output pointers may be NULL. */
gbopt_status gbopt_net_oracle_batched(const gbopt_net* net, size_t batch,
                                      const double* X, size_t n,
                                      const double* Lambda, size_t m,
                                      double* Y, double* J, double* H);

/* As gbopt_net_oracle_batched, but the Hessian comes back as the packed
 * lower triangle, row by row: Hl[b * n (n + 1) / 2 + a (a + 1) / 2 + c] =
 * H_b(a, c) for c <= a -- the value order of the reduced-space Lagrangian-
 * Hessian callback (proj/src/formulations.cpp:298-315, 332-340; for
 * non-ascending host indices the reference flips the (row, col) pattern
 * entries, not the values).  Packed on the device: half the transfer, no
 * host gather.  hl_len = batch * n * (n + 1) / 2; Y and J may be NULL. */
gbopt_status gbopt_net_oracle_lower(const gbopt_net* net, size_t batch,
                                    const double* X, size_t n,
                                    const double* Lambda, size_t m, double* Y,
                                    double* J, double* Hl, size_t hl_len);

/* Same as gbopt_net_oracle_batched on DEVICE pointers of the bound device,
 * enqueued on `stream` (a cudaStream_t, or NULL for the legacy default
 * stream) and NOT synchronised: the caller orders work on `stream`.  This
 * is the entry the multi-GPU driver uses so results can be gathered with
 * NCCL without a host round trip. */
gbopt_status gbopt_net_oracle_batched_device(const gbopt_net* net,
                                             size_t batch, const double* dX,
                                             size_t n, const double* dLambda,
                                             size_t m, double* dY, double* dJ,
                                             double* dH, void* stream);

/* Multi-device evaluation inside one process (new in this build; SURVEY
 * §8e "batched points and contingency copies sharded across the GPUs of one
 * box").  The handle's host weights are replicated to every listed device
 * (uploaded once per device, kept for later calls); `devices[i]` runs slot
 * i, a device may be listed more than once (independent workspaces on one
 * GPU).  The `batch` points are split into contiguous shards, the first
 * batch % n_devices slots taking one extra point, each slot on its own host
 * thread.  No reduction between devices.  Replaces a loop of
 * NeuralNet::lagrangian_hessian calls (reference nn.hpp:58-74) for callers
 * holding one network (formulations.cpp:276).
 *
 * _multi: host buffers as gbopt_net_oracle_batched; every device writes its
 *   rows of Y / J / H straight into the caller's buffers.  Synchronous.
 * _multi_gather: X, Lambda, Y, J, H are device buffers on devices[0]; each
 *   other device pulls its shard of X / Lambda and pushes its rows of the
 *   results back into devices[0]'s buffers with peer copies over NVLink
 *   (the result gather; copy engines, no SM time).  Returns when every
 *   shard has landed (synchronous, no stream argument).
 * The per-shard results are bit-identical to evaluating each shard alone
 * with gbopt_net_oracle_batched on one device. */
gbopt_status gbopt_net_oracle_batched_multi(const gbopt_net* net,
                                            const int* devices,
                                            size_t n_devices, size_t batch,
                                            const double* X, size_t n,
                                            const double* Lambda, size_t m,
                                            double* Y, double* J, double* H);
gbopt_status gbopt_net_oracle_batched_multi_gather(
    const gbopt_net* net, const int* devices, size_t n_devices, size_t batch,
    const double* dX, size_t n, const double* dLambda, size_t m, double* dY,
    double* dJ, double* dH);

/* Oracle schedule of this handle's fused (y, J, H) evaluations:
 *   -1  automatic (default; GBOPT_DATAFLOW=0/1/-2 in the environment at bind
 *       time forces 0/1/-2): a fixed rule on the shape -- the persistent
 *       dataflow launch for chains of >= 8 layers whose tangent GEMM tiles
 *       leave >= 10% of the layer-by-layer waves idle, else layer by layer
 *       -- so every process runs the same kernels for the same call and the
 *       results are reproducible bit for bit;
 *    0  layer-by-layer launches (two streams, CUDA graph);
 *    1  the persistent dataflow launch whenever the shape allows it
 *       (batch <= 112, output width <= 16, no softmax output);
 *   -2  measured: the first call of a shape times both and keeps the faster
 *       (opt-in; two processes may pick differently).
 * Both schedules compute the same quantities (equal to rounding). */
gbopt_status gbopt_net_set_schedule(gbopt_net* net, int schedule);

/* Diagnostics: one eager dataflow evaluation of `batch` points (device
 * pointers) with a per-item trace.  Writes up to `cap` doubles to `out`,
 * 12 per item in claim order: {kind (0 fwd, 1 adj, 2 tangent GEMM, 3 SYRK),
 * job, point, tm, tn, kb0, kb1, SM id, t_claimed, t_ready, t_begin, t_end}
 * (microseconds from the first claim); *n_items = number of items.  `out`
 * may be NULL to query the count.  GBOPT_ERR_STRUCTURE if the dataflow
 * schedule does not apply to this handle and batch. */
gbopt_status gbopt_net_dataflow_trace(const gbopt_net* net, size_t batch,
                                      const double* dX, const double* dLambda,
                                      double* out, size_t cap, size_t* n_items);

/* 1 if the most recent oracle call used the dataflow launch, 0 if it ran
 * layer by layer, -1 if the handle is not bound to a device. */
int gbopt_net_last_schedule(const gbopt_net* net);

/* Number of kernels the most recent oracle call on this handle launched
 * (graph replays count their kernel nodes). */
int64_t gbopt_net_last_launch_count(const gbopt_net* net);

/* Profiling hook used by bench.py's roofline leg: runs one evaluation of
 * `batch` points (device pointers, as gbopt_net_oracle_batched_device)
 * eagerly with CUDA events around every kernel on the launching stream and
 * reports, per launch, its kernel tag, duration (ms), algorithmic FP64
 * flops and algorithmic HBM bytes.  *count receives the number of launches
 * (at most cap are written).  Synchronous. */
gbopt_status gbopt_net_profile(const gbopt_net* net, size_t batch,
                               const double* dX, const double* dLambda,
                               int32_t* tags, float* ms, double* flops,
                               double* bytes, size_t cap, size_t* count);
/* Concurrent-timeline variant of gbopt_net_profile: the launches keep
 * their two streams (0 = critical path, 1 = side stream) and each reports
 * start/end in ms from the start of the evaluation.  Synchronous. */
gbopt_status gbopt_net_profile_timeline(const gbopt_net* net, size_t batch,
                                        const double* dX,
                                        const double* dLambda, int32_t* tags,
                                        int32_t* streams, float* t_start,
                                        float* t_end, size_t cap,
                                        size_t* count);
/* Name of a kernel tag reported by gbopt_net_profile ("nt_mma.gemm", ...). */
const char* gbopt_kernel_tag_name(int tag);

/* White-box access for tests: copies the per-layer vector `name` ("z", "y",
 * "s1", "s2", "ybar", "gz", "d": pre-activation, activation, sigma',
 * sigma'', adjoint dL/dy_l, ybar .* sigma', ybar .* sigma'') of layer
 * `layer` for the first `batch` points of the most recent evaluation into
 * out (batch x rows(layer), row-major; len == batch * rows). */
gbopt_status gbopt_net_debug_intermediate(const gbopt_net* net,
                                          const char* name, int64_t layer,
                                          size_t batch, double* out,
                                          size_t len);

/* Enables/disables CUDA-graph capture of the oracle sequence (default on). */
gbopt_status gbopt_net_set_graphs(gbopt_net* net, int enabled);

/* ---- KKT factorisation --------------------------------
 * Dense symmetric-indefinite LDL^T with the contract of the reference
 * ldlt_factor / LdltFactorization (proj/include/gbopt/linalg.hpp:24-78):
 * finite (NUMERIC) and symmetric to 1e-12*max(1,max|A|) (STRUCTURAL)
 * input, symmetric Ruiz equilibration, Bunch-Kaufman factorisation on the
 * GPU, inertia with zero threshold 1e-11*max|SAS|, solve with iterative
 * refinement when keep_input != 0; solve on a factorisation with zero
 * pivots is GBOPT_ERR_SINGULAR.  A is n x n row-major. */
typedef struct gbopt_ldlt gbopt_ldlt;
gbopt_status gbopt_ldlt_factor(const double* A, size_t n, int keep_input,
                               gbopt_ldlt** out);
gbopt_status gbopt_ldlt_inertia(const gbopt_ldlt* f, int64_t* n_pos,
                                int64_t* n_neg, int64_t* n_zero);
gbopt_status gbopt_ldlt_solve(const gbopt_ldlt* f, const double* b, size_t n,
                              double* x);
void gbopt_ldlt_free(gbopt_ldlt* f);

/* ---- KKT assembly and inertia correction -------------
 * The reference assembles the IPM's dense Newton system in C++ only
 * (assemble_kkt / inertia_correct, proj/include/gbopt/ipm.hpp:80-118,
 * proj/src/ipm.cpp:466-557) -- no C entry exists; these are the C-ABI form,
 * with the system kept on the device between the calls.
 *
 * gbopt_kkt_create analyses one NLP's pattern once: n variables, m
 * constraints, the Lagrangian-Hessian triplets (hess_rows/cols, nnz_h;
 * mirrored, duplicates summed) and the Jacobian triplets (jac_rows/cols,
 * nnz_j).  An index out of range is GBOPT_ERR_STRUCTURAL.
 *
 * gbopt_kkt_assemble (assemble_kkt, ipm.cpp:466-518) scatters one
 * iteration's values: x, lower (-inf = unbounded), z, grad_f: n entries;
 * lambda, g: m; hess_values: nnz_h; jac_values: nnz_j.  The matrix
 * [[H + Sigma + delta_w I, J^T], [J, -delta_c I]] (Sigma_ii = z_i / (x_i -
 * lower_i) on bounded rows) and rhs [-grad_f - J^T lambda + mu / (x -
 * lower); -g] equal the reference's bit for bit (same additions in the same
 * order; products rounded separately).
 *
 * gbopt_kkt_matrix / gbopt_kkt_rhs copy them out ((n+m)^2 row-major / n+m).
 *
 * gbopt_kkt_inertia_correct (inertia_correct, ipm.cpp:520-557) factors
 * the device-resident matrix with delta_w = delta_w_start, then delta0, then
 * *= delta_growth (and delta_c = 1e-8 .. 1e-2 while zero pivots persist with
 * m > 0) until the inertia is (n, m, 0); the factorisation (keep_input on)
 * goes to *fact (free with gbopt_ldlt_free), the shifts to *delta_w and
 * *delta_c.  GBOPT_ERR_SINGULAR once delta_w exceeds delta_max.
 *
 * gbopt_kkt_solve: fact.solve(rhs) with the assembled right-hand side
 * (sol: n + m entries). */
typedef struct gbopt_kkt gbopt_kkt;
gbopt_status gbopt_kkt_create(size_t n, size_t m, const int64_t* hess_rows,
                              const int64_t* hess_cols, size_t nnz_h,
                              const int64_t* jac_rows, const int64_t* jac_cols,
                              size_t nnz_j, gbopt_kkt** out);
gbopt_status gbopt_kkt_assemble(gbopt_kkt* kkt, const double* x,
                                const double* lower, const double* z,
                                const double* lambda, const double* grad_f,
                                const double* g, const double* jac_values,
                                const double* hess_values, double mu,
                                double delta_w, double delta_c);
gbopt_status gbopt_kkt_matrix(const gbopt_kkt* kkt, double* out, size_t len);
gbopt_status gbopt_kkt_rhs(const gbopt_kkt* kkt, double* out, size_t len);
gbopt_status gbopt_kkt_inertia_correct(const gbopt_kkt* kkt, double delta0,
                                       double delta_growth, double delta_max,
                                       double delta_w_start, gbopt_ldlt** fact,
                                       double* delta_w, double* delta_c);
gbopt_status gbopt_kkt_solve(const gbopt_kkt* kkt, const gbopt_ldlt* fact,
                             double* sol, size_t len);
void gbopt_kkt_free(gbopt_kkt* kkt);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* GBOPT_B200_H */
