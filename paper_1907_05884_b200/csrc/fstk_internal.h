// Internal (non-ABI) declarations shared by the fstk B200 library sources.
#pragma once

#include <cublas_v2.h>
#include <cusolverDn.h>
#include <cuda_runtime.h>

#include <functional>
#include <future>
#include <memory>
#include <mutex>
#include <vector>

#include "fstk_common.cuh"

namespace fstk_gpu {

constexpr int kMaxOrder = 8;
constexpr int kMaxShards = 32;  // ranks of a column-sharded refit (fstk_gpu_refit_begin_columns)   // proj/include/fstk/tensor.hpp:16
struct Int64x8 {
  int64_t v[8];
};
constexpr int kMaxDegree = 64; // proj/src/basis.cpp:31

// Per-mode device parameters for the mode-value kernel.
struct ModeDev {
  double lo, hi, span, slack;  // basis.cpp:215-222 (slack = 1e-12 * span)
  int r;                       // rank r_k
  int pmax;                    // max Legendre degree over the mode's functions
  const int* rowptr;           // r+1 CSR offsets into idx/coef
  const uint32_t* idx;         // ascending basis indices per function
  const double* coef;
  const double* dense;         // (pmax+1) x ldc dense coefficients (0 where absent)
  int ldc;                     // nchunk * jc
  int jc;                      // functions per dense-kernel thread (multiple of 8, <= 64)
  int nchunk;
  const double* h_dense;       // host copy of `dense` (builds the kernel-parameter blocks)
};
struct ModesDev {
  int d;
  ModeDev m[kMaxOrder];
};

// Modes with wavelet bases (or several distinct bases): per-thread scratch
// layout of each distinct basis and the function -> basis map.
constexpr int kMaxSpec = 8;
struct SpecDev {
  int family;              // 0 Legendre, 1 wavelet
  int p, s;                // degree, resolution
  int voff;                // offset (doubles) in the per-thread scratch
  const double* coords;    // wavelet: 2(p+1) x (p+1) mother coords * sqrt(2)
};
struct GenModeDev {
  ModeDev md;
  int nspec;               // 0 => the mode uses the Legendre fast paths
  int vtot;                // per-thread scratch doubles
  SpecDev sp[kMaxSpec];
  const int* fn_spec;      // r entries
};

// Host copy of one mode.
struct ModeHost {
  int r = 0, pmax = 0;
  bool sorted = true;  // every function's indices strictly increasing (format.md:67)
  std::vector<int> spec_family, spec_p, spec_s;  // distinct bases, first-seen order
  std::vector<int> fn_spec;                      // function -> distinct basis
  bool general = false;                          // any wavelet basis in the mode
  double lo = 0, hi = 0;
  std::vector<int> rowptr;
  std::vector<uint32_t> idx;
  std::vector<double> coef;
};

// Layout of the DMMA contraction: K = mode 0 padded to a
// multiple of 4, N = (j1 chunk) x (outer modes m = j2 + r2 (j3 + ...)).
struct ContractLayout {
  bool fast = false;   // DMMA tile path usable for this shape
  int Kp = 0;          // r0 padded to 4
  int N1p = 0;         // j1 columns per B tile (multiple of 16, <= 64)
  int NC = 0;          // j1 chunks
  int Mout = 0;        // prod_{k>=2} r_k
  int nsw = 0;         // 8-column subtiles per warp = N1p / (8 nh)
  int nh = 2;          // column groups per 32-point group
  bool kr = false;     // Khatri-Rao form (K = r0 r1, one epilogue per tile)
  int kr_np = 0;       // padded N = prod_{k>=2} r_k of the KR form
  int nstage = 0;      // B pipeline depth
  int tp = 128;        // points per CTA tile (64 or 128)
  int ctas_per_sm = 1; // resident CTAs per SM at this shared-memory footprint
  size_t smem = 0;     // dynamic shared memory bytes
  int64_t btile_elems = 0;  // Kp * N1p
};

// Workspace for one in-flight chunk.
struct Chunk {
  DevBuf<double> points;   // d x CH (column-major, ld = CH)
  DevBuf<double> tables;   // sum_k rp_k x CHp
  DevBuf<double> out;      // CH
  DevBuf<unsigned long long> err;  // lowest failing row (ULLONG_MAX = none)
  std::vector<unsigned long long> err_host;
  cudaStream_t stream = nullptr;
  cudaEvent_t done = nullptr;
  cudaEvent_t host_done = nullptr;  // pageable staging: this slot's D2H landed
  double* h_stage = nullptr;        // pageable staging: pinned d x CH points + CH outputs
};

}  // namespace fstk_gpu

struct fstk_gpu_model {
  int device = 0;
  // fstk_gpu_set_devices: replicas on the other listed devices; a host
  // evaluate_batch splits its points across this model and the replicas.
  std::vector<fstk_gpu_model*> replicas;
  int d = 0;
  std::vector<int64_t> ranks;
  int64_t R = 0;
  int num_sms = 148;
  std::vector<fstk_gpu::ModeHost> modes;
  std::vector<double> core;  // host copy, mode-0 fastest

  fstk_gpu::DevBuf<double> d_core;
  fstk_gpu::DevBuf<int> d_rowptr;
  fstk_gpu::DevBuf<uint32_t> d_idx;
  fstk_gpu::DevBuf<double> d_coef;
  fstk_gpu::DevBuf<double> d_dense;  // all modes' dense coefficient blocks
  std::vector<double> h_dense;       // host copy (kernel-parameter coefficient blocks)
  fstk_gpu::GenModeDev gen[fstk_gpu::kMaxOrder] = {};  // wavelet-capable per-mode params
  fstk_gpu::DevBuf<int> d_fn_spec;
  std::vector<std::shared_ptr<fstk_gpu::DevBuf<double>>> mother_refs;
  bool dense_ok = true;              // dense kernel is bit-equivalent (sorted indices)
  fstk_gpu::ModesDev modes_dev{};

  fstk_gpu::ContractLayout lay;
  fstk_gpu::DevBuf<double> d_bpack;  // DMMA fragment-ordered core

  // Per-mode padded table heights: rp[k] = rows of table k stored.
  int rp[fstk_gpu::kMaxOrder] = {0};

  // Evaluation workspace (guarded by mu).
  mutable std::mutex mu;
  mutable fstk_gpu::Chunk chunk[2];
  mutable fstk_gpu::DevBuf<unsigned long long> chunk_err;  // one slot per chunk
  cudaEvent_t fork_ev = nullptr;
  int64_t chunk_points = 0;

  ~fstk_gpu_model();
};

namespace fstk_gpu {

// Mode-value tables for n points.  points: column k at pts + k*ldp.  Output
// table k, function j, row i at tables + toff[k] + j*ldt + i; rows in
// [n, n_out) are zero-filled.  row_src (optional): output row i takes input
// point row_src[i] (negative => zero row).  exact=true reproduces the
// reference sparse dot bit for bit (separate multiply and add).
void launch_mode_tables(const fstk_gpu_model* m, const double* pts, int64_t ldp, int64_t n,
                        int64_t n_out, const int64_t* row_src, double* tables,
                        const int64_t* toff, int64_t ldt, bool exact,
                        unsigned long long* err_row, cudaStream_t s);
// Only mode `mode` (table at `out`, ld = ldt).
void launch_mode_table_one(const fstk_gpu_model* m, int mode, const double* x, int64_t n,
                           double* out, int64_t ldt, bool exact, unsigned long long* err_row,
                           cudaStream_t s);

// Contraction of precomputed tables with the core: out[i] for i < n.
void launch_contract(const fstk_gpu_model* m, const double* tables, const int64_t* toff,
                     int64_t ldt, int64_t n, double* out, cudaStream_t s,
                     const double* bpack_override = nullptr, const double* core_override = nullptr);

// Table offsets/heights used by evaluation for a chunk with ldt rows.
void eval_table_offsets(const fstk_gpu_model* m, int64_t ldt, int64_t* toff, int64_t* total);

// Full device evaluation of n points (points column-major, ld = ldp) into
// out, using the model's chunk workspace; err_row receives the lowest failing
// row index.  Caller holds m->mu.
void evaluate_device(const fstk_gpu_model* m, const double* pts, int64_t ldp, int64_t n,
                     double* out, cudaStream_t s);
void evaluate_device_core(const fstk_gpu_model* m, const double* core_host, const double* pts,
                          int64_t ldp, int64_t n, double* out, cudaStream_t s);
int64_t evaluate_device_error(const fstk_gpu_model* m, int64_t n, cudaStream_t s);

// Throws the reference's Domain error for point `row` (coordinates given on
// the host), mirroring basis.cpp:218-219.
[[noreturn]] void throw_domain(const fstk_gpu_model* m, int64_t row, const double* y);

int device_sm_count(int device);
cublasHandle_t blas_handle(int device);
cublasHandle_t blas_side_handle(int device);
cusolverDnHandle_t solver_handle(int device);

// Wavelet support (fstk_wavelet.cu).
std::shared_ptr<DevBuf<double>> mother_coords_device(int device, int p);
void upload_wavelet_constants(int device);
void launch_mode_general(const GenModeDev& G, const double* xs, int64_t n, int64_t n_out,
                         const int64_t* row_src, double* tk, int64_t ldt, bool exact,
                         unsigned long long* err_row, cudaStream_t s, int device);

// Sliced int8 tensor-core Gram (fstk_gram.cu).  Scratch is per refit so
// concurrent refits on one device never share buffers.
struct GramScratch {
  DevBuf<int8_t> X, Y;     // digit planes, column a at a * ns * kp
  DevBuf<int32_t> C;       // ns planes of one column block (digit scheme / cuBLASLt engine)
  DevBuf<uint8_t> C8;      // per-CTA residue scratch of the tcgen05 SYRK engine
  DevBuf<int> ex;          // per-column exponents of the current segment
  DevBuf<uint8_t> ws;      // cuBLASLt workspace
  int64_t kp = 0;          // segment rows, fixed by the first call
  int64_t last_block_w = 0;  // column-block width of the latest CRT call (0: no block order)
};
int gram_slices();                      // 0 = native fp64 DSYRK/DGEMM Gram
int crt_level_bits(int level);          // bits per entry of CRT level 2..7 (at 32,768-row segments)
// Int8 GEMM engine of the CRT Gram: 1 = the hand-written tcgen05 SYRK
// (fstk_syrk.cu, default), 2 = cuBLASLt IMMA GEMMs (comparison).
int gram_engine();
int set_gram_engine(int engine);        // returns the previous setting; 0 = query
// fstk_syrk.cu: G (lower triangle, n x n, ldg) = [G +] (-1)^negate sum over
// the rows of one segment of the exact CRT Gram: the int8 planes R_t (kp x np,
// column-major, plane t at planes + t kp np) give C_t = R_t^T R_t on the
// tcgen05 tensor cores; Garner folds the nm residues of every entry and scales
// by 2^(ex_a + ex_b - 2k).  scratch: syrk_crt_scratch_bytes(nm) bytes.
// Returns the int8 ops issued.
constexpr int kSyrkMaxModuli = 20;
size_t syrk_crt_scratch_bytes(int nm, int device);
// Unfused variants (default "permod"): residues of the column block
// [c0, c0 + wn) x [c0, np) for every modulus into C (ld m, plane stride
// cstride), folded afterwards by crt_fold_kernel.
bool syrk_fused();
int syrk_mode();
double syrk_i8_residues_one(const int8_t* planes, int nm, int t, int64_t kp, int64_t np, int64_t c0, int64_t wn,
                            int64_t m, int8_t* C, int* counter, int device, cudaStream_t s);
double syrk_i8_residues(const int8_t* planes, int nm, int64_t kp, int64_t np, int64_t c0, int64_t wn,
                        int64_t m, int8_t* C, int64_t cstride, int* counter, int device, cudaStream_t s);
double syrk_crt_fold(const int8_t* planes, int nm, int64_t kp, int64_t np, int n, int k, const int* ex,
                     double* G, int64_t ldg, bool accumulate, bool negate, uint8_t* scratch, int device,
                     cudaStream_t s);
int set_gram_slices(int slices);        // returns the previous setting
bool gram_sliced_applies(int64_t rows, int n);
// gram = beta * gram + the plane sums t_lo..slices+1 of A^T A (t_lo = 2:
// the whole sliced Gram; t_lo = s0 + 2 upgrades an s0-plane Gram to
// `slices` planes exactly).  Returns the int8 tensor-core ops issued.
double gram_accumulate_sliced(const double* A, int64_t lda, int64_t rows, int n, double* gram,
                              double beta, int slices, int t_lo, cudaStream_t s, int device,
                              GramScratch& sc);
constexpr int kGramUpgradeSlices = 7;   // escalation target before the native Gram
constexpr double kDoneFloor = 1e-14;    // refinement: extrapolated remaining ||dx||/||x|| that ends it
// transform = "none" design rows A[r][ell] = scale ((u0 u1) u2 ...)(row0 + r)
// generated from mode tables (column j_k of mode k at toff[k] + j_k ldt).
struct DesignSpec {
  const double* tables;
  Int64x8 toff;
  int64_t ldt;
  int d;
  Int64x8 ranks;
  int64_t row0;
  double scale;
};
// G (lower triangle, n x n inside a matrix of leading dimension ldg) -= T^T T
// for T = rows x n (column-major, ldt), through the CRT int8 Gram at `slices`
// plane-accuracy: the trailing update of the blocked Cholesky (chol_crt).
// first_block_done (optional) is recorded on s once the update's first column
// block (*first_block_cols columns wide, 0 when the engine has no block order)
// has been folded into G: the blocked Cholesky's lookahead starts the next
// panel there.  after_first_block (optional) is called right after that record
// when the block is at least need_cols wide (else *first_block_cols = 0).
double gram_update_crt(const double* T, int64_t ldt, int64_t rows, int n, double* G, int64_t ldg,
                       int slices, cudaStream_t s, int device, GramScratch& sc,
                       cudaEvent_t first_block_done = nullptr, int64_t* first_block_cols = nullptr,
                       const std::function<void()>* after_first_block = nullptr, int64_t need_cols = 0);
// The sliced (CRT) Gram of those rows without materialising them.
bool gram_scheme_crt();
double gram_accumulate_sliced_design(const DesignSpec& spec, int64_t rows, int n, double* gram,
                                     double beta, int slices, cudaStream_t s, int device,
                                     GramScratch& sc);


// ---- multi-device refit (fstk_multi.cu) ----
int refit_device(const fstk_gpu_refit* rf);
int64_t refit_order(const fstk_gpu_refit* rf);
bool refit_awaits_exchange(const fstk_gpu_refit* rf);
int refit_gram_used(const fstk_gpu_refit* rf);
bool refit_is_factored(const fstk_gpu_refit* rf);
int32_t reestimate_core_multi(const fstk_gpu_model* m, const double* points, const double* values,
                              int64_t q, int32_t d, const fstk_sketch_cfg* cfg, double* core_out,
                              fstk_reestimate_info* info, fstk_gpu_error* err);

// ---- rank decision (fstk_rank.cu; randls.cpp:112-123) ----
// Streaming TSQR of a tall matrix with n1 columns, fed in row blocks of at
// most bmax rows: after fold(), the leading n1 x n1 block of W (ld ldw) is
// the upper-triangular R of everything folded so far (zeros below).
struct QrStream {
  int n1 = 0;
  int64_t bmax = 0, ldw = 0;
  DevBuf<double> W, tau;
  DevBuf<uint8_t> work;
  size_t work_bytes = 0;
  std::vector<uint8_t> host_work;
  DevBuf<int> info;
  cusolverDnParams_t params = nullptr;
  bool has_r = false;
  cudaStream_t s = nullptr;
  int device = 0;
  QrStream() = default;
  QrStream(const QrStream&) = delete;
  QrStream& operator=(const QrStream&) = delete;
  ~QrStream();
  void init(int n1, int64_t bmax, cudaStream_t s, int device);
  double* block() { return W.p + n1; }  // rows [n1, n1 + rows) of W, ld = ldw
  void fold(int64_t rows);              // R := R of [R; block rows]
  void fold_upper(const double* R2, int64_t ld2);  // R := R of [R; R2] (n1 x n1)
  void get_r(double* dst, int64_t ld) const;
};
// Pivoted QR of the (n+1) x (n+1) upper R of [A b] (ld ldr), Eigen's rank
// rule with diag_size = min(rows of A, n), then the QR solution (full rank)
// or the COD minimum-norm solution.  Returns the rank; x is device memory.
int cpqr_solve(const double* Raug, int64_t ldr, int n, int64_t diag_size, double* x,
               bool* deficient, cudaStream_t s, int device);
// X := (L L^T)^{-1} X (nrhs columns, ld ldx) for a lower factor L (ld n).
void chol_solve_blocked_multi(cublasHandle_t h, const double* L, int n, double* X, int64_t ldx,
                              int nrhs);
// Upper estimate of lambda_min(L L^T) (block power iteration on the inverse),
// enqueued without host synchronisation (start) and read back (result), so
// it can overlap other work on another stream.
struct LambdaMinEstimate {
  static constexpr int kVectors = 4;
  DevBuf<double> X, norms;
  int n = 0, device = 0;
  cudaStream_t s = nullptr;
  bool started = false;
  // The enqueue job of start_async on the library's side worker thread.
  std::shared_future<void> enqueued;
  void start(const double* L, int n, int iters, cudaStream_t s, int device);
  // start() on the side worker: the chain is ~400 cuBLAS calls and more
  // kernels than the driver queues at once, so enqueueing it blocks the
  // calling thread for about as long as the chain runs (80 ms at C2).
  void start_async(const double* L, int n, int iters, cudaStream_t s, int device);
  // Blocks until the chain is enqueued (rethrows what the job threw).
  void wait_enqueued();
  double result();
  LambdaMinEstimate() = default;
  LambdaMinEstimate(const LambdaMinEstimate&) = delete;
  LambdaMinEstimate& operator=(const LambdaMinEstimate&) = delete;
  ~LambdaMinEstimate();
};
// Runs jobs in submission order on one long-lived host thread (its own
// thread-local cuBLAS handles are created once).
std::shared_future<void> side_worker_submit(std::function<void()> job);
double chol_lambda_min_estimate(const double* L, int n, int iters, cudaStream_t s, int device);
}  // namespace fstk_gpu
