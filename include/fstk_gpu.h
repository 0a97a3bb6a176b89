/*
 * fstk_gpu.h — C-ABI of the B200-native functional-sparse-Tucker hot path.
 *
 * Drop-in boundary for the reference library `fstk` (arXiv 1907.05884
 * reference, /root/reference/proj).  Each entry point replaces one reference
 * C++ call on the hot path; the reference signature it replaces is cited next
 * to it.  Conventions:
 *   - plain pointers and sizes only; no C++ or torch types cross the ABI;
 *   - every function returns 0 on success or (fstk ErrorKind + 1) on failure
 *     (proj/include/fstk/error.hpp:11-19) and never throws; the optional
 *     fstk_gpu_error* receives the kind, a message and, for Domain errors,
 *     the first offending point/mode/coordinate;
 *   - the caller owns host buffers (pinned or pageable); the library owns
 *     device memory and streams; a model handle may be shared by threads.
 *   - matrices are column-major ("Eigen default", proj/include/fstk/tensor.hpp:12)
 *     and tensors are mode-0 fastest (tensor.hpp:18-22).
 */
#ifndef FSTK_GPU_H_
#define FSTK_GPU_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FSTK_GPU_ABI_VERSION 3

/* Status codes = fstk::ErrorKind + 1 (error.hpp:11-19). */
enum {
  FSTK_OK = 0,
  FSTK_E_PARAMETER = 1,
  FSTK_E_SHAPE = 2,
  FSTK_E_DOMAIN = 3,
  FSTK_E_DATA = 4,
  FSTK_E_IO = 5,
  FSTK_E_DECODE = 6,
  FSTK_E_COMPUTE = 7
};

/* Mixing transforms, fstk::MixingTransform (randls.hpp:13), plus NONE: the
 * north_star's literal estimator (extension, not in the reference): S of the
 * Q_w working rows sampled uniformly without replacement from the sketch RNG
 * stream, scaled by sqrt(Q_w/S), no mixing; A^T A is accumulated from design
 * rows generated block by block so A is never materialised.  reestimate_core /
 * refit_* only. */
enum { FSTK_TRANSFORM_DCT = 0, FSTK_TRANSFORM_WHT = 1, FSTK_TRANSFORM_FFT = 2,
       FSTK_TRANSFORM_NONE = 3 };

typedef struct fstk_gpu_error {
  int32_t kind;     /* FSTK_E_* or 0 */
  int32_t mode;     /* Domain: offending mode, else -1 */
  int64_t index;    /* Domain: lowest offending point index, else -1 */
  double value;     /* Domain: offending coordinate */
  char message[256];
} fstk_gpu_error;

/*
 * Model descriptor: the content of fstk::FunctionalSparseTuckerModel
 * (model.hpp:33-59) flattened.  Functions are listed mode-major (all r_0
 * functions of mode 0, then mode 1, ...); per function: basis family
 * (0 = Legendre, 1 = wavelet), degree, resolution, domain [lo, hi] and its
 * SparseFit coefficients (lars.hpp:41-50): nnz strictly increasing u32 basis
 * indices with matching f64 values, concatenated over functions in order.
 */
typedef struct fstk_model_desc {
  int32_t d;                 /* 1..8 (kMaxOrder, tensor.hpp:16) */
  const int64_t* ranks;      /* d */
  const double* core;        /* prod(ranks), mode-0 fastest */
  const int32_t* family;     /* sum(ranks) */
  const int32_t* degree;     /* sum(ranks) */
  const int32_t* resolution; /* sum(ranks) */
  const double* lo;          /* sum(ranks) */
  const double* hi;          /* sum(ranks) */
  const uint32_t* nnz;       /* sum(ranks) */
  const uint32_t* indices;   /* sum(nnz) */
  const double* coeffs;      /* sum(nnz) */
} fstk_model_desc;

/* fstk::SketchConfig (randls.hpp:15-24). */
typedef struct fstk_sketch_cfg {
  uint64_t seed;
  uint64_t working_subset;   /* 0 = all training points; default 1<<20 */
  uint64_t sample_rows;      /* S; 0 = ceil(2.5 R) */
  int32_t transform;         /* FSTK_TRANSFORM_* */
  double validation_fraction;/* default 0.05 */
} fstk_sketch_cfg;

/* fstk::ReestimateResult fields (randls.hpp:52-60) plus stage timings. */
typedef struct fstk_reestimate_info {
  double residual_before;
  double residual_after;
  uint64_t sample_rows;
  uint64_t working_rows;
  uint64_t padded_rows;
  int32_t rank_deficient;
  int32_t held_out;
  /* device-timed stage seconds (CUDA events) */
  double t_prepare;   /* host RNG plan + gathers + mode tables */
  double t_sketch;    /* design-column generation + mixing + sampling */
  double t_gram;      /* A^T A and A^T b */
  double t_solve;     /* Cholesky (cuSOLVER), timed outside the hot-path claim */
  double t_residual;  /* validation residuals */
  double t_alloc;     /* host wall time of the sketch (A) allocation */
  int32_t gram_slices;  /* int8 digit planes of the Gram used (0 = native fp64) */
  int32_t refine_steps; /* iterative-refinement steps against A */
  double gram_int8_ops; /* int8 tensor-core ops (2 x multiply-adds) of the sliced Gram */
  /* Rank decision (randls.cpp:112-123).  The Cholesky route certifies full
   * rank when sigma_min(A) / max column norm > 100 R eps (sigma_ratio, its
   * estimate); otherwise qr_path = 1: streaming TSQR + pivoted QR of A with
   * Eigen's threshold decides, and a deficient system gets the COD's
   * minimum-norm solution. */
  int32_t qr_path;
  double sigma_ratio;
  /* Multi-device refit (fstk_gpu_set_devices(n > 1) before the model was
   * created; fstk_multi.cu): host wall seconds of the column-to-row
   * all-to-all and of the packed normal-equation reductions, the device
   * count (0 = single device) and the transport (1 = NCCL, 2 = peer copies). */
  double t_exchange;
  double t_reduce;
  int32_t devices;
  int32_t multi_transport;
} fstk_reestimate_info;

typedef struct fstk_gpu_model fstk_gpu_model;
typedef struct fstk_gpu_refit fstk_gpu_refit;

int32_t fstk_gpu_abi_version(void);
int32_t fstk_gpu_device_count(void);
/* Kernel launches issued by this process so far (evidence counter). */
uint64_t fstk_gpu_launch_count(void);
/* Device block cache (see fstk_common.cuh): released blocks >= 256 MB are
 * reused by size class, smaller ones in power-of-two buckets (<= 4 GB in
 * total), instead of going through cudaFree/cudaMalloc each time.  policy
 * 0 = off; 1 = per session (default): blocks are reused only while a refit
 * session is open and all go back to the driver when the last one ends, so
 * reestimate_core returns holding no idle HBM; 2 = persistent across
 * sessions (repeated refits of one size) until trimmed.  Returns the previous
 * policy.  FSTK_DEVICE_CACHE=0/1/2 sets the initial policy.  No reference
 * counterpart (the reference has no device memory). */
int32_t fstk_gpu_set_device_cache(int32_t policy);
/* Measurement mode (no reference counterpart): on != 0 runs every chunk of a
 * device-resident evaluation on one stream, so the mode-table and DMMA
 * contraction kernels do not overlap and their profiled durations are their
 * own (bench.py's roofline).  Values are unchanged.  Returns the previous. */
int32_t fstk_gpu_eval_serialize(int32_t on);
/* Returns the cached blocks to the driver: one device, or all when
 * device < 0.  Returns the bytes released. */
uint64_t fstk_gpu_trim_device_cache(int32_t device);

/* Builds the device-resident model.  Validates like the reference ctor
 * (model.cpp:22-53): Shape on count/domain mismatch, Parameter on invalid
 * bases.  Legendre and Alpert multiwavelet bases are both evaluated on the
 * GPU (basis.cpp:226-253); the evaluation workspaces are
 * allocated on the first evaluate call, not here. */
/* The devices of this process: a model created with device = -1
 * lives on ids[0] with replicas on the others, and a host evaluate_batch on it
 * splits the points into contiguous slabs, one per device, concurrently (the
 * reference's single-process call, spread over several GPUs).  n = 0 resets
 * to the current device.  Other entry points use the first device. */
int32_t fstk_gpu_set_devices(int32_t n, const int32_t* ids, fstk_gpu_error* err);
int32_t fstk_gpu_model_create(const fstk_model_desc* desc, int32_t device,
                              fstk_gpu_model** out, fstk_gpu_error* err);
void fstk_gpu_model_destroy(fstk_gpu_model* model);
/* FunctionalSparseTuckerModel::with_core (model.cpp:62-69), in place. */
int32_t fstk_gpu_model_set_core(fstk_gpu_model* model, const double* core,
                                fstk_gpu_error* err);
int32_t fstk_gpu_model_get_core(const fstk_gpu_model* model, double* core,
                                fstk_gpu_error* err);

/* Vector evaluate_batch(const Model&, const Matrix& points)  (model.cpp:208-227).
 * points: host, Q x d column-major (the Eigen buffer as-is); out: host, Q. */
int32_t fstk_gpu_evaluate_batch(const fstk_gpu_model* model, const double* points,
                                int64_t q, int32_t d, double* out,
                                fstk_gpu_error* err);
/* double evaluate(const Model&, const std::vector<double>& y) (model.cpp:195-206). */
int32_t fstk_gpu_evaluate(const fstk_gpu_model* model, const double* y, int32_t d,
                          double* out, fstk_gpu_error* err);
/* Device-resident variant: points column-major with leading dimension ld >= q,
 * out device, enqueued on `stream` (cudaStream_t or NULL for the legacy
 * stream); returns after enqueue unless a Domain error must be reported, which
 * requires one 16-byte read-back of the error flag (done on the same stream). */
int32_t fstk_gpu_evaluate_batch_device(const fstk_gpu_model* model,
                                       const double* points, int64_t ld,
                                       int64_t q, int32_t d, double* out,
                                       void* stream, fstk_gpu_error* err);
/* Vector Model::mode_values(int mode, double x) (model.cpp:71-94), batched:
 * out is n x r_mode column-major (host). */
int32_t fstk_gpu_mode_values(const fstk_gpu_model* model, int32_t mode,
                             const double* x, int64_t n, double* out,
                             fstk_gpu_error* err);

/* Matrix build_design_rows(const Model&, const Matrix& points) (randls.cpp:134-145):
 * w is Q x R column-major (host). */
int32_t fstk_gpu_build_design_rows(const fstk_gpu_model* model,
                                   const double* points, int64_t q, int32_t d,
                                   double* w, fstk_gpu_error* err);
/* SketchedSystem sketch(const Matrix& w, const Vector& u, const SketchConfig&)
 * (randls.cpp:147-184): a is rows x r column-major with rows = S (2S for FFT),
 * b has rows entries; padded_rows receives Q_pad. */
int32_t fstk_gpu_sketch(const double* w, const double* u, int64_t q, int64_t r,
                        const fstk_sketch_cfg* cfg, double* a, double* b,
                        uint64_t* padded_rows, fstk_gpu_error* err);
/* Matrix mixed_matrix(const Matrix& w, const SketchConfig&) (randls.cpp:186-225):
 * out is Q_pad x r (2 Q_pad x r for FFT) column-major. */
int32_t fstk_gpu_mixed_matrix(const double* w, int64_t q, int64_t r,
                              const fstk_sketch_cfg* cfg, double* out,
                              fstk_gpu_error* err);

/* ReestimateResult reestimate_core(const Model&, const PointCloud&, const SketchConfig&)
 * (randls.cpp:360-383).  points: host Q x d column-major, values: host Q.
 * core_out: host prod(ranks) (the new core, mode-0 fastest); the caller
 * builds the new model with with_core.  The refit runs on one GPU. */
int32_t fstk_gpu_reestimate_core(const fstk_gpu_model* model, const double* points,
                                 const double* values, int64_t q, int32_t d,
                                 const fstk_sketch_cfg* cfg, double* core_out,
                                 fstk_reestimate_info* info, fstk_gpu_error* err);

/* Staged refit for point/row-sharded multi-GPU runs (one process per GPU):
 * begin() does the host RNG plan (bit-exact, identical on every rank), the
 * gathers, mode tables and the sketch of the rows this shard owns
 * (sampled rows [S*shard/shards, S*(shard+1)/shards)); normal_equations()
 * writes this shard's partial A^T A (R x R, column-major, lower triangle) and
 * A^T b into caller-provided DEVICE buffers so the caller can sum them across
 * ranks (one NCCL all-reduce); solve() runs the Cholesky solve on the summed
 * system and the validation residuals. */
/* Host-only diagnostics of the bit-exact RNG replay (no device work, callable
 * without a GPU): rng.cpp sample_without_replacement of Rng(seed) (sorted,
 * min(n, k) values; the library replays the partial Fisher-Yates with O(k)
 * state) and make_plan (randls.cpp:54-75: signs[q_pad], rows[s], scale,
 * q_pad = next_pow2(q_w)). */
int32_t fstk_gpu_sample_without_replacement(uint64_t seed, uint64_t n, uint64_t k,
                                            uint64_t* out, fstk_gpu_error* err);
int32_t fstk_gpu_make_plan(uint64_t q_w, uint64_t s, uint64_t seed, double* signs,
                           uint64_t* rows, double* scale, uint64_t* q_pad, fstk_gpu_error* err);
int32_t fstk_gpu_refit_begin(const fstk_gpu_model* model, const double* points,
                             const double* values, int64_t q, int32_t d,
                             const fstk_sketch_cfg* cfg, int32_t shard,
                             int32_t shards, fstk_gpu_refit** out,
                             fstk_reestimate_info* info, fstk_gpu_error* err);
/* Column-sharded begin: the sketch transform -- replicated by
 * refit_begin's row sharding -- is split instead: this shard transforms
 * columns [(R+1) shard / shards, (R+1)(shard+1) / shards) of the R design
 * columns + rhs, for all S sample rows, written straight into a send buffer
 * packed per destination rank.  exchange_layout() then returns that buffer,
 * the receive buffer (this shard's S/shards-row slab, column-major, the
 * blocks of source g at its columns) and the per-peer element counts of one
 * all-to-all (ncclAllToAll / torch all_to_all_single); adopt_rows() finishes
 * the switch, after which the refit continues exactly as a row-sharded one
 * (normal_equations, factor, ...).  The rows are bit-identical to
 * refit_begin's.  transform = none (no transform) behaves like refit_begin. */
int32_t fstk_gpu_refit_begin_columns(const fstk_gpu_model* model, const double* points,
                                     const double* values, int64_t q, int32_t d,
                                     const fstk_sketch_cfg* cfg, int32_t shard,
                                     int32_t shards, fstk_gpu_refit** out,
                                     fstk_reestimate_info* info, fstk_gpu_error* err);
int32_t fstk_gpu_refit_exchange_layout(fstk_gpu_refit* refit, double** send,
                                       int64_t* send_counts, double** recv,
                                       int64_t* recv_counts, fstk_gpu_error* err);
int32_t fstk_gpu_refit_adopt_rows(fstk_gpu_refit* refit, fstk_gpu_error* err);
int32_t fstk_gpu_refit_normal_equations(fstk_gpu_refit* refit, double* gram,
                                        double* rhs, fstk_reestimate_info* info,
                                        fstk_gpu_error* err);
/* Same, always with the native fp64 DSYRK/DGEMM Gram (the fallback when the
 * sliced Gram is not positive definite or refinement stalls). */
int32_t fstk_gpu_refit_normal_equations_native(fstk_gpu_refit* refit, double* gram,
                                               double* rhs, fstk_reestimate_info* info,
                                               fstk_gpu_error* err);
/* Process-wide Gram arithmetic: slices > 0 runs A^T A on the int8 tensor
 * cores at the accuracy of that many 7-bit planes (levels 4..7: entries
 * rounded to (7 slices - 1)-bit integers per column and segment), or at the
 * preconditioner grades 3 and 2: 23- and 19-bit entries, the most that 8 and
 * 7 CRT moduli carry.  The default ($FSTK_GRAM_SLICES) is 2; the refinement
 * against A corrects what the Gram rounds away; transform = none and
 * sketches with fewer than 8 R rows take at least level 3 from this setting
 * (their systems are worse conditioned).
 * Products are exact (CRT over int8 residues; the
 * digit-plane split with FSTK_GRAM_SCHEME=digits); 0 selects the native fp64
 * Gram; < 0 only queries.  Returns the previous setting.  No reference
 * counterpart (an arithmetic choice of this backend; the solution still
 * matches the reference's QR). */
int32_t fstk_gpu_gram_slices(int32_t slices);

/* ---- scattered-to-grid interpolation ----
 * interpolate_to_grid (proj/src/ingest.cpp:265-383; ingest.hpp:44-62):
 * k-nearest-neighbour inverse-distance weighting over the reference's
 * uniform-binning spatial index, on the GPU.  points: Q x d column-major
 * (Eigen layout), values: Q; box_lo/box_hi: the cloud's bounding box (NULL =
 * the points' own, as PointCloud::from_data computes it); sizes / grid_lo /
 * grid_hi: the StructuredGrid (sizes >= 2, lo < hi); neighbors <= 0 selects
 * 2d + 2 (at most 64); power > 0.  out: prod(sizes) values, mode-0 fastest
 * (DenseTensor order).  report (optional) mirrors InterpolationReport;
 * neighbor_ids (optional): per node the k retained sample ids in ascending
 * (distance, id) order.  Errors as the reference: Shape (dimension), Data
 * (empty, non-finite, box), Parameter (grid, power).  The _device variant
 * takes device pointers and a stream. */
typedef struct fstk_interp_report {
  int32_t box_covered;
  double max_nearest_distance;
  double extrapolated_fraction;
} fstk_interp_report;
int32_t fstk_gpu_interpolate_to_grid(const double* points, const double* values, int64_t q, int32_t d,
                                     const double* box_lo, const double* box_hi, const int64_t* sizes,
                                     const double* grid_lo, const double* grid_hi, int32_t neighbors,
                                     double power, double* out, fstk_interp_report* report,
                                     uint32_t* neighbor_ids, int32_t device, fstk_gpu_error* err);
int32_t fstk_gpu_interpolate_to_grid_device(const double* points, const double* values, int64_t q, int32_t d,
                                            const double* box_lo, const double* box_hi, const int64_t* sizes,
                                            const double* grid_lo, const double* grid_hi, int32_t neighbors,
                                            double power, double* out, fstk_interp_report* report,
                                            uint32_t* neighbor_ids, void* stream, fstk_gpu_error* err);
/* The int8 GEMM engine of the CRT Gram: 1 = the hand-written sm_100a
 * tcgen05 SYRK (default: lower-triangle 256x256 tiles, 2-CTA UTCIMMA, TMA,
 * TMEM accumulators, residues reduced in the epilogue, dynamic tile
 * scheduler; fstk_syrk.cu), 2 = cuBLASLt IMMA GEMMs (kept for comparison;
 * $FSTK_GRAM_GEMM=cublaslt).  Both produce the
 * identical Gram bit for bit.  0 only queries.  Returns the previous setting. */
int32_t fstk_gpu_gram_engine(int32_t engine);
/* Packed normal equations (device pointers): unpack = 0 writes the lower
 * triangle of gram (n x n, column-major) column by column followed by rhs
 * into packed (n(n+1)/2 + n doubles); unpack != 0 restores gram's lower
 * triangle and rhs from packed.  The reduction payload of a row-sharded
 * refit (4.3 GB at R = 32,768 instead of the 8.6 GB square). */
int32_t fstk_gpu_pack_normal_equations(const double* gram, const double* rhs, int64_t n, double* packed,
                                       int32_t unpack, void* stream, fstk_gpu_error* err);
/* Measurement only (no reference counterpart): the tcgen05 int8 SYRK alone
 * on device residue planes (nm planes of kp x np int8, column-major; kp a
 * multiple of 128, np of 256), symmetric residues of the lower-triangle tile
 * sums into c (nm planes of np x np bytes). */
int32_t fstk_gpu_debug_syrk(const int8_t* planes, int32_t nm, int64_t kp, int64_t np, int8_t* c,
                            int32_t device, void* stream, fstk_gpu_error* err);
/* normal_equations() at an explicit Gram precision: slices 2..7 (sliced,
 * int8 tensor cores) or 0 (native fp64).  solve() and dist.refine_distributed
 * escalate with it: a sliced Gram that cannot precondition the system is
 * recomputed at 7, then at 0. */
int32_t fstk_gpu_refit_normal_equations_level(fstk_gpu_refit* refit, int32_t slices,
                                              double* gram, double* rhs,
                                              fstk_reestimate_info* info, fstk_gpu_error* err);
/* gram (n x n, column-major, lower triangle written) = A^T A for a DEVICE
 * matrix A (rows x n, column-major, lda), at `slices` plane-accuracy (2..7)
 * or native fp64 DSYRK/DGEMM (0), on `stream` (cudaStream_t, NULL = default).
 * The Gram stage of normal_equations() on its own, for tests and callers
 * that build their own design matrices. */
int32_t fstk_gpu_gram_device(const double* a, int64_t lda, int64_t rows, int32_t n,
                             double* gram, int32_t slices, int32_t device, void* stream,
                             fstk_gpu_error* err);
/* Lower Cholesky factor (in place, lower triangle) of a DEVICE n x n matrix
 * (column-major, ld n): blocked, panels of nb, with the trailing updates on
 * the int8 tensor cores at `slices` plane-accuracy (4..7), or cuSOLVER
 * dpotrf (0).  *info = 0 on success, nonzero when a block is not positive
 * definite.  The factor stage of fstk_gpu_refit_factor on its own (it uses
 * the int8 path for R >= 8192 unless FSTK_CHOL_CRT=0). */
int32_t fstk_gpu_cholesky_device(double* g, int32_t n, int32_t nb, int32_t slices, int32_t device,
                                 void* stream, int32_t* info, fstk_gpu_error* err);
int32_t fstk_gpu_refit_solve(fstk_gpu_refit* refit, const double* gram,
                             const double* rhs, double* core_out,
                             fstk_reestimate_info* info, fstk_gpu_error* err);
/* solve() for shards > 1, as explicit stages (device vectors of R doubles):
 * factor() Cholesky-factors the summed Gram (every rank) and writes the
 * normal-equations solution x; correction() writes this shard's
 * s = A_loc^T (b_loc - A_loc x); the caller sums s over ranks; apply() does
 * x += (A^T A)^{-1} s and reports ||dx||/||x||; repeat until it stalls
 * (iterative refinement = corrected semi-normal equations, converging to the
 * reference's QR least-squares solution); finish() copies x to the host core
 * and computes the validation residuals. */
/* factor(): info->rank_deficient = 1 means the Gram was not positive
 * definite (x = 0); the rank question then goes to the pivoted-QR stages
 * below.  */
int32_t fstk_gpu_refit_factor(fstk_gpu_refit* refit, const double* gram,
                              const double* rhs, double* x, fstk_reestimate_info* info,
                              fstk_gpu_error* err);
/* Rank decision of a sharded refit (randls.cpp:112-123), in stages:
 * certify() after the refinement has converged: estimates sigma_min(A) from
 * the Cholesky factor and the summed Gram's diagonal; *certified = 1 when
 * sigma_min / max column norm > 100 R eps, i.e. Eigen's ColPivHouseholderQR
 * would report full rank.  Otherwise, or when the Gram cannot be factored:
 * local_qr() writes the (R+1) x (R+1) upper R of this shard's [A b] (device,
 * column-major, streaming TSQR; A is left intact); the caller stacks the
 * shards' factors with fstk_gpu_qr_stack on one rank and calls qr_solve():
 * pivoted QR, Eigen's rank rule (threshold min(rows, R) eps max|R_ii|), the
 * QR solution or the COD minimum-norm solution into x, and
 * info->rank_deficient. */
/* Columns cols[0..ncols) of this shard's sketched A (index R = the
 * right-hand side b) in the reference's row order, column c at
 * out + c * rows_local (x2 for FFT): single-column parity checks at full size
 * without copying A (68.7 GB at C2) to the host. */
int32_t fstk_gpu_refit_sketched_columns(const fstk_gpu_refit* refit, const int64_t* cols,
                                        int64_t ncols, double* out, fstk_gpu_error* err);
int32_t fstk_gpu_refit_certify(fstk_gpu_refit* refit, const double* gram, double* sigma_ratio,
                               int32_t* certified, fstk_gpu_error* err);
int32_t fstk_gpu_refit_local_qr(fstk_gpu_refit* refit, double* raug, fstk_gpu_error* err);
int32_t fstk_gpu_refit_qr_solve(fstk_gpu_refit* refit, const double* raug, double* x,
                                fstk_reestimate_info* info, fstk_gpu_error* err);
/* top := R of [top; other] for two (n1 x n1) upper-triangular device
 * factors (column-major, ld n1): the stacking step of a sharded TSQR. */
int32_t fstk_gpu_qr_stack(double* top, const double* other, int64_t n1, int32_t device,
                          void* stream, fstk_gpu_error* err);
/* solve_system (randls.cpp:112-123) on the GPU for a host system a (m x n,
 * column-major) and b: ColPivHouseholderQR's rank with Eigen's default
 * threshold; x = the QR solution when rank == n, else the
 * CompleteOrthogonalDecomposition minimum-norm solution (*rank_deficient = 1). */
int32_t fstk_gpu_solve_system(const double* a, int64_t m, int64_t n, const double* b, double* x,
                              int32_t* rank, int32_t* rank_deficient, fstk_gpu_error* err);
int32_t fstk_gpu_refit_correction(fstk_gpu_refit* refit, const double* x, double* s,
                                  fstk_gpu_error* err);
int32_t fstk_gpu_refit_apply(fstk_gpu_refit* refit, const double* s, double* x,
                             double* rel_step, fstk_gpu_error* err);
int32_t fstk_gpu_refit_finish(fstk_gpu_refit* refit, const double* x, double* core_out,
                              fstk_reestimate_info* info, fstk_gpu_error* err);
void fstk_gpu_refit_end(fstk_gpu_refit* refit);
/* Diagnostics/tests: host copies of the sampled padded rows (S u64) and, when
 * the refit kept it, this shard's sketched block A (rows_local x R col-major)
 * and b. */
int32_t fstk_gpu_refit_rows(const fstk_gpu_refit* refit, uint64_t* rows,
                            fstk_gpu_error* err);
int32_t fstk_gpu_refit_sketched(const fstk_gpu_refit* refit, double* a,
                                double* b, int64_t* rows_local,
                                fstk_gpu_error* err);

/* ---- refit diagnostics ----------------------------------- */
/* std::vector<std::pair<uint64_t,double>> self_convergence(const Model&,
 * const PointCloud&, const std::vector<uint64_t>& s_values, const SketchConfig&)
 * (randls.hpp:70-75, randls.cpp:385-413): deltas[i] = ||a_{i+1}-a_i|| / ||a_{i+1}||
 * for i < n_s - 1 (the pair's first element is s_values[i]). */
int32_t fstk_gpu_self_convergence(const fstk_gpu_model* model, const double* points,
                                  const double* values, int64_t q, int32_t d,
                                  const fstk_sketch_cfg* cfg, const uint64_t* s_values,
                                  int32_t n_s, double* deltas, fstk_gpu_error* err);
/* Vector leverage_scores(const Matrix& w) (randls.hpp:50, randls.cpp:227-233):
 * w is q x r column-major (host), scores has q entries; rank_out (optional)
 * receives the numerical rank used. */
int32_t fstk_gpu_leverage_scores(const double* w, int64_t q, int64_t r, double* scores,
                                 int32_t* rank_out, fstk_gpu_error* err);

/* ---- tensor-product grids --------------------------------- */
/* All nodes of the Cartesian grid coords_0 x coords_1 x ... (coords: the
 * sizes[k] coordinates of mode k, concatenated mode by mode); out is
 * prod(sizes) values, mode-0 fastest (the FTEN layout).  Replaces the
 * point-by-point evaluate_batch of reconstruct --grid (pipeline.cpp:531-569)
 * and slice (:571-696) by a chain of mode products.  A coordinate outside its
 * mode's domain is a Domain error whose index is the node along that mode. */
int32_t fstk_gpu_evaluate_grid(const fstk_gpu_model* model, const double* coords,
                               const int64_t* sizes, int32_t d, double* out,
                               fstk_gpu_error* err);
/* reconstruct --grid: uniform nodes lo + (hi-lo) i/(I-1) on each mode's domain
 * (StructuredGrid::node, ingest.cpp:57-61); sizes >= 2. */
int32_t fstk_gpu_reconstruct_grid(const fstk_gpu_model* model, const int64_t* sizes,
                                  int32_t d, double* out, fstk_gpu_error* err);

/* FPTC ingest (format.md:29-44, ingest.cpp:706-742): converts the
 * file's point-major payload (device, Q x d row-major) into the column-major
 * SoA buffer the evaluation/refit entry points take, on `stream`. */
int32_t fstk_gpu_point_major_to_soa(const double* in, int64_t q, int32_t d, double* out,
                                    void* stream, fstk_gpu_error* err);

/* ---- measurement hooks (bench.py) ------------------------------------- */
/* Kernel classes timed by the profiling hook. */
enum {
  FSTK_PROF_MODE_TABLES = 0, /* K1a mode-value tables */
  FSTK_PROF_CONTRACT = 1,    /* K1b DMMA core contraction */
  FSTK_PROF_TRANSFORM = 2,   /* K3 design-column generation + mixing passes */
  FSTK_PROF_GRAM = 3,        /* K4 A^T A / A^T b */
  FSTK_PROF_SOLVE = 4,       /* Cholesky solve */
  FSTK_PROF_KINDS = 5
};
/* enable != 0: record a CUDA event pair around every launch of the classes
 * above, on the stream the kernel is launched on. */
void fstk_gpu_profile_enable(int32_t enable);
/* Synchronises the recorded events, writes per-class summed milliseconds and
 * launch counts (arrays of FSTK_PROF_KINDS) and clears the record. */
int32_t fstk_gpu_profile_read(double* ms, uint64_t* launches, fstk_gpu_error* err);
/* Measured fp64 tensor-core (DMMA m8n8k4) throughput of `device` in TFLOP/s:
 * the roofline denominator for the fp64 kernels (not in MEASURED_PEAKS.json). */
int32_t fstk_gpu_fp64_peak(int32_t device, double* dmma_tflops, double* dfma_tflops,
                           fstk_gpu_error* err);

#ifdef __cplusplus
}
#endif
#endif /* FSTK_GPU_H_ */
