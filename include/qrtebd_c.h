/*
 * qrtebd_c.h — C-ABI of the B200-native QR-TEBD bond update.
 *
 * This is the drop-in boundary for the hot path named in BASELINE.json:
 * the two-site QR/QR+CBE update of arXiv 2212.09782 and the observables that
 * read its output.  Every entry point replaces one function of the reference
 * C++ library (/root/reference/proj, cited as file:line below); the C++
 * mirror in include/qrtebd/qrtebd.hpp re-exposes them under the reference's
 * own names and types.
 *
 * Conventions (reference proj/include/qrtebd/tensor.hpp:14-61):
 *   - tensors are dense, row-major (last axis fastest), interleaved
 *     complex128: element k occupies doubles [2k, 2k+1] = (re, im);
 *   - site tensors are (d, chi_left, chi_right); bond matrices chi x chi;
 *     gates are (i_out, j_out, i_in, j_in) (gates.hpp:16-23);
 *   - qt_tensor handles live in device memory (HBM) and are owned by the
 *     caller; outputs are freshly allocated handles, inputs are never
 *     mutated (value semantics);
 *   - all work on a context is ordered on that context's CUDA stream; a
 *     context must not be used from two host threads at once;
 *   - errors map onto the reference taxonomy (errors.hpp:9-30):
 *     ShapeError -> QT_ERR_SHAPE, InputError -> QT_ERR_INPUT,
 *     NumericError -> QT_ERR_NUMERIC, CapacityError -> QT_ERR_CAPACITY;
 *     qt_last_error() returns the thread-local message of the last failure.
 *
 * There is no CPU fallback: every compute entry point runs sm_100a kernels
 * and fails with QT_ERR_CUDA when no suitable device is present.
 */
#ifndef QRTEBD_C_H
#define QRTEBD_C_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum qt_status {
  QT_OK = 0,
  QT_ERR_SHAPE = 1,
  QT_ERR_INPUT = 2,
  QT_ERR_NUMERIC = 3,
  QT_ERR_CAPACITY = 4,
  QT_ERR_CUDA = 5,
  QT_ERR_NCCL = 6,
  QT_ERR_INTERNAL = 7
} qt_status;

/* Scheme, proj/include/qrtebd/gates.hpp:30.  Only QR and QR_CBE run on the
 * device; SVD/EIG are the CPU comparators of the reference and are rejected
 * with QT_ERR_INPUT. */
typedef enum qt_scheme { QT_SCHEME_SVD = 0, QT_SCHEME_EIG = 1, QT_SCHEME_QR = 2, QT_SCHEME_QR_CBE = 3 } qt_scheme;

/* TruncationPolicy, proj/include/qrtebd/gates.hpp:43-55 (same fields, same
 * defaults via qt_policy_default). */
typedef struct qt_policy {
  uint64_t chi_max;            /* 1024 */
  double sv_cutoff;            /* 1e-14 */
  double target_eps;           /* 0 */
  uint64_t delta_chi_abs;      /* 100 */
  double delta_chi_rel;        /* 0.1 */
  uint64_t chi_max_expansion;  /* 0 = no cap */
  int32_t qr_sweeps;           /* 1 */
  int32_t compute_explicit_error; /* 1 */
  int32_t skip_renormalize;    /* 0 */
  int32_t reserved;
} qt_policy;

/* TruncationReport, proj/include/qrtebd/gates.hpp:57-64. */
typedef struct qt_report {
  uint64_t chi_before;
  uint64_t chi_expanded;
  uint64_t chi_after;
  double eps_trunc;
  double discarded_weight;
  int32_t scheme;
  int32_t reserved;
} qt_report;

/* BondReport, proj/include/qrtebd/gates.hpp:106-109. */
typedef struct qt_bond_report {
  uint64_t bond;
  qt_report report;
} qt_bond_report;

typedef struct qt_ctx qt_ctx;
typedef struct qt_tensor qt_tensor;

/* ---- library ------------------------------------------------------------ */
const char* qt_last_error(void);
const char* qt_version(void);
/* TruncationPolicy{} defaults, gates.hpp:44-53. */
void qt_policy_default(qt_policy* p);
/* TruncationPolicy::expanded_dim, proj/src/gates.cpp:94-101. */
uint64_t qt_expanded_dim(const qt_policy* p, uint64_t chi, uint64_t d);
/* number of device kernels this library has launched (bench bookkeeping) */
uint64_t qt_kernel_launches(void);

/* ---- context ------------------------------------------------------------ */
/* stream == NULL: the context creates and owns a non-blocking stream. */
qt_status qt_ctx_create(int device, void* stream, qt_ctx** out);
qt_status qt_ctx_destroy(qt_ctx* ctx);
qt_status qt_ctx_synchronize(qt_ctx* ctx);
void* qt_ctx_stream(qt_ctx* ctx);
/* Performance knob: the smallest two-site block height (d * chi_left rows)
 * whose update takes the pipelined QR pair on this context (default 128;
 * rows < 0 restores the default).  Contexts that run concurrently with
 * other contexts (sharded chains) set 256: there the pair's side streams
 * cost more than they hide.  Results agree with the other path to rounding. */
qt_status qt_ctx_set_qr_pair_min_rows(qt_ctx* ctx, int64_t rows);

/* ---- device tensors (ComplexTensor, tensor.hpp:18-61) --------------------- */
qt_status qt_tensor_create(qt_ctx* ctx, int rank, const uint64_t* shape, qt_tensor** out);
/* non-owning view of caller device memory (interleaved complex128) */
qt_status qt_tensor_wrap(qt_ctx* ctx, int rank, const uint64_t* shape, void* device_ptr, qt_tensor** out);
qt_status qt_tensor_free(qt_tensor* t);
/* shape4 receives up to 4 extents; *rank the number of axes */
qt_status qt_tensor_shape(const qt_tensor* t, int* rank, uint64_t* shape4);
void* qt_tensor_data(const qt_tensor* t);
/* synchronous host<->device copies of 2*numel doubles */
qt_status qt_tensor_upload(qt_tensor* t, const double* host);
qt_status qt_tensor_download(const qt_tensor* t, double* host);
/* asynchronous variants (host memory should be pinned) */
qt_status qt_tensor_upload_async(qt_tensor* t, const double* host);
qt_status qt_tensor_download_async(const qt_tensor* t, double* host);
/* device-to-device copy of equal element counts (stream-ordered on dst's context) */
qt_status qt_tensor_copy(qt_tensor* dst, const qt_tensor* src);

/* ---- linear algebra (proj/src/linalg.cpp:40-64) --------------------------- */
/* qr_reduced: m (p x q) = Q (p x k) R (k x q), k = min(p,q), R_ii real >= 0 */
qt_status qt_qr_reduced(qt_ctx* ctx, const qt_tensor* m, qt_tensor** q_out, qt_tensor** r_out);
/* lq_reduced: m (p x q) = L (p x k) Q (k x q), L_ii real >= 0 */
qt_status qt_lq_reduced(qt_ctx* ctx, const qt_tensor* m, qt_tensor** l_out, qt_tensor** q_out);

/* Batched complex GEMM on raw device pointers (interleaved complex128):
 * C[b] = alpha * op(A[b]) op(B[b]) + beta * C[b], op: 0 = N, 1 = conjugate
 * transpose.  Strides/leading dimensions in complex elements.  This is the
 * contraction kernel behind contract() (proj/src/tensor.cpp:172-233). */
qt_status qt_zgemm(qt_ctx* ctx, int op_a, int op_b, int64_t m, int64_t n, int64_t k, int batch,
                   const void* a, int64_t lda, int64_t stride_a, const void* b, int64_t ldb, int64_t stride_b,
                   void* c, int64_t ldc, int64_t stride_c, double alpha, double beta);

/* ---- two-site updates (proj/include/qrtebd/gates.hpp:84-92) --------------- */
/* apply_gate_qr     gates.cpp:343-386
 * apply_gate_qr_cbe gates.cpp:388-450
 * Outputs: b_m (d, chi_l, chi~), xi (chi~ x chi~), b_n (d, chi~, chi_r) and,
 * for QR only, left_iso (d, chi_l, chi~) (pass NULL to skip it). */
qt_status qt_apply_gate(qt_ctx* ctx, qt_scheme scheme, const qt_tensor* xi, const qt_tensor* b_m,
                        const qt_tensor* b_n, const qt_tensor* u, const qt_policy* policy, qt_tensor** b_m_out,
                        qt_tensor** xi_out, qt_tensor** b_n_out, qt_tensor** left_iso_out, qt_report* report);
qt_status qt_apply_gate_qr(qt_ctx* ctx, const qt_tensor* xi, const qt_tensor* b_m, const qt_tensor* b_n,
                           const qt_tensor* u, const qt_policy* policy, qt_tensor** b_m_out, qt_tensor** xi_out,
                           qt_tensor** b_n_out, qt_tensor** left_iso_out, qt_report* report);
qt_status qt_apply_gate_qr_cbe(qt_ctx* ctx, const qt_tensor* xi, const qt_tensor* b_m, const qt_tensor* b_n,
                               const qt_tensor* u, const qt_policy* policy, qt_tensor** b_m_out,
                               qt_tensor** xi_out, qt_tensor** b_n_out, qt_report* report);

/* truncation_error_explicit, gates.cpp:464-485: ||theta - A (C B)||^2/||theta||^2 */
qt_status qt_truncation_error_explicit(qt_ctx* ctx, const qt_tensor* theta, const qt_tensor* left,
                                       const qt_tensor* center, const qt_tensor* right, double* out);

/* ---- uniform TEBD step (gates.cpp:513-540) -------------------------------- */
/* State of a UniformMPS (mps.hpp:18-26): sites[m] (d, chi, chi), bonds[m]
 * (chi x chi).  layers[l] has parity parity[l] (0 even, 1 odd) and gate
 * gates[l].  New handles are written to sites_out / bonds_out (the inputs
 * are untouched); reports receives one entry per update (capacity
 * *n_reports on entry, count on exit). */
qt_status qt_tebd_step_uniform(qt_ctx* ctx, uint64_t cell_length, qt_tensor* const* sites, qt_tensor* const* bonds,
                               uint64_t n_layers, const int32_t* parity, qt_tensor* const* gates, qt_scheme scheme,
                               const qt_policy* policy, qt_tensor** sites_out, qt_tensor** bonds_out,
                               qt_bond_report* reports, uint64_t* n_reports);

/* ---- device-resident uniform state (fast path) ----------------------------- */
/* A UniformMPS kept in HBM across steps (double-buffered site tensors and bond
 * matrices).  qt_uniform_step performs tebd_step (gates.cpp:513-540) in place;
 * with use_graph != 0 and stationary bond dimensions (QR scheme, eta == chi)
 * the step is captured once per buffer-parity pattern and replayed as a
 * single CUDA graph launch.  Views returned by qt_uniform_view alias the live
 * buffers (non-owning; invalid after the next step, free the handle with
 * qt_tensor_free). */
typedef struct qt_uniform qt_uniform;
qt_status qt_uniform_create(qt_ctx* ctx, uint64_t cell_length, qt_tensor* const* sites, qt_tensor* const* bonds,
                            qt_uniform** out);
qt_status qt_uniform_destroy(qt_uniform* u);
qt_status qt_uniform_step(qt_uniform* u, uint64_t n_layers, const int32_t* parity, qt_tensor* const* gates,
                          qt_scheme scheme, const qt_policy* policy, int32_t use_graph, qt_bond_report* reports,
                          uint64_t* n_reports);
/* which: 0 = site tensor m, 1 = bond matrix m (bond left of site m) */
qt_status qt_uniform_view(qt_uniform* u, int which, uint64_t m, qt_tensor** out);

/* ---- observables (proj/src/mps.cpp) --------------------------------------- */
/* expectation_local(UniformMPS), mps.cpp:168-186: <op> on a site given the
 * bond matrix to its left and the site tensor; out = (re, im). */
qt_status qt_expectation_local(qt_ctx* ctx, const qt_tensor* xi_left, const qt_tensor* b, const qt_tensor* op,
                               double* out2);
/* schmidt_values, mps.cpp:198-201: singular values of the bond matrix,
 * descending; out has capacity *n on entry, count on exit. */
qt_status qt_schmidt_values(qt_ctx* ctx, const qt_tensor* xi, double* out, uint64_t* n);
/* eigh, proj/src/linalg.cpp:79-101: Hermitian (symmetrized) n x n matrix ->
 * eigenvalues descending (host array of n) and eigenvectors as the columns of
 * a new n x n device tensor (device block-Jacobi solver). */
qt_status qt_eigh(qt_ctx* ctx, const qt_tensor* h, double* w_host, qt_tensor** v_out);
/* right_defect, mps.cpp:34-36: || sum_i B^i B^i^H - 1 ||_max */
qt_status qt_right_defect(qt_ctx* ctx, const qt_tensor* b, double* out);
/* check_isometric(UniformMPS, tol), proj/src/mps.cpp:105-141 (IsometryReport,
 * proj/include/qrtebd/mps.hpp:40-53): per site the right defect; per bond the
 * cell fixed-point ("left") and translation defects of the left weight
 * lambda = Xi^T conj(Xi) and | ||Xi|| - 1 |.  Each per-index array (length
 * cell_length) may be NULL; pass = max defect <= tol. */
typedef struct qt_isometry_report {
  double max_right_defect;
  double max_left_defect;
  double max_translation_defect;
  double max_norm_defect;
  int32_t pass;
  int32_t reserved;
} qt_isometry_report;
qt_status qt_check_isometric_uniform(qt_ctx* ctx, uint64_t cell_length, qt_tensor* const* sites,
                                     qt_tensor* const* bonds, double tol, double* right_defects,
                                     double* left_defects, double* translation_defects, double* norm_defects,
                                     qt_isometry_report* out);
/* Bond energy <theta0|h|theta0>/<theta0|theta0>, theta0 = Xi B^m B^n
 * (an extension, not in the reference). */
qt_status qt_bond_energy(qt_ctx* ctx, const qt_tensor* xi, const qt_tensor* b_m, const qt_tensor* b_n,
                         const qt_tensor* h_bond, double* out);

/* ---- finite chain, reference semantics (FiniteMPS, proj/include/qrtebd/mps.hpp:31-38) ----
 * An open-chain MPS with an explicit orthogonality-center bond kept in HBM:
 * n site tensors (d, chi_l, chi_r), center_bond in [0, n], and the center
 * matrix (possibly rectangular after a rank-revealing gauge move,
 * proj/src/mps.cpp:328-330).  qt_finite_create copies its inputs. */
typedef struct qt_finite qt_finite;
qt_status qt_finite_create(qt_ctx* ctx, uint64_t n_sites, qt_tensor* const* sites, uint64_t center_bond,
                           const qt_tensor* center, qt_finite** out);
qt_status qt_finite_destroy(qt_finite* f);
qt_status qt_finite_clone(const qt_finite* f, qt_finite** out);
qt_status qt_finite_center_bond(const qt_finite* f, uint64_t* out);
/* which: 0 = site tensor m, 1 = the center matrix (m ignored); non-owning view */
qt_status qt_finite_view(qt_finite* f, int which, uint64_t m, qt_tensor** out);
/* move_center, proj/src/mps.cpp:226-257 (in place; QR moves right, LQ moves left) */
qt_status qt_finite_move_center(qt_finite* f, uint64_t new_center);
/* tebd_step(FiniteMPS), proj/src/gates.cpp:542-578, in place: layers[l] has
 * parity parity[l] and one gate per bond, gates[l * (n - 1) + m] acting on
 * sites (m, m+1) (FiniteLayer, proj/include/qrtebd/gates.hpp:130-137).  The
 * center is moved onto bond m before every update; QR keeps left_iso and
 * moves the center to m+1, QR_CBE keeps the center and renormalizes b_m. */
qt_status qt_finite_step(qt_finite* f, uint64_t n_layers, const int32_t* parity, qt_tensor* const* gates,
                         qt_scheme scheme, const qt_policy* policy, qt_bond_report* reports, uint64_t* n_reports);
/* The same with an observer (FiniteGateObserver, proj/include/qrtebd/gates.hpp:
 * 120-123, :149-152) called after every gate with that gate's report; the
 * state (qt_finite_view) is consistent and synchronized inside the call.  A
 * nonzero return aborts the step with QT_ERR_INTERNAL. */
typedef int (*qt_gate_observer)(void* user, const qt_bond_report* report);
qt_status qt_finite_step_observed(qt_finite* f, uint64_t n_layers, const int32_t* parity, qt_tensor* const* gates,
                                  qt_scheme scheme, const qt_policy* policy, qt_bond_report* reports,
                                  uint64_t* n_reports, qt_gate_observer observer, void* user);
/* expectation_local(FiniteMPS) (mps.cpp:188-196) on every site and
 * schmidt_values(FiniteMPS) (mps.cpp:203-207) of every bond 0..n, from one
 * gauge sweep over a copy of the state.  z_out: 2n doubles or NULL (op NULL
 * skips them); bond b's values land at schmidt_out[offsets[b] ..
 * offsets[b+1]) when offsets[n+1] <= cap; offsets (n+2 entries) is always
 * filled, so a first call with cap = 0 sizes the buffer. */
qt_status qt_finite_observables(const qt_finite* f, const qt_tensor* op, double* z_out, double* schmidt_out,
                                uint64_t cap, uint64_t* offsets);

/* left_defect, proj/src/mps.cpp:39-41: || sum_i B^i^H B^i - 1 ||_max */
qt_status qt_left_defect(qt_ctx* ctx, const qt_tensor* b, double* out);
/* check_isometric(FiniteMPS, tol), proj/src/mps.cpp:143-164: left defects of
 * the sites left of the center, right defects of the others, | ||C|| - 1 | of
 * the center matrix; per-site arrays (length n) may be NULL. */
qt_status qt_check_isometric_finite(const qt_finite* f, double tol, double* right_defects, double* left_defects,
                                    double* norm_defect, qt_isometry_report* out);

/* ---- sharded finite chain (Hastings form), SURVEY.md §8(a) a10, §8(e) ------
 * An open chain of n sites cut into contiguous, even-aligned site blocks, one
 * per rank (process + GPU); the bond matrix Xi[m] sits left of site m (Xi[0] =
 * [[1]]).  A layer of parity P updates every bond (m, m+1), m = P mod 2
 * (proj/src/gates.cpp:513-540 without the wraparound); interior bonds run
 * concurrently on n_workers worker contexts, and the bond straddling a block
 * boundary is updated by the left rank after the right rank sent it its first
 * site tensor (ncclSend / ncclRecv of raw device buffers on a dedicated
 * stream; shapes travel in a small header first), Xi[e] and B[e] going back.
 * The result is bitwise the single-rank chain's.  world == 1 needs no
 * transport; world > 1 takes an NCCL unique id (qt_nccl_get_unique_id on
 * rank 0, broadcast by the caller) or an in-process loopback shared by one
 * chain per rank in separate host threads (tests on one GPU). */
typedef struct qt_chain qt_chain;
typedef struct qt_loopback qt_loopback;
qt_status qt_nccl_get_unique_id(uint8_t* id128);
/* diagnostics: a one-rank NCCL communicator sends `bytes` to itself through a
 * grouped ncclSend/ncclRecv on `device`; *ok = 1 when the bytes round-trip */
qt_status qt_nccl_selftest(int device, uint64_t bytes, int* ok);
qt_status qt_loopback_create(int world, qt_loopback** out);
qt_status qt_loopback_destroy(qt_loopback* l);
/* the owned sites [*begin, *end) of rank in world */
qt_status qt_chain_partition(uint64_t n_sites, int world, int rank, uint64_t* begin, uint64_t* end);
/* sites / bonds: the owned site tensors and the bond matrices left of them,
 * indexed from *begin (copied) */
qt_status qt_chain_create(qt_ctx* ctx, uint64_t n_sites, int rank, int world, const uint8_t* nccl_id,
                          qt_loopback* loopback, qt_tensor* const* sites, qt_tensor* const* bonds, int n_workers,
                          qt_chain** out);
qt_status qt_chain_destroy(qt_chain* c);
qt_status qt_chain_range(const qt_chain* c, uint64_t* begin, uint64_t* end);
/* which: 0 = site tensor m, 1 = bond matrix left of site m (owned m; non-owning view) */
qt_status qt_chain_view(qt_chain* c, int which, uint64_t m, qt_tensor** out);
/* one Trotter step: layers[l] has parity parity[l] and gates[l * (n - 1) + m]
 * on bond (m, m+1) (entries of bonds this rank does not update may be NULL);
 * reports: this rank's updates, bond order per layer */
qt_status qt_tebd_step_finite_sharded(qt_chain* c, uint64_t n_layers, const int32_t* parity, qt_tensor* const* gates,
                                      qt_scheme scheme, const qt_policy* policy, qt_bond_report* reports,
                                      uint64_t* n_reports);

/* ---- diagnostics ---------------------------------------------------------- */
/* Per-launch CUDA-event profile of the DMMA GEMM kernel (roofline evidence):
 * between begin and end every GEMM launch is bracketed by events; end
 * synchronizes and returns summed algorithmic flops, device ms and launches.
 * Only launches of at least min_flops algorithmic flops are bracketed (each
 * event pair is a node of the captured step graph; the small Householder
 * block-reflector products are left out to keep the graph lean). */
qt_status qt_profile_begin(qt_ctx* ctx, double min_flops);
qt_status qt_profile_end(qt_ctx* ctx, double* gemm_flops, double* gemm_ms, uint64_t* gemm_launches);
/* measured FP64 peak of this device in TFLOP/s: kind 0 = DMMA, 1 = DFMA */
qt_status qt_fp64_peak(qt_ctx* ctx, int kind, double* tflops);

#ifdef __cplusplus
}
#endif

#endif /* QRTEBD_C_H */
