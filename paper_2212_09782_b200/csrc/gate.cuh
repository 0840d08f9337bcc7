// Two-site update engine (apply_gate_qr / apply_gate_qr_cbe) and the
// observable contractions, device-resident.
#pragma once

#include <functional>
#include <utility>
#include <vector>

#include "engine.cuh"
#include "../../include/qrtebd_c.h"

namespace qt {

struct Dims {
  long long d = 0, chi_l = 0, chi_m = 0, chi_n = 0, chi_r = 0;
  long long rows() const { return chi_l * d; }
  long long cols() const { return d * chi_r; }
};

// TruncationPolicy::expanded_dim, proj/src/gates.cpp:94-101
unsigned long long expanded_dim(const qt_policy& p, unsigned long long chi, unsigned long long d);

// working width of apply_gate_qr, proj/src/gates.cpp:354-355
long long qr_eta(const qt_policy& p, const Dims& D);
// working width of apply_gate_qr_cbe, proj/src/gates.cpp:398-401 (throws InputError past d*chi)
long long cbe_eta(const qt_policy& p, const Dims& D);

struct GateBuffers {
  double2* b_m = nullptr;       // (d, chi_m, chi~)
  double2* xi = nullptr;        // chi~ x chi~
  double2* b_n = nullptr;       // (d, chi~, chi_r)
  double2* left_iso = nullptr;  // (d, chi_l, chi~) or nullptr
};

struct HostReport {
  double theta2 = 0, kept2 = 0, resid = 0;
  bool finite = true;
};

// theta build (K1a/K1b/K1c, proj/src/gates.cpp:123-182): fills the engine
// slots S_PHIEV (beta,i,j,delta) and S_THETA (alpha,i,j,delta); ||theta||^2 is
// written to dscal[out_scalar].
void build_theta(Engine& e, const Dims& D, const double2* xi, const double2* bm, const double2* bn,
                 const double2* u, int out_scalar);

// apply_gate_qr (proj/src/gates.cpp:343-386) with outputs written into
// caller-allocated buffers sized for eta = qr_eta(policy, D).  Fully
// asynchronous on e.stream; the report scalars stay in e.dscal.
void gate_qr_async(Engine& e, const Dims& D, const double2* xi, const double2* bm, const double2* bn,
                   const double2* u, const qt_policy& pol, long long eta, const GateBuffers& out);

// Y = Q_m^H theta through the reflectors of QR(X) (QrOpts::capply): used for
// one sweep on matrices up to QT_QTHETA_MAX_ROWS rows (default 2048)
bool use_qtheta(const Engine& e, const qt_policy& pol, long long rows);
// Y^H (cols x eta) from Q_full^H theta (rows x cols) with the gauge phases of
// the factored X (diag of a, ld eta)
// (rows [ibeg, iend) only, on stream st; iend < 0: all eta rows, st null: e.stream)
void qtheta_yh(Engine& e, const double2* qt, long long cols, const double2* a, long long eta, double2* yh,
               long long ibeg = 0, long long iend = -1, cudaStream_t st = nullptr);
// the two QRs of the sweep run as a pipelined pair (qr_pair_pipelined) when
// both heights fit one block-reflector cluster (QT_NO_QR_PAIR disables it)
bool use_qr_pair(long long rows, long long cols);
// X = theta xb^H (xb_h) or theta xb for the pipelined pair, in two column
// blocks: the first two panels' kXHead columns on e.stream, the rest on
// e.side concurrently with panel 0 (e.side carries the pair's wide
// look-ahead updates, the first work to touch those columns, so stream order
// is the dependency; e.side2, where the pair first writes theta, waits for
// it).  Non-finite entries set *flag.  C2: 203 -> 216 steps/s.
// QT_NO_X_SPLIT=1 forms X in one GEMM.
constexpr long long kXHead = 64;
long long x_head_cols();  // kXHead, or QT_X_HEAD (a multiple of 32, >= 64; diagnostics)
bool x_split_applies(const Engine& e, long long eta);
void x_gemm_split(Engine& e, long long rows, long long eta, long long cols, const double2* theta,
                  const double2* xb, bool xb_h, double2* X, int* flag);
// *out = ||Y - W||^2 + ||Z||^2 = ||theta - Q_m W||^2 (W: eta x cols), fixed-order reduction
void qtheta_resid(Engine& e, const double2* qt, long long rows, long long cols, const double2* a, long long eta,
                  const double2* w, double* out, cudaStream_t st = nullptr);

// Collects the report of the last gate_qr_async / CBE update (synchronizes).
HostReport read_report(Engine& e);

// apply_gate_qr_cbe (proj/src/gates.cpp:388-450).  Data-dependent kept
// width: allocates outputs through `alloc` once kk is known (one host sync).
struct CbeResult {
  long long eta = 0, kk = 0;
  HostReport rep;
};
CbeResult gate_cbe(Engine& e, const Dims& D, const double2* xi, const double2* bm, const double2* bn,
                   const double2* u, const qt_policy& pol, const std::function<GateBuffers(long long)>& alloc);

// eigh of a Hermitian n x n matrix on the device (proj/src/linalg.cpp:79-101):
// eigenvalues descending into w (device), eigenvectors as columns of v (device, ld n)
// Returns a device pointer to the solver status (sweeps > 0: a full sweep
// rotated nothing; < 0: stopped at the sweep cap -- then the off-diagonal mass
// left decides, require_eigh_converged).
struct EighStatus {
  int sweeps;
  int pad;
  double offdiag2;  // ||offdiag(G_final)||_F^2 (scaled frame)
  double fro2;      // ||G||_F^2 (scaled frame)
};
const EighStatus* eigh_device(Engine& e, const double2* h, long long n, double* w, double2* v);
void require_eigh_converged(const EighStatus& st, long long n);
// out2[0] = ||h - h^H||_F^2, out2[1] = ||h||_F^2 (device, deterministic)
void hermitian_defect(Engine& e, const double2* h, long long n, double* out2);
// singular values of an arbitrary p x q matrix, descending; returns a device
// pointer (engine slot S_EIG_W) to min(p,q) values
double* singular_values_device(Engine& e, const double2* m, long long p, long long q);

// check_isometric(UniformMPS), proj/src/mps.cpp:105-141: per-site right
// defects, per-bond cell fixed-point ("left") and translation defects of the
// left weights, and per-bond norm defects
struct IsometryParts {
  std::vector<double> right, left, translation, norm;
};
IsometryParts check_isometric_uniform(Engine& e, long long d, const std::vector<long long>& chi,
                                      const std::vector<const double2*>& sites,
                                      const std::vector<const double2*>& bonds);

// device-resident UniformMPS with graph-replayed steps (uniform.cu)
struct UniformDev;
UniformDev* uniform_create(Engine& e, int L, long long d, const std::vector<long long>& chi,
                           const std::vector<const double2*>& sites, const std::vector<const double2*>& bonds);
void uniform_destroy(UniformDev* s);
double2* uniform_live(UniformDev* s, int which, int m, long long* shape);
struct StepRecord {
  int bond;
  long long before, eta, after;
  HostReport rep;
};
std::vector<StepRecord> uniform_step(UniformDev* s, const std::vector<std::pair<int, const double2*>>& layers,
                                     int scheme_qr, const qt_policy& pol, bool use_graph);

// observables (proj/src/mps.cpp)
void expectation_local(Engine& e, const double2* xi, long long xi_rows, long long chi_l, const double2* b,
                       long long d, long long chi_r, const double2* op, double* out2_host);
double right_defect(Engine& e, const double2* b, long long d, long long chi_l, long long chi_r);
double left_defect(Engine& e, const double2* b, long long d, long long chi_l, long long chi_r);
double bond_energy(Engine& e, const Dims& D, const double2* xi, const double2* bm, const double2* bn,
                   const double2* h);
double explicit_error(Engine& e, const double2* theta, long long rows, long long cols, const double2* left,
                      long long kdim, const double2* center, long long kdim2, const double2* right);

}  // namespace qt
