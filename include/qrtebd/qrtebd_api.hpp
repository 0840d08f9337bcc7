// qrtebd_api.hpp -- the reference's C++ API, B200-backed.
//
// Declares, in namespace qrtebd, the public types and functions of the
// reference library's tensor, error, linalg, gates and MPS headers
// (/root/reference/proj/include/qrtebd/{tensor,errors,linalg,gates,mps}.hpp)
// with identical names, signatures and class layouts, so code written
// against the reference -- including the reference's own test suites,
// compiled unmodified -- links against libqrtebd_api.so
// (paper_2212_09782_b200/cpp/qrtebd_api.cpp) instead.
//
// libqrtebd_api.so implements the hot path on the B200 through the C-ABI
// (include/qrtebd_c.h): the tensor layer (contract on the device GEMM),
// qr_reduced / lq_reduced / eigh, apply_gate_qr / apply_gate_qr_cbe /
// apply_gate / truncation_error_explicit, tebd_step (uniform and finite, with
// observers), move_center and the observables.  The host-side rest of the
// reference -- the clock model and ED oracle, gate construction (make_gate,
// trotter_schedule), the SVD/EIG comparators, product states, checkpoint
// I/O, the driver -- stays in the reference library: a maintainer links
// libqrtebd_api.so AHEAD of the reference's libqrtebd and those symbols
// resolve there.  Every call is synchronous and uses a
// per-thread default device context (qrtebd::b200::set_device).
#ifndef QRTEBD_API_HPP
#define QRTEBD_API_HPP

#include <complex>
#include <cstddef>
#include <functional>
#include <initializer_list>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <variant>
#include <vector>

namespace qrtebd {

using cplx = std::complex<double>;

// ---- error taxonomy (exit codes 1 / 1 / 2 / 3 in the reference CLI) -----------
class ShapeError : public std::invalid_argument {
 public:
  explicit ShapeError(const std::string& what) : std::invalid_argument(what) {}
};
class InputError : public std::invalid_argument {
 public:
  explicit InputError(const std::string& what) : std::invalid_argument(what) {}
};
class NumericError : public std::runtime_error {
 public:
  explicit NumericError(const std::string& what) : std::runtime_error(what) {}
};
class CapacityError : public std::runtime_error {
 public:
  explicit CapacityError(const std::string& what) : std::runtime_error(what) {}
};

// ---- host tensor: row-major complex128, last axis fastest -------------------------
class ComplexTensor {
 public:
  ComplexTensor() = default;
  explicit ComplexTensor(std::vector<std::size_t> shape);
  ComplexTensor(std::vector<std::size_t> shape, std::vector<cplx> data);

  static ComplexTensor zeros(std::vector<std::size_t> shape);
  static ComplexTensor identity(std::size_t n);
  static ComplexTensor matrix(std::size_t rows, std::size_t cols, std::vector<cplx> data);

  std::size_t rank() const { return shape_.size(); }
  const std::vector<std::size_t>& shape() const { return shape_; }
  std::size_t dim(std::size_t axis) const;
  std::size_t size() const { return data_.size(); }

  cplx& at(std::initializer_list<std::size_t> idx);
  const cplx& at(std::initializer_list<std::size_t> idx) const;

  std::vector<cplx>& data() { return data_; }
  const std::vector<cplx>& data() const { return data_; }

  ComplexTensor reshape(std::vector<std::size_t> new_shape) const&;
  ComplexTensor reshape(std::vector<std::size_t> new_shape) &&;
  ComplexTensor transpose(const std::vector<std::size_t>& perm) const;
  ComplexTensor conj() const;

  double norm() const;
  bool all_finite() const;

  ComplexTensor& operator*=(cplx factor);
  friend ComplexTensor operator*(cplx factor, ComplexTensor t) {
    t *= factor;
    return t;
  }

 private:
  std::vector<std::size_t> shape_;
  std::vector<cplx> data_;
};

/// Sum over the (axis of a, axis of b) pairs; the result keeps a's free axes,
/// then b's.  Computed on the device GEMM (qt_zgemm).
ComplexTensor contract(const ComplexTensor& a, const ComplexTensor& b,
                       const std::vector<std::pair<std::size_t, std::size_t>>& axes);

// ---- linear algebra ------------------------------------------------------------------
struct QrResult {
  ComplexTensor q;  // p x k
  ComplexTensor r;  // k x q, diag real >= 0
};
struct LqResult {
  ComplexTensor l;  // p x k, diag real >= 0
  ComplexTensor q;  // k x q
};
struct SvdResult {
  ComplexTensor u;
  std::vector<double> s;
  ComplexTensor vdag;
};
struct EighResult {
  std::vector<double> w;  // descending
  ComplexTensor v;
};

QrResult qr_reduced(const ComplexTensor& m);  // device Householder QR
LqResult lq_reduced(const ComplexTensor& m);  // device, QR of the adjoint
EighResult eigh(const ComplexTensor& h);      // device block Jacobi
SvdResult svd(const ComplexTensor& m);        // host library (comparators)
ComplexTensor expm_hermitian(const ComplexTensor& h, double t);  // host library

// ---- MPS containers and observables -----------------------------------------------
struct UniformMPS {
  std::size_t phys_dim = 0;
  std::vector<ComplexTensor> site_tensors;   // (d, chi_left, chi_right), right-isometric
  std::vector<ComplexTensor> bond_matrices;  // bond LEFT of site m, unit norm
  std::size_t cell_length() const { return site_tensors.size(); }
  std::size_t bond_dim(std::size_t m) const { return bond_matrices[m].dim(0); }
};

struct FiniteMPS {
  std::size_t phys_dim = 0;
  std::vector<ComplexTensor> site_tensors;
  std::size_t center_bond = 0;
  ComplexTensor center_matrix;
  std::size_t length() const { return site_tensors.size(); }
};

struct IsometryReport {
  std::vector<double> right_defects;
  std::vector<double> left_defects;
  std::vector<double> translation_defects;
  std::vector<double> norm_defects;
  double max_right_defect = 0.0;
  double max_left_defect = 0.0;
  double max_translation_defect = 0.0;
  double max_norm_defect = 0.0;
  bool pass = false;
  double max_defect() const;
};

UniformMPS product_state_uniform(std::size_t d, std::size_t cell_length, const std::vector<cplx>& local_vector);
FiniteMPS product_state_finite(std::size_t d, std::size_t n_sites, const std::vector<cplx>& local_vector);
IsometryReport check_isometric(const UniformMPS& mps, double tol);
IsometryReport check_isometric(const FiniteMPS& mps, double tol);
cplx expectation_local(const UniformMPS& mps, const ComplexTensor& op, std::size_t site);
cplx expectation_local(const FiniteMPS& mps, const ComplexTensor& op, std::size_t site);
std::vector<double> schmidt_values(const UniformMPS& mps, std::size_t bond);
std::vector<double> schmidt_values(const FiniteMPS& mps, std::size_t bond);
double entropy_from_schmidt(const std::vector<double>& values);
double entanglement_entropy(const UniformMPS& mps, std::size_t bond);
double entanglement_entropy(const FiniteMPS& mps, std::size_t bond);
FiniteMPS move_center(FiniteMPS mps, std::size_t new_center);
void save_mps(const UniformMPS& mps, const std::string& path);
void save_mps(const FiniteMPS& mps, const std::string& path);
std::variant<UniformMPS, FiniteMPS> load_mps(const std::string& path);

// ---- TEBD: gates, policy, updates, steps -------------------------------------------
struct TwoSiteGate {
  ComplexTensor u;  // (i_out, j_out, i_in, j_in)
  std::size_t phys_dim() const { return u.dim(0); }
  ComplexTensor matrix() const;
};

TwoSiteGate make_gate(const ComplexTensor& h_bond, double dt);
TwoSiteGate identity_gate(std::size_t d);
TwoSiteGate gate_from_unitary(const ComplexTensor& u_matrix);

enum class Scheme { svd, eig, qr, qr_cbe };
std::string scheme_name(Scheme s);
Scheme scheme_from_name(const std::string& name);

struct TruncationPolicy {
  std::size_t chi_max = 1024;
  double sv_cutoff = 1e-14;
  double target_eps = 0.0;
  std::size_t delta_chi_abs = 100;
  double delta_chi_rel = 0.1;
  std::size_t chi_max_expansion = 0;
  int qr_sweeps = 1;
  bool compute_explicit_error = true;
  bool skip_renormalize = false;
  std::size_t expanded_dim(std::size_t chi, std::size_t d) const;
};

struct TruncationReport {
  std::size_t chi_before = 0;
  std::size_t chi_expanded = 0;
  std::size_t chi_after = 0;
  double eps_trunc = 0.0;
  double discarded_weight = 0.0;
  Scheme scheme = Scheme::svd;
};

struct GateUpdate {
  ComplexTensor b_m;                      // (d, chi_l, chi~)
  ComplexTensor xi_n;                     // chi~ x chi~
  ComplexTensor b_n;                      // (d, chi~, chi_r)
  std::optional<ComplexTensor> left_iso;  // (d, chi_l, chi~), QR only
  TruncationReport report;
};

GateUpdate apply_gate_svd(const ComplexTensor& xi, const ComplexTensor& b_m, const ComplexTensor& b_n,
                          const TwoSiteGate& u, const TruncationPolicy& policy);  // host comparator
GateUpdate apply_gate_eig(const ComplexTensor& xi, const ComplexTensor& b_m, const ComplexTensor& b_n,
                          const TwoSiteGate& u, const TruncationPolicy& policy);  // host comparator
GateUpdate apply_gate_qr(const ComplexTensor& xi, const ComplexTensor& b_m, const ComplexTensor& b_n,
                         const TwoSiteGate& u, const TruncationPolicy& policy);
GateUpdate apply_gate_qr_cbe(const ComplexTensor& xi, const ComplexTensor& b_m, const ComplexTensor& b_n,
                             const TwoSiteGate& u, const TruncationPolicy& policy);
GateUpdate apply_gate(Scheme scheme, const ComplexTensor& xi, const ComplexTensor& b_m, const ComplexTensor& b_n,
                      const TwoSiteGate& u, const TruncationPolicy& policy);
double truncation_error_explicit(const ComplexTensor& theta, const ComplexTensor& left_isometry,
                                 const ComplexTensor& center, const ComplexTensor& right_isometry);

enum class BondParity { even, odd };
std::vector<std::pair<BondParity, TwoSiteGate>> trotter_schedule(const ComplexTensor& h_bond, double dt, int order);

struct BondReport {
  std::size_t bond = 0;
  TruncationReport report;
};
struct UniformStepResult {
  UniformMPS state;
  std::vector<BondReport> reports;
};
using UniformGateObserver = std::function<void(const UniformMPS&, const BondReport&)>;
using FiniteGateObserver = std::function<void(const FiniteMPS&, const BondReport&)>;

UniformStepResult tebd_step(const UniformMPS& state, const std::vector<std::pair<BondParity, TwoSiteGate>>& schedule,
                            Scheme scheme, const TruncationPolicy& policy, const UniformGateObserver& on_gate = {});

struct FiniteLayer {
  BondParity parity;
  double dt = 0.0;
  std::vector<TwoSiteGate> gates;  // gates[m] acts on sites (m, m+1)
};
struct FiniteStepResult {
  FiniteMPS state;
  std::vector<BondReport> reports;
};
FiniteStepResult tebd_step(const FiniteMPS& state, const std::vector<FiniteLayer>& layers, Scheme scheme,
                           const TruncationPolicy& policy, const FiniteGateObserver& on_gate = {});

namespace detail_gates {
std::vector<std::pair<BondParity, double>> layer_structure(double dt, int order);
}

template <typename BondHamFn>
std::vector<FiniteLayer> finite_trotter_layers(BondHamFn&& h_of_bond, std::size_t n_sites, double dt, int order) {
  std::vector<FiniteLayer> layers;
  for (const auto& [parity, dt_eff] : detail_gates::layer_structure(dt, order)) {
    FiniteLayer layer{parity, dt_eff, {}};
    layer.gates.reserve(n_sites > 0 ? n_sites - 1 : 0);
    for (std::size_t m = 0; m + 1 < n_sites; ++m) layer.gates.push_back(make_gate(h_of_bond(m), dt_eff));
    layers.push_back(std::move(layer));
  }
  return layers;
}

// ---- B200 controls (not in the reference) ----------------------------------------
namespace b200 {
/// Device of the calling thread's default context (default 0; the
/// QRTEBD_DEVICE environment variable overrides the default).  Takes effect
/// for threads whose context does not exist yet.
void set_device(int device);
/// The calling thread's context (qt_ctx*, include/qrtebd_c.h), created on
/// first use.
void* context();
}  // namespace b200

}  // namespace qrtebd

#endif
