// qrtebd_b200.hpp -- C++ mirror of the reference API over the C-ABI.
//
// Drop-in shape of /root/reference/proj/include/qrtebd/{tensor,gates,mps,
// errors}.hpp for the QR-TEBD hot path: the same namespace, type and function
// names (ComplexTensor, TruncationPolicy, TruncationReport, GateUpdate,
// apply_gate_qr, apply_gate_qr_cbe, apply_gate, tebd_step, UniformMPS,
// expectation_local, schmidt_values, entanglement_entropy, exception types),
// implemented by calls into libqrtebd_b200.so (include/qrtebd_c.h).  Host
// ComplexTensors are copied to HBM per call (value semantics of the reference,
// SPEC.md:216); DeviceUniformMPS keeps a state resident across steps.
//
// Header-only; link with -lqrtebd_b200 (paper_2212_09782_b200/).
#ifndef QRTEBD_B200_HPP
#define QRTEBD_B200_HPP

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstddef>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../qrtebd_c.h"

namespace qrtebd {

using cplx = std::complex<double>;

// ---- errors (proj/include/qrtebd/errors.hpp:9-30) ---------------------------
class ShapeError : public std::invalid_argument {
 public:
  explicit ShapeError(const std::string& w) : std::invalid_argument(w) {}
};
class InputError : public std::invalid_argument {
 public:
  explicit InputError(const std::string& w) : std::invalid_argument(w) {}
};
class NumericError : public std::runtime_error {
 public:
  explicit NumericError(const std::string& w) : std::runtime_error(w) {}
};
class CapacityError : public std::runtime_error {
 public:
  explicit CapacityError(const std::string& w) : std::runtime_error(w) {}
};
class DeviceError : public std::runtime_error {
 public:
  explicit DeviceError(const std::string& w) : std::runtime_error(w) {}
};

inline void check(qt_status s) {
  if (s == QT_OK) return;
  const std::string msg = qt_last_error();
  switch (s) {
    case QT_ERR_SHAPE: throw ShapeError(msg);
    case QT_ERR_INPUT: throw InputError(msg);
    case QT_ERR_NUMERIC: throw NumericError(msg);
    case QT_ERR_CAPACITY: throw CapacityError(msg);
    default: throw DeviceError(msg);
  }
}

// ---- host tensor (proj/include/qrtebd/tensor.hpp:18-61, row-major) -----------
class ComplexTensor {
 public:
  ComplexTensor() = default;
  explicit ComplexTensor(std::vector<std::size_t> shape) : shape_(std::move(shape)), data_(numel(shape_)) {}
  ComplexTensor(std::vector<std::size_t> shape, std::vector<cplx> data) : shape_(std::move(shape)), data_(std::move(data)) {
    if (data_.size() != numel(shape_)) throw ShapeError("data size does not match shape");
  }
  static ComplexTensor identity(std::size_t n) {
    ComplexTensor t({n, n});
    for (std::size_t i = 0; i < n; ++i) t.data_[i * n + i] = 1.0;
    return t;
  }
  std::size_t rank() const { return shape_.size(); }
  const std::vector<std::size_t>& shape() const { return shape_; }
  std::size_t dim(std::size_t a) const { return shape_.at(a); }
  std::size_t size() const { return data_.size(); }
  std::vector<cplx>& data() { return data_; }
  const std::vector<cplx>& data() const { return data_; }
  double norm() const {
    double s = 0;
    for (const cplx& v : data_) s += std::norm(v);
    return std::sqrt(s);
  }

 private:
  static std::size_t numel(const std::vector<std::size_t>& s) {
    std::size_t n = 1;
    for (std::size_t x : s) n *= x;
    return n;
  }
  std::vector<std::size_t> shape_;
  std::vector<cplx> data_;
};

// ---- device context + tensor handles --------------------------------------------
class Context {
 public:
  explicit Context(int device = 0) { check(qt_ctx_create(device, nullptr, &h_)); }
  ~Context() {
    if (h_) qt_ctx_destroy(h_);
  }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  qt_ctx* get() const { return h_; }

 private:
  qt_ctx* h_ = nullptr;
};

class DeviceTensor {
 public:
  DeviceTensor() = default;
  explicit DeviceTensor(qt_tensor* h) : h_(h, qt_tensor_free) {}
  DeviceTensor(Context& ctx, const ComplexTensor& t) {
    std::vector<uint64_t> shp(t.shape().begin(), t.shape().end());
    qt_tensor* h = nullptr;
    check(qt_tensor_create(ctx.get(), static_cast<int>(shp.size()), shp.data(), &h));
    h_.reset(h, qt_tensor_free);
    check(qt_tensor_upload(h, reinterpret_cast<const double*>(t.data().data())));
  }
  qt_tensor* get() const { return h_.get(); }
  explicit operator bool() const { return static_cast<bool>(h_); }
  ComplexTensor host() const {
    int rank = 0;
    uint64_t s4[4];
    check(qt_tensor_shape(h_.get(), &rank, s4));
    ComplexTensor t(std::vector<std::size_t>(s4, s4 + rank));
    check(qt_tensor_download(h_.get(), reinterpret_cast<double*>(t.data().data())));
    return t;
  }

 private:
  std::shared_ptr<qt_tensor> h_;
};

// ---- policy / report / update (proj/include/qrtebd/gates.hpp:17-76) ------------
struct TwoSiteGate {
  ComplexTensor u;  // (i_out, j_out, i_in, j_in)
  std::size_t phys_dim() const { return u.dim(0); }
};

enum class Scheme { svd, eig, qr, qr_cbe };

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

  qt_policy c() const {
    qt_policy p;
    qt_policy_default(&p);
    p.chi_max = chi_max;
    p.sv_cutoff = sv_cutoff;
    p.target_eps = target_eps;
    p.delta_chi_abs = delta_chi_abs;
    p.delta_chi_rel = delta_chi_rel;
    p.chi_max_expansion = chi_max_expansion;
    p.qr_sweeps = qr_sweeps;
    p.compute_explicit_error = compute_explicit_error ? 1 : 0;
    p.skip_renormalize = skip_renormalize ? 1 : 0;
    return p;
  }
  std::size_t expanded_dim(std::size_t chi, std::size_t d) const {
    const qt_policy p = c();
    return static_cast<std::size_t>(qt_expanded_dim(&p, chi, d));
  }
};

struct TruncationReport {
  std::size_t chi_before = 0, chi_expanded = 0, chi_after = 0;
  double eps_trunc = 0.0, discarded_weight = 0.0;
  Scheme scheme = Scheme::qr;
};

inline TruncationReport from_c(const qt_report& r) {
  TruncationReport t;
  t.chi_before = r.chi_before;
  t.chi_expanded = r.chi_expanded;
  t.chi_after = r.chi_after;
  t.eps_trunc = r.eps_trunc;
  t.discarded_weight = r.discarded_weight;
  t.scheme = static_cast<Scheme>(r.scheme);
  return t;
}

struct GateUpdate {
  ComplexTensor b_m;
  ComplexTensor xi_n;
  ComplexTensor b_n;
  std::optional<ComplexTensor> left_iso;
  TruncationReport report;
};

// apply_gate_qr, proj/src/gates.cpp:343-386 (host tensors in, host tensors out)
inline GateUpdate apply_gate_qr(Context& ctx, const ComplexTensor& xi, const ComplexTensor& b_m,
                                const ComplexTensor& b_n, const TwoSiteGate& u, const TruncationPolicy& policy) {
  DeviceTensor dxi(ctx, xi), dbm(ctx, b_m), dbn(ctx, b_n), du(ctx, u.u);
  const qt_policy p = policy.c();
  qt_tensor *obm = nullptr, *oxi = nullptr, *obn = nullptr, *oli = nullptr;
  qt_report rep;
  check(qt_apply_gate_qr(ctx.get(), dxi.get(), dbm.get(), dbn.get(), du.get(), &p, &obm, &oxi, &obn, &oli, &rep));
  DeviceTensor tbm(obm), txi(oxi), tbn(obn), tli(oli);
  return GateUpdate{tbm.host(), txi.host(), tbn.host(), tli.host(), from_c(rep)};
}

// apply_gate_qr_cbe, proj/src/gates.cpp:388-450
inline GateUpdate apply_gate_qr_cbe(Context& ctx, const ComplexTensor& xi, const ComplexTensor& b_m,
                                    const ComplexTensor& b_n, const TwoSiteGate& u, const TruncationPolicy& policy) {
  DeviceTensor dxi(ctx, xi), dbm(ctx, b_m), dbn(ctx, b_n), du(ctx, u.u);
  const qt_policy p = policy.c();
  qt_tensor *obm = nullptr, *oxi = nullptr, *obn = nullptr;
  qt_report rep;
  check(qt_apply_gate_qr_cbe(ctx.get(), dxi.get(), dbm.get(), dbn.get(), du.get(), &p, &obm, &oxi, &obn, &rep));
  DeviceTensor tbm(obm), txi(oxi), tbn(obn);
  return GateUpdate{tbm.host(), txi.host(), tbn.host(), std::nullopt, from_c(rep)};
}

// apply_gate, proj/src/gates.cpp:452-462 (device schemes)
inline GateUpdate apply_gate(Context& ctx, Scheme scheme, const ComplexTensor& xi, const ComplexTensor& b_m,
                             const ComplexTensor& b_n, const TwoSiteGate& u, const TruncationPolicy& policy) {
  if (scheme == Scheme::qr) return apply_gate_qr(ctx, xi, b_m, b_n, u, policy);
  if (scheme == Scheme::qr_cbe) return apply_gate_qr_cbe(ctx, xi, b_m, b_n, u, policy);
  throw InputError("svd/eig are CPU comparators of the reference, not device schemes");
}

// ---- uniform MPS + tebd_step (proj/include/qrtebd/mps.hpp:18-26, gates.cpp:513-540)
struct UniformMPS {
  std::size_t phys_dim = 0;
  std::vector<ComplexTensor> site_tensors;
  std::vector<ComplexTensor> bond_matrices;
  std::size_t cell_length() const { return site_tensors.size(); }
};

enum class BondParity { even, odd };

struct BondReport {
  std::size_t bond = 0;
  TruncationReport report;
};

struct UniformStepResult {
  UniformMPS state;
  std::vector<BondReport> reports;
};

inline UniformStepResult tebd_step(Context& ctx, const UniformMPS& state,
                                   const std::vector<std::pair<BondParity, TwoSiteGate>>& schedule, Scheme scheme,
                                   const TruncationPolicy& policy) {
  const std::size_t L = state.cell_length();
  std::vector<DeviceTensor> s, b, g;
  for (std::size_t m = 0; m < L; ++m) {
    s.emplace_back(ctx, state.site_tensors[m]);
    b.emplace_back(ctx, state.bond_matrices[m]);
  }
  std::vector<int32_t> par;
  for (const auto& [p, gate] : schedule) {
    g.emplace_back(ctx, gate.u);
    par.push_back(p == BondParity::even ? 0 : 1);
  }
  std::vector<qt_tensor*> sh(L), bh(L), gh(g.size()), so(L), bo(L);
  for (std::size_t m = 0; m < L; ++m) {
    sh[m] = s[m].get();
    bh[m] = b[m].get();
  }
  for (std::size_t k = 0; k < g.size(); ++k) gh[k] = g[k].get();
  std::vector<qt_bond_report> reps(schedule.size() * (L / 2 + 1));
  uint64_t n = reps.size();
  const qt_policy p = policy.c();
  check(qt_tebd_step_uniform(ctx.get(), L, sh.data(), bh.data(), schedule.size(), par.data(), gh.data(),
                             scheme == Scheme::qr ? QT_SCHEME_QR : (scheme == Scheme::qr_cbe ? QT_SCHEME_QR_CBE
                                                                                             : QT_SCHEME_SVD),
                             &p, so.data(), bo.data(), reps.data(), &n));
  UniformStepResult out;
  out.state.phys_dim = state.phys_dim;
  for (std::size_t m = 0; m < L; ++m) {
    out.state.site_tensors.push_back(DeviceTensor(so[m]).host());
    out.state.bond_matrices.push_back(DeviceTensor(bo[m]).host());
  }
  for (uint64_t i = 0; i < n; ++i) out.reports.push_back({reps[i].bond, from_c(reps[i].report)});
  return out;
}

// ---- observables (proj/src/mps.cpp) ----------------------------------------------
inline cplx expectation_local(Context& ctx, const UniformMPS& mps, const ComplexTensor& op, std::size_t site) {
  if (site >= mps.cell_length()) throw InputError("site out of range");
  DeviceTensor xi(ctx, mps.bond_matrices[site]), b(ctx, mps.site_tensors[site]), o(ctx, op);
  double out[2];
  check(qt_expectation_local(ctx.get(), xi.get(), b.get(), o.get(), out));
  return {out[0], out[1]};
}

inline std::vector<double> schmidt_values(Context& ctx, const UniformMPS& mps, std::size_t bond) {
  if (bond >= mps.cell_length()) throw InputError("bond out of range");
  DeviceTensor xi(ctx, mps.bond_matrices[bond]);
  std::vector<double> s(std::min(mps.bond_matrices[bond].dim(0), mps.bond_matrices[bond].dim(1)));
  uint64_t n = s.size();
  check(qt_schmidt_values(ctx.get(), xi.get(), s.data(), &n));
  s.resize(n);
  return s;
}

inline double entropy_from_schmidt(const std::vector<double>& values) {
  double s = 0;
  for (double v : values) {
    const double p = v * v;
    if (p > 0.0) s -= p * std::log(p);
  }
  return s;
}

inline double entanglement_entropy(Context& ctx, const UniformMPS& mps, std::size_t bond) {
  return entropy_from_schmidt(schmidt_values(ctx, mps, bond));
}

// proj/include/qrtebd/mps.hpp:40-53
struct IsometryReport {
  std::vector<double> right_defects, left_defects, translation_defects, norm_defects;
  double max_right_defect = 0.0, max_left_defect = 0.0, max_translation_defect = 0.0, max_norm_defect = 0.0;
  bool pass = false;
  double max_defect() const {
    return std::max(std::max(max_right_defect, max_left_defect), std::max(max_translation_defect, max_norm_defect));
  }
};

// check_isometric(UniformMPS, tol), proj/src/mps.cpp:105-141
inline IsometryReport check_isometric(Context& ctx, const UniformMPS& mps, double tol) {
  const std::size_t L = mps.cell_length();
  std::vector<DeviceTensor> s, b;
  std::vector<qt_tensor*> sh(L), bh(L);
  for (std::size_t m = 0; m < L; ++m) {
    s.emplace_back(ctx, mps.site_tensors[m]);
    b.emplace_back(ctx, mps.bond_matrices[m]);
  }
  for (std::size_t m = 0; m < L; ++m) {
    sh[m] = s[m].get();
    bh[m] = b[m].get();
  }
  IsometryReport r;
  r.right_defects.resize(L);
  r.left_defects.resize(L);
  r.translation_defects.resize(L);
  r.norm_defects.resize(L);
  qt_isometry_report c{};
  check(qt_check_isometric_uniform(ctx.get(), L, sh.data(), bh.data(), tol, r.right_defects.data(),
                                   r.left_defects.data(), r.translation_defects.data(), r.norm_defects.data(), &c));
  r.max_right_defect = c.max_right_defect;
  r.max_left_defect = c.max_left_defect;
  r.max_translation_defect = c.max_translation_defect;
  r.max_norm_defect = c.max_norm_defect;
  r.pass = c.pass != 0;
  return r;
}

// ---- FiniteMPS (proj/include/qrtebd/mps.hpp:31-38) with reference semantics -------
struct FiniteMPS {
  std::size_t phys_dim = 0;
  std::vector<ComplexTensor> site_tensors;
  std::size_t center_bond = 0;
  ComplexTensor center_matrix;
  std::size_t length() const { return site_tensors.size(); }
};

/// One FiniteLayer (proj/include/qrtebd/gates.hpp:130-137).
struct FiniteLayer {
  BondParity parity = BondParity::even;
  double dt = 0.0;
  std::vector<TwoSiteGate> gates;  // one per bond, indexed by left site
};

struct FiniteStepResult {
  FiniteMPS state;
  std::vector<BondReport> reports;
};

namespace detail {
// RAII handle of a device-resident chain (qt_finite)
class DeviceFinite {
 public:
  DeviceFinite(Context& ctx, const FiniteMPS& s) {
    std::vector<DeviceTensor> sites;
    std::vector<qt_tensor*> sh;
    for (const ComplexTensor& t : s.site_tensors) {
      sites.emplace_back(ctx, t);
      sh.push_back(sites.back().get());
    }
    DeviceTensor c(ctx, s.center_matrix);
    check(qt_finite_create(ctx.get(), sh.size(), sh.data(), s.center_bond, c.get(), &h_));
  }
  ~DeviceFinite() {
    if (h_) qt_finite_destroy(h_);
  }
  DeviceFinite(const DeviceFinite&) = delete;
  DeviceFinite& operator=(const DeviceFinite&) = delete;
  qt_finite* get() const { return h_; }
  FiniteMPS host(std::size_t d, std::size_t n) const {
    FiniteMPS out;
    out.phys_dim = d;
    uint64_t c = 0;
    check(qt_finite_center_bond(h_, &c));
    out.center_bond = c;
    for (std::size_t m = 0; m < n; ++m) {
      qt_tensor* v = nullptr;
      check(qt_finite_view(h_, 0, m, &v));
      out.site_tensors.push_back(DeviceTensor(v).host());
    }
    qt_tensor* v = nullptr;
    check(qt_finite_view(h_, 1, 0, &v));
    out.center_matrix = DeviceTensor(v).host();
    return out;
  }

 private:
  qt_finite* h_ = nullptr;
};
}  // namespace detail

/// move_center, proj/src/mps.cpp:226-257 (value semantics, device QR/LQ)
inline FiniteMPS move_center(Context& ctx, const FiniteMPS& mps, std::size_t new_center) {
  detail::DeviceFinite f(ctx, mps);
  check(qt_finite_move_center(f.get(), new_center));
  return f.host(mps.phys_dim, mps.length());
}

/// tebd_step(FiniteMPS), proj/src/gates.cpp:542-578
inline FiniteStepResult tebd_step(Context& ctx, const FiniteMPS& state, const std::vector<FiniteLayer>& layers,
                                  Scheme scheme, const TruncationPolicy& policy) {
  const std::size_t n = state.length();
  detail::DeviceFinite f(ctx, state);
  std::vector<DeviceTensor> g;
  std::vector<qt_tensor*> gh;
  std::vector<int32_t> par;
  for (const FiniteLayer& l : layers) {
    if (l.gates.size() + 1 != n) throw ShapeError("layer gate count must equal the bond count");
    par.push_back(l.parity == BondParity::even ? 0 : 1);
    for (const TwoSiteGate& u : l.gates) {
      g.emplace_back(ctx, u.u);
      gh.push_back(g.back().get());
    }
  }
  std::vector<qt_bond_report> reps(layers.size() * (n / 2 + 1) + 1);
  uint64_t cnt = reps.size();
  const qt_policy p = policy.c();
  check(qt_finite_step(f.get(), layers.size(), par.data(), gh.data(),
                       scheme == Scheme::qr ? QT_SCHEME_QR : (scheme == Scheme::qr_cbe ? QT_SCHEME_QR_CBE
                                                                                       : QT_SCHEME_SVD),
                       &p, reps.data(), &cnt));
  FiniteStepResult out;
  out.state = f.host(state.phys_dim, n);
  for (uint64_t i = 0; i < cnt; ++i) out.reports.push_back({reps[i].bond, from_c(reps[i].report)});
  return out;
}

/// expectation_local(FiniteMPS), proj/src/mps.cpp:188-196
inline cplx expectation_local(Context& ctx, const FiniteMPS& mps, const ComplexTensor& op, std::size_t site) {
  if (site >= mps.length()) throw InputError("site out of range");
  const FiniteMPS c = move_center(ctx, mps, site);
  DeviceTensor xi(ctx, c.center_matrix), b(ctx, c.site_tensors[site]), o(ctx, op);
  double out[2];
  check(qt_expectation_local(ctx.get(), xi.get(), b.get(), o.get(), out));
  return {out[0], out[1]};
}

/// schmidt_values(FiniteMPS), proj/src/mps.cpp:203-207
inline std::vector<double> schmidt_values(Context& ctx, const FiniteMPS& mps, std::size_t bond) {
  if (bond > mps.length()) throw InputError("bond out of range");
  const FiniteMPS c = move_center(ctx, mps, bond);
  DeviceTensor xi(ctx, c.center_matrix);
  std::vector<double> s(std::min(c.center_matrix.dim(0), c.center_matrix.dim(1)));
  uint64_t cnt = s.size();
  check(qt_schmidt_values(ctx.get(), xi.get(), s.data(), &cnt));
  s.resize(cnt);
  return s;
}

}  // namespace qrtebd

#endif
