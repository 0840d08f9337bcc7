// qrtebd_api.cpp -- the reference's C++ API (include/qrtebd/qrtebd_api.hpp)
// implemented on the B200 through the C-ABI (include/qrtebd_c.h).
//
// Value semantics as in the reference: host ComplexTensors are
// uploaded per call, the update runs on the device, results are downloaded.
// Each host thread gets its own device context (stream + workspace), so the
// functions are safe to call concurrently like the reference's (the
// reference's bench pool calls apply_gate from several threads,
// proj/src/run.cpp:440-463).  All arithmetic of the hot path runs in the
// sm_100a kernels of libqrtebd_b200.so; this file only moves data, checks
// shapes and maps status codes onto the reference's exception types
// (proj/include/qrtebd/errors.hpp:9-30).
//
// The svd/eig schemes, the clock model, gate construction, product states
// and checkpoint I/O are the reference library's host code: they are weak
// references here and resolve to the reference's libqrtebd when it is linked
// after this library.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <memory>
#include <numeric>
#include <sstream>

#include "qrtebd/qrtebd_api.hpp"
#include "qrtebd_c.h"

namespace qrtebd {

// host comparators of the reference library (proj/src/gates.cpp:312-341)
GateUpdate apply_gate_svd(const ComplexTensor&, const ComplexTensor&, const ComplexTensor&, const TwoSiteGate&,
                          const TruncationPolicy&) __attribute__((weak));
GateUpdate apply_gate_eig(const ComplexTensor&, const ComplexTensor&, const ComplexTensor&, const TwoSiteGate&,
                          const TruncationPolicy&) __attribute__((weak));

namespace {

// ---------------------------------------------------------------- context
int g_device = -1;

struct ThreadCtx {
  qt_ctx* h = nullptr;
  ~ThreadCtx() {
    if (h) qt_ctx_destroy(h);
  }
};
thread_local ThreadCtx t_ctx;

[[noreturn]] void raise(qt_status s) {
  const std::string msg = qt_last_error();
  switch (s) {
    case QT_ERR_SHAPE: throw ShapeError(msg);
    case QT_ERR_INPUT: throw InputError(msg);
    case QT_ERR_NUMERIC: throw NumericError(msg);
    case QT_ERR_CAPACITY: throw CapacityError(msg);
    default: throw std::runtime_error("qrtebd device error: " + msg);
  }
}
inline void check(qt_status s) {
  if (s != QT_OK) raise(s);
}

qt_ctx* ctx() {
  if (!t_ctx.h) {
    int dev = g_device;
    if (dev < 0) {
      const char* e = std::getenv("QRTEBD_DEVICE");
      dev = e ? std::atoi(e) : 0;
    }
    check(qt_ctx_create(dev, nullptr, &t_ctx.h));
  }
  return t_ctx.h;
}

// ---------------------------------------------------------------- device tensors
struct Dev {
  qt_tensor* h = nullptr;
  Dev() = default;
  explicit Dev(qt_tensor* t) : h(t) {}
  explicit Dev(const ComplexTensor& t) {
    if (t.rank() == 0 || t.rank() > 4) throw ShapeError("device tensors have rank 1..4");
    std::vector<uint64_t> shp(t.shape().begin(), t.shape().end());
    check(qt_tensor_create(ctx(), static_cast<int>(shp.size()), shp.data(), &h));
    check(qt_tensor_upload(h, reinterpret_cast<const double*>(t.data().data())));
  }
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
  Dev(Dev&& o) noexcept : h(o.h) { o.h = nullptr; }
  Dev& operator=(Dev&& o) noexcept {
    std::swap(h, o.h);
    return *this;
  }
  ~Dev() {
    if (h) qt_tensor_free(h);
  }
  ComplexTensor host() const {
    int rank = 0;
    uint64_t s4[4];
    check(qt_tensor_shape(h, &rank, s4));
    ComplexTensor t(std::vector<std::size_t>(s4, s4 + rank));
    check(qt_tensor_download(h, reinterpret_cast<double*>(t.data().data())));
    return t;
  }
};

qt_policy c_policy(const TruncationPolicy& p) {
  qt_policy c;
  qt_policy_default(&c);
  c.chi_max = p.chi_max;
  c.sv_cutoff = p.sv_cutoff;
  c.target_eps = p.target_eps;
  c.delta_chi_abs = p.delta_chi_abs;
  c.delta_chi_rel = p.delta_chi_rel;
  c.chi_max_expansion = p.chi_max_expansion;
  c.qr_sweeps = p.qr_sweeps;
  c.compute_explicit_error = p.compute_explicit_error ? 1 : 0;
  c.skip_renormalize = p.skip_renormalize ? 1 : 0;
  return c;
}

TruncationReport from_c(const qt_report& r) {
  TruncationReport t;
  t.chi_before = r.chi_before;
  t.chi_expanded = r.chi_expanded;
  t.chi_after = r.chi_after;
  t.eps_trunc = r.eps_trunc;
  t.discarded_weight = r.discarded_weight;
  t.scheme = static_cast<Scheme>(r.scheme);
  return t;
}

qt_scheme c_scheme(Scheme s) {
  switch (s) {
    case Scheme::qr: return QT_SCHEME_QR;
    case Scheme::qr_cbe: return QT_SCHEME_QR_CBE;
    case Scheme::eig: return QT_SCHEME_EIG;
    default: return QT_SCHEME_SVD;
  }
}

bool device_scheme(Scheme s) { return s == Scheme::qr || s == Scheme::qr_cbe; }

std::size_t shape_product(const std::vector<std::size_t>& shape) {
  std::size_t n = 1;
  for (std::size_t s : shape) n *= s;
  return n;
}

std::string shape_str(const std::vector<std::size_t>& shape) {
  std::ostringstream os;
  os << "(";
  for (std::size_t i = 0; i < shape.size(); ++i) os << (i ? "," : "") << shape[i];
  os << ")";
  return os.str();
}

// one device update on device handles (the kernels qt_tebd_step_uniform runs)
struct DevUpdate {
  Dev b_m, xi, b_n, left;
  TruncationReport report;
};
DevUpdate device_update(Scheme scheme, const Dev& xi, const Dev& bm, const Dev& bn, const Dev& u,
                        const TruncationPolicy& policy, bool want_left) {
  const qt_policy p = c_policy(policy);
  qt_tensor *obm = nullptr, *oxi = nullptr, *obn = nullptr, *oli = nullptr;
  qt_report rep{};
  check(qt_apply_gate(ctx(), c_scheme(scheme), xi.h, bm.h, bn.h, u.h, &p, &obm, &oxi, &obn,
                      want_left && scheme == Scheme::qr ? &oli : nullptr, &rep));
  DevUpdate out;
  out.b_m = Dev(obm);
  out.xi = Dev(oxi);
  out.b_n = Dev(obn);
  out.left = Dev(oli);
  out.report = from_c(rep);
  return out;
}

GateUpdate host_comparator(Scheme scheme, const ComplexTensor& xi, const ComplexTensor& b_m,
                           const ComplexTensor& b_n, const TwoSiteGate& u, const TruncationPolicy& policy) {
  auto fn = scheme == Scheme::svd ? &apply_gate_svd : &apply_gate_eig;
  if (fn == nullptr)
    throw InputError("scheme " + std::string(scheme == Scheme::svd ? "svd" : "eig") +
                     " is a host comparator of the reference library, which is not linked");
  return fn(xi, b_m, b_n, u, policy);
}

}  // namespace

namespace b200 {
void set_device(int device) { g_device = device; }
void* context() { return ctx(); }
}  // namespace b200

// ================================================================ tensor layer
// proj/src/tensor.cpp semantics: zero-length axes and size mismatches are
// ShapeErrors; transposes and reshapes are host data movement.
ComplexTensor::ComplexTensor(std::vector<std::size_t> shape) : shape_(std::move(shape)), data_(shape_product(shape_)) {
  for (std::size_t s : shape_)
    if (s == 0) throw ShapeError("tensor axis of dimension 0");
}

ComplexTensor::ComplexTensor(std::vector<std::size_t> shape, std::vector<cplx> data)
    : shape_(std::move(shape)), data_(std::move(data)) {
  for (std::size_t s : shape_)
    if (s == 0) throw ShapeError("tensor axis of dimension 0");
  if (shape_product(shape_) != data_.size())
    throw ShapeError("tensor data length does not match shape " + shape_str(shape_));
}

ComplexTensor ComplexTensor::zeros(std::vector<std::size_t> shape) { return ComplexTensor(std::move(shape)); }

ComplexTensor ComplexTensor::identity(std::size_t n) {
  ComplexTensor t({n, n});
  for (std::size_t i = 0; i < n; ++i) t.data_[i * n + i] = 1.0;
  return t;
}

ComplexTensor ComplexTensor::matrix(std::size_t rows, std::size_t cols, std::vector<cplx> data) {
  return ComplexTensor({rows, cols}, std::move(data));
}

std::size_t ComplexTensor::dim(std::size_t axis) const {
  if (axis >= shape_.size()) throw ShapeError("axis out of range");
  return shape_[axis];
}

const cplx& ComplexTensor::at(std::initializer_list<std::size_t> idx) const {
  if (idx.size() != shape_.size()) throw ShapeError("index rank mismatch for shape " + shape_str(shape_));
  std::size_t lin = 0, k = 0;
  for (std::size_t i : idx) {
    if (i >= shape_[k]) throw ShapeError("index out of range");
    lin = lin * shape_[k++] + i;
  }
  return data_[lin];
}

cplx& ComplexTensor::at(std::initializer_list<std::size_t> idx) {
  return const_cast<cplx&>(static_cast<const ComplexTensor&>(*this).at(idx));
}

ComplexTensor ComplexTensor::reshape(std::vector<std::size_t> new_shape) const& {
  if (shape_product(new_shape) != data_.size())
    throw ShapeError("reshape " + shape_str(shape_) + " -> " + shape_str(new_shape) + " changes size");
  return ComplexTensor(std::move(new_shape), data_);
}

ComplexTensor ComplexTensor::reshape(std::vector<std::size_t> new_shape) && {
  if (shape_product(new_shape) != data_.size())
    throw ShapeError("reshape " + shape_str(shape_) + " -> " + shape_str(new_shape) + " changes size");
  return ComplexTensor(std::move(new_shape), std::move(data_));
}

ComplexTensor ComplexTensor::transpose(const std::vector<std::size_t>& perm) const {
  const std::size_t r = rank();
  if (perm.size() != r) throw ShapeError("permutation rank mismatch");
  std::vector<char> seen(r, 0);
  for (std::size_t p : perm) {
    if (p >= r || seen[p]) throw ShapeError("invalid axis permutation");
    seen[p] = 1;
  }
  std::vector<std::size_t> out_shape(r), src_stride(r), in_stride(r, 1);
  for (std::size_t k = r; k-- > 1;) in_stride[k - 1] = in_stride[k] * shape_[k];
  for (std::size_t k = 0; k < r; ++k) {
    out_shape[k] = shape_[perm[k]];
    src_stride[k] = in_stride[perm[k]];
  }
  ComplexTensor out(out_shape);
  if (r == 0) {
    out.data_ = data_;
    return out;
  }
  // odometer over the output index; the innermost output axis is a strided
  // gather from the input
  const std::size_t inner = out_shape[r - 1], inner_stride = src_stride[r - 1];
  std::vector<std::size_t> idx(r, 0);
  std::size_t src = 0;
  for (std::size_t dst = 0; dst < data_.size(); dst += inner) {
    for (std::size_t j = 0; j < inner; ++j) out.data_[dst + j] = data_[src + j * inner_stride];
    for (std::size_t k = r - 1; k-- > 0;) {
      src += src_stride[k];
      if (++idx[k] < out_shape[k]) break;
      src -= src_stride[k] * out_shape[k];
      idx[k] = 0;
    }
  }
  return out;
}

ComplexTensor ComplexTensor::conj() const {
  ComplexTensor out(shape_, data_);
  for (cplx& v : out.data_) v = std::conj(v);
  return out;
}

double ComplexTensor::norm() const {
  double s = 0;
  for (const cplx& v : data_) s += std::norm(v);
  return std::sqrt(s);
}

bool ComplexTensor::all_finite() const {
  return std::all_of(data_.begin(), data_.end(),
                     [](const cplx& v) { return std::isfinite(v.real()) && std::isfinite(v.imag()); });
}

ComplexTensor& ComplexTensor::operator*=(cplx factor) {
  for (cplx& v : data_) v *= factor;
  return *this;
}

// contract (proj/src/tensor.cpp:172-233): the free axes of a, then of b; the
// contraction itself is one device GEMM (qt_zgemm, DMMA)
ComplexTensor contract(const ComplexTensor& a, const ComplexTensor& b,
                       const std::vector<std::pair<std::size_t, std::size_t>>& axes) {
  const std::size_t ra = a.rank(), rb = b.rank();
  std::vector<char> ca(ra, 0), cb(rb, 0);
  std::size_t kdim = 1;
  for (const auto& [ia, ib] : axes) {
    if (ia >= ra || ib >= rb) throw ShapeError("contraction axis out of range");
    if (ca[ia] || cb[ib]) throw ShapeError("axis contracted twice");
    if (a.dim(ia) != b.dim(ib)) throw ShapeError("contracted axes have unequal dimensions");
    ca[ia] = cb[ib] = 1;
    kdim *= a.dim(ia);
  }
  std::vector<std::size_t> pa, pb, out_shape;
  for (std::size_t k = 0; k < ra; ++k)
    if (!ca[k]) {
      pa.push_back(k);
      out_shape.push_back(a.dim(k));
    }
  for (const auto& [ia, ib] : axes) {
    pa.push_back(ia);
    pb.push_back(ib);
  }
  for (std::size_t k = 0; k < rb; ++k)
    if (!cb[k]) {
      pb.push_back(k);
      out_shape.push_back(b.dim(k));
    }
  auto identity_perm = [](const std::vector<std::size_t>& p) {
    for (std::size_t k = 0; k < p.size(); ++k)
      if (p[k] != k) return false;
    return true;
  };
  const ComplexTensor at = identity_perm(pa) ? a : a.transpose(pa);
  const ComplexTensor bt = identity_perm(pb) ? b : b.transpose(pb);
  const std::size_t m = a.size() / kdim, n = b.size() / kdim;
  ComplexTensor out(out_shape);
  const Dev da(at.reshape({m, kdim})), db(bt.reshape({kdim, n}));
  const uint64_t cs[2] = {m, n};
  Dev dc;
  check(qt_tensor_create(ctx(), 2, cs, &dc.h));
  check(qt_zgemm(ctx(), 0, 0, static_cast<int64_t>(m), static_cast<int64_t>(n), static_cast<int64_t>(kdim), 1,
                 qt_tensor_data(da.h), static_cast<int64_t>(kdim), 0, qt_tensor_data(db.h), static_cast<int64_t>(n), 0,
                 qt_tensor_data(dc.h), static_cast<int64_t>(n), 0, 1.0, 0.0));
  check(qt_tensor_download(dc.h, reinterpret_cast<double*>(out.data().data())));
  return out;
}

// ================================================================ linalg (device)
QrResult qr_reduced(const ComplexTensor& m) {
  if (m.rank() != 2) throw ShapeError("qr_reduced: expected a matrix");
  const Dev dm(m);
  qt_tensor *q = nullptr, *r = nullptr;
  check(qt_qr_reduced(ctx(), dm.h, &q, &r));
  const Dev dq(q), dr(r);
  return {dq.host(), dr.host()};
}

LqResult lq_reduced(const ComplexTensor& m) {
  if (m.rank() != 2) throw ShapeError("lq_reduced: expected a matrix");
  const Dev dm(m);
  qt_tensor *l = nullptr, *q = nullptr;
  check(qt_lq_reduced(ctx(), dm.h, &l, &q));
  const Dev dl(l), dq(q);
  return {dl.host(), dq.host()};
}

EighResult eigh(const ComplexTensor& h) {
  if (h.rank() != 2) throw ShapeError("eigh: expected a matrix");
  if (!h.all_finite()) throw InputError("eigh: non-finite entries");
  if (h.dim(0) != h.dim(1)) throw ShapeError("eigh: matrix not square");
  const Dev dh(h);
  EighResult out;
  out.w.resize(h.dim(0));
  qt_tensor* v = nullptr;
  check(qt_eigh(ctx(), dh.h, out.w.data(), &v));
  out.v = Dev(v).host();
  return out;
}

// ================================================================ gates
std::size_t TruncationPolicy::expanded_dim(std::size_t chi, std::size_t d) const {
  const qt_policy p = c_policy(*this);
  return static_cast<std::size_t>(qt_expanded_dim(&p, chi, d));
}

GateUpdate apply_gate_qr(const ComplexTensor& xi, const ComplexTensor& b_m, const ComplexTensor& b_n,
                         const TwoSiteGate& u, const TruncationPolicy& policy) {
  const Dev dxi(xi), dbm(b_m), dbn(b_n), du(u.u);
  DevUpdate r = device_update(Scheme::qr, dxi, dbm, dbn, du, policy, true);
  return GateUpdate{r.b_m.host(), r.xi.host(), r.b_n.host(), r.left.host(), r.report};
}

GateUpdate apply_gate_qr_cbe(const ComplexTensor& xi, const ComplexTensor& b_m, const ComplexTensor& b_n,
                             const TwoSiteGate& u, const TruncationPolicy& policy) {
  const Dev dxi(xi), dbm(b_m), dbn(b_n), du(u.u);
  DevUpdate r = device_update(Scheme::qr_cbe, dxi, dbm, dbn, du, policy, false);
  return GateUpdate{r.b_m.host(), r.xi.host(), r.b_n.host(), std::nullopt, r.report};
}

GateUpdate apply_gate(Scheme scheme, const ComplexTensor& xi, const ComplexTensor& b_m, const ComplexTensor& b_n,
                      const TwoSiteGate& u, const TruncationPolicy& policy) {
  switch (scheme) {
    case Scheme::qr: return apply_gate_qr(xi, b_m, b_n, u, policy);
    case Scheme::qr_cbe: return apply_gate_qr_cbe(xi, b_m, b_n, u, policy);
    case Scheme::svd:
    case Scheme::eig: return host_comparator(scheme, xi, b_m, b_n, u, policy);
  }
  throw InputError("unknown scheme");
}

double truncation_error_explicit(const ComplexTensor& theta, const ComplexTensor& left_isometry,
                                 const ComplexTensor& center, const ComplexTensor& right_isometry) {
  if (theta.rank() != 4 && theta.rank() != 2)
    throw ShapeError("truncation_error_explicit expects a matrix or a rank-4 block");
  if (left_isometry.rank() != 2 || center.rank() != 2 || right_isometry.rank() != 2)
    throw ShapeError("truncation_error_explicit expects matrix factors");
  const Dev dt(theta), dl(left_isometry), dc(center), dr(right_isometry);
  double out = 0.0;
  check(qt_truncation_error_explicit(ctx(), dt.h, dl.h, dc.h, dr.h, &out));
  return out;
}

// tebd_step(UniformMPS), proj/src/gates.cpp:513-540: the state stays on the
// device for the whole step (the same update kernels qt_tebd_step_uniform
// runs); the observer sees a host snapshot after every gate
UniformStepResult tebd_step(const UniformMPS& state, const std::vector<std::pair<BondParity, TwoSiteGate>>& schedule,
                            Scheme scheme, const TruncationPolicy& policy, const UniformGateObserver& on_gate) {
  const std::size_t L = state.cell_length();
  if (L % 2 != 0) throw InputError("uniform TEBD needs an even unit cell");
  UniformStepResult result{state, {}};
  UniformMPS& s = result.state;
  if (!device_scheme(scheme)) {
    for (const auto& [parity, gate] : schedule) {
      if (gate.phys_dim() != s.phys_dim) throw ShapeError("gate physical dimension mismatch");
      for (std::size_t m = parity == BondParity::even ? 0 : 1; m < L; m += 2) {
        const std::size_t n = (m + 1) % L;
        GateUpdate upd = host_comparator(scheme, s.bond_matrices[m], s.site_tensors[m], s.site_tensors[n], gate, policy);
        s.site_tensors[m] = std::move(upd.b_m);
        s.bond_matrices[n] = std::move(upd.xi_n);
        s.site_tensors[n] = std::move(upd.b_n);
        result.reports.push_back({n, upd.report});
        if (on_gate) on_gate(s, result.reports.back());
      }
    }
    return result;
  }
  std::vector<Dev> sites, bonds;
  for (std::size_t m = 0; m < L; ++m) {
    sites.emplace_back(s.site_tensors[m]);
    bonds.emplace_back(s.bond_matrices[m]);
  }
  std::vector<bool> dirty_s(L, false), dirty_b(L, false);
  auto sync_host = [&] {
    for (std::size_t m = 0; m < L; ++m) {
      if (dirty_s[m]) s.site_tensors[m] = sites[m].host();
      if (dirty_b[m]) s.bond_matrices[m] = bonds[m].host();
      dirty_s[m] = dirty_b[m] = false;
    }
  };
  for (const auto& [parity, gate] : schedule) {
    if (gate.phys_dim() != s.phys_dim) throw ShapeError("gate physical dimension mismatch");
    const Dev du(gate.u);
    for (std::size_t m = parity == BondParity::even ? 0 : 1; m < L; m += 2) {
      const std::size_t n = (m + 1) % L;
      DevUpdate upd = device_update(scheme, bonds[m], sites[m], sites[n], du, policy, false);
      sites[m] = std::move(upd.b_m);
      bonds[n] = std::move(upd.xi);
      sites[n] = std::move(upd.b_n);
      dirty_s[m] = dirty_b[n] = dirty_s[n] = true;
      result.reports.push_back({n, upd.report});
      if (on_gate) {
        sync_host();
        on_gate(s, result.reports.back());
      }
    }
  }
  sync_host();
  return result;
}

namespace {
// a host FiniteMPS <-> a device-resident chain (qt_finite)
struct DevFinite {
  qt_finite* h = nullptr;
  explicit DevFinite(const FiniteMPS& s) {
    std::vector<Dev> sites;
    std::vector<qt_tensor*> sh;
    for (const ComplexTensor& t : s.site_tensors) {
      sites.emplace_back(t);
      sh.push_back(sites.back().h);
    }
    const Dev c(s.center_matrix);
    check(qt_finite_create(ctx(), sh.size(), sh.data(), s.center_bond, c.h, &h));
  }
  ~DevFinite() {
    if (h) qt_finite_destroy(h);
  }
  DevFinite(const DevFinite&) = delete;
  DevFinite& operator=(const DevFinite&) = delete;
  FiniteMPS host(std::size_t d, std::size_t n) const {
    FiniteMPS out;
    out.phys_dim = d;
    uint64_t c = 0;
    check(qt_finite_center_bond(h, &c));
    out.center_bond = c;
    for (std::size_t m = 0; m < n; ++m) {
      qt_tensor* v = nullptr;
      check(qt_finite_view(h, 0, m, &v));
      out.site_tensors.push_back(Dev(v).host());
    }
    qt_tensor* v = nullptr;
    check(qt_finite_view(h, 1, 0, &v));
    out.center_matrix = Dev(v).host();
    return out;
  }
};

struct FiniteObserverCtx {
  const DevFinite* f;
  std::size_t d, n;
  const FiniteGateObserver* obs;
  std::exception_ptr err;
};

int finite_observer_tramp(void* user, const qt_bond_report* rep) {
  auto* c = static_cast<FiniteObserverCtx*>(user);
  try {
    const FiniteMPS snap = c->f->host(c->d, c->n);
    (*c->obs)(snap, BondReport{rep->bond, from_c(rep->report)});
    return 0;
  } catch (...) {
    c->err = std::current_exception();
    return 1;
  }
}
}  // namespace

// tebd_step(FiniteMPS), proj/src/gates.cpp:542-578 (reference semantics:
// center moved onto every bond; QR keeps left_iso and advances the center,
// CBE renormalizes b_m by 1/sqrt(1 - eps))
FiniteStepResult tebd_step(const FiniteMPS& state, const std::vector<FiniteLayer>& layers, Scheme scheme,
                           const TruncationPolicy& policy, const FiniteGateObserver& on_gate) {
  const std::size_t n = state.length();
  for (const FiniteLayer& l : layers)
    if (l.gates.size() + 1 != n) throw ShapeError("layer gate count must equal the bond count");
  if (!device_scheme(scheme)) {
    FiniteStepResult result{state, {}};
    FiniteMPS& s = result.state;
    for (const FiniteLayer& layer : layers)
      for (std::size_t m = layer.parity == BondParity::even ? 0 : 1; m + 1 < n; m += 2) {
        s = move_center(std::move(s), m);
        GateUpdate upd =
            host_comparator(scheme, s.center_matrix, s.site_tensors[m], s.site_tensors[m + 1], layer.gates[m], policy);
        if (upd.left_iso) {
          s.site_tensors[m] = std::move(*upd.left_iso);
          s.center_matrix = std::move(upd.xi_n);
          s.center_bond = m + 1;
        } else {
          if (!policy.skip_renormalize && upd.report.eps_trunc > 0.0 && upd.report.eps_trunc < 1.0)
            upd.b_m *= 1.0 / std::sqrt(1.0 - upd.report.eps_trunc);
          s.site_tensors[m] = std::move(upd.b_m);
        }
        s.site_tensors[m + 1] = std::move(upd.b_n);
        result.reports.push_back({m + 1, upd.report});
        if (on_gate) on_gate(s, result.reports.back());
      }
    return result;
  }
  DevFinite f(state);
  std::vector<Dev> g;
  std::vector<qt_tensor*> gh;
  std::vector<int32_t> par;
  for (const FiniteLayer& l : layers) {
    par.push_back(l.parity == BondParity::even ? 0 : 1);
    for (const TwoSiteGate& u : l.gates) {
      g.emplace_back(u.u);
      gh.push_back(g.back().h);
    }
  }
  std::vector<qt_bond_report> reps(layers.size() * (n / 2 + 1) + 1);
  uint64_t cnt = reps.size();
  const qt_policy p = c_policy(policy);
  FiniteObserverCtx oc{&f, state.phys_dim, n, &on_gate, nullptr};
  const qt_status st = qt_finite_step_observed(f.h, layers.size(), par.data(), gh.data(), c_scheme(scheme), &p,
                                               reps.data(), &cnt, on_gate ? finite_observer_tramp : nullptr, &oc);
  if (oc.err) std::rethrow_exception(oc.err);
  check(st);
  FiniteStepResult out;
  out.state = f.host(state.phys_dim, n);
  for (uint64_t i = 0; i < cnt; ++i) out.reports.push_back({reps[i].bond, from_c(reps[i].report)});
  return out;
}

// ================================================================ mps
double IsometryReport::max_defect() const {
  return std::max({max_right_defect, max_left_defect, max_translation_defect, max_norm_defect});
}

IsometryReport check_isometric(const UniformMPS& mps, double tol) {
  const std::size_t L = mps.cell_length();
  std::vector<Dev> s, b;
  std::vector<qt_tensor*> sh, bh;
  for (std::size_t m = 0; m < L; ++m) {
    s.emplace_back(mps.site_tensors[m]);
    b.emplace_back(mps.bond_matrices[m]);
    sh.push_back(s.back().h);
    bh.push_back(b.back().h);
  }
  IsometryReport r;
  r.right_defects.resize(L);
  r.left_defects.resize(L);
  r.translation_defects.resize(L);
  r.norm_defects.resize(L);
  qt_isometry_report c{};
  check(qt_check_isometric_uniform(ctx(), L, sh.data(), bh.data(), tol, r.right_defects.data(),
                                   r.left_defects.data(), r.translation_defects.data(), r.norm_defects.data(), &c));
  r.max_right_defect = c.max_right_defect;
  r.max_left_defect = c.max_left_defect;
  r.max_translation_defect = c.max_translation_defect;
  r.max_norm_defect = c.max_norm_defect;
  r.pass = r.max_defect() <= tol;
  return r;
}

IsometryReport check_isometric(const FiniteMPS& mps, double tol) {
  const std::size_t n = mps.length();
  const DevFinite f(mps);
  IsometryReport r;
  r.right_defects.assign(n, 0.0);
  r.left_defects.assign(n, 0.0);
  r.norm_defects.assign(1, 0.0);
  qt_isometry_report c{};
  check(qt_check_isometric_finite(f.h, tol, r.right_defects.data(), r.left_defects.data(), r.norm_defects.data(), &c));
  r.max_right_defect = c.max_right_defect;
  r.max_left_defect = c.max_left_defect;
  r.max_translation_defect = 0.0;
  r.max_norm_defect = c.max_norm_defect;
  r.pass = r.max_defect() <= tol;
  return r;
}

namespace {
cplx expectation_on_device(const ComplexTensor& xi, const ComplexTensor& b, const ComplexTensor& op) {
  const Dev dxi(xi), db(b), dop(op);
  double out[2];
  check(qt_expectation_local(ctx(), dxi.h, db.h, dop.h, out));
  return {out[0], out[1]};
}

std::vector<double> schmidt_on_device(const ComplexTensor& xi) {
  const Dev d(xi);
  std::vector<double> s(std::min(xi.dim(0), xi.dim(1)));
  uint64_t cnt = s.size();
  check(qt_schmidt_values(ctx(), d.h, s.data(), &cnt));
  s.resize(cnt);
  return s;
}
}  // namespace

cplx expectation_local(const UniformMPS& mps, const ComplexTensor& op, std::size_t site) {
  if (op.rank() != 2 || op.dim(0) != mps.phys_dim || op.dim(1) != mps.phys_dim)
    throw ShapeError("operator must be d x d");
  if (site >= mps.cell_length()) throw InputError("site out of range");
  return expectation_on_device(mps.bond_matrices[site], mps.site_tensors[site], op);
}

cplx expectation_local(const FiniteMPS& mps, const ComplexTensor& op, std::size_t site) {
  if (op.rank() != 2 || op.dim(0) != mps.phys_dim || op.dim(1) != mps.phys_dim)
    throw ShapeError("operator must be d x d");
  if (site >= mps.length()) throw InputError("site out of range");
  const FiniteMPS c = move_center(mps, site);
  return expectation_on_device(c.center_matrix, c.site_tensors[site], op);
}

std::vector<double> schmidt_values(const UniformMPS& mps, std::size_t bond) {
  if (bond >= mps.cell_length()) throw InputError("bond out of range");
  return schmidt_on_device(mps.bond_matrices[bond]);
}

std::vector<double> schmidt_values(const FiniteMPS& mps, std::size_t bond) {
  if (bond > mps.length()) throw InputError("bond out of range");
  return schmidt_on_device(move_center(mps, bond).center_matrix);
}

double entropy_from_schmidt(const std::vector<double>& values) {
  double s = 0;
  for (double v : values) {
    const double p = v * v;
    if (p > 0.0) s -= p * std::log(p);
  }
  return s;
}

double entanglement_entropy(const UniformMPS& mps, std::size_t bond) {
  return entropy_from_schmidt(schmidt_values(mps, bond));
}

double entanglement_entropy(const FiniteMPS& mps, std::size_t bond) {
  return entropy_from_schmidt(schmidt_values(mps, bond));
}

FiniteMPS move_center(FiniteMPS mps, std::size_t new_center) {
  if (new_center > mps.length()) throw InputError("center bond out of range");
  if (new_center == mps.center_bond) return mps;
  const DevFinite f(mps);
  check(qt_finite_move_center(f.h, new_center));
  return f.host(mps.phys_dim, mps.length());
}

}  // namespace qrtebd
