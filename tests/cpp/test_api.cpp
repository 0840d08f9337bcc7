// C++ drop-in check: the reference-shaped API (include/qrtebd/qrtebd_b200.hpp)
// driven the way proj/tests/test_gates.cc:271-309 drives the reference.
#include <cmath>
#include <cstdio>
#include <random>

#include "qrtebd/qrtebd_b200.hpp"

using namespace qrtebd;

static ComplexTensor random_tensor(std::vector<std::size_t> shape, unsigned seed) {
  std::mt19937 rng(seed);
  std::normal_distribution<double> nd;
  ComplexTensor t(std::move(shape));
  for (cplx& v : t.data()) v = cplx(nd(rng), nd(rng));
  return t;
}

int main() {
  Context ctx(0);
  int fails = 0;
  // identity gate is an exact fixed point (test_gates.cc:271-287): eps <= 1e-14
  const std::size_t d = 2, chi = 2;
  ComplexTensor xi({chi, chi});
  xi.data()[0] = std::sqrt(0.8);
  xi.data()[3] = std::sqrt(0.2);
  // right-isometric site tensors from LQ of Gaussians through the device LQ
  auto right_iso = [&](unsigned seed) {
    ComplexTensor g = random_tensor({chi, d * chi}, seed);
    DeviceTensor dg(ctx, g);
    qt_tensor *l = nullptr, *q = nullptr;
    check(qt_lq_reduced(ctx.get(), dg.get(), &l, &q));
    DeviceTensor tl(l), tq(q);
    ComplexTensor qh = tq.host();  // (chi, d*chi) -> (d, chi, chi)
    ComplexTensor b({d, chi, chi});
    for (std::size_t a = 0; a < chi; ++a)
      for (std::size_t i = 0; i < d; ++i)
        for (std::size_t c = 0; c < chi; ++c) b.data()[(i * chi + a) * chi + c] = qh.data()[a * d * chi + i * chi + c];
    return b;
  };
  const ComplexTensor bm = right_iso(240), bn = right_iso(241);
  TwoSiteGate id{ComplexTensor::identity(d * d)};
  id.u = ComplexTensor({d, d, d, d}, id.u.data());
  TruncationPolicy p;
  p.chi_max = 2;
  p.delta_chi_abs = 0;
  p.delta_chi_rel = 0.0;
  const GateUpdate upd = apply_gate_qr(ctx, xi, bm, bn, id, p);
  if (!(upd.report.eps_trunc <= 1e-14)) {
    std::printf("eps %g\n", upd.report.eps_trunc);
    ++fails;
  }
  if (upd.report.chi_after != 2) ++fails;
  if (!upd.left_iso) ++fails;
  // B~n right-isometric (test_gates.cc:289-309)
  double defect = 0;
  for (std::size_t a = 0; a < chi; ++a)
    for (std::size_t c = 0; c < chi; ++c) {
      cplx s = 0;
      for (std::size_t i = 0; i < d; ++i)
        for (std::size_t b = 0; b < chi; ++b)
          s += upd.b_n.data()[(i * chi + a) * chi + b] * std::conj(upd.b_n.data()[(i * chi + c) * chi + b]);
      defect = std::max(defect, std::abs(s - (a == c ? 1.0 : 0.0)));
    }
  if (defect > 1e-12) ++fails;
  // errors map onto the reference taxonomy
  try {
    apply_gate_qr(ctx, ComplexTensor::identity(3), bm, bn, id, p);
    ++fails;
  } catch (const ShapeError&) {
  }
  // uniform step + observables
  UniformMPS st;
  st.phys_dim = d;
  st.site_tensors = {bm, bn};
  st.bond_matrices = {xi, xi};
  std::vector<std::pair<BondParity, TwoSiteGate>> sched = {{BondParity::even, id}, {BondParity::odd, id}};
  const UniformStepResult r = tebd_step(ctx, st, sched, Scheme::qr, p);
  if (r.reports.size() != 2) ++fails;
  const double s0 = entanglement_entropy(ctx, r.state, 0);
  if (!(s0 >= 0.0)) ++fails;
  // finite chain with the reference's sequential semantics (gates.cpp:542-578):
  // a product state under the identity gate stays put; the center moves to bond 1
  {
    FiniteMPS f;
    f.phys_dim = d;
    ComplexTensor v({d, 1, 1});
    v.data()[0] = 1.0;
    f.site_tensors = {v, v, v};
    f.center_bond = 0;
    f.center_matrix = ComplexTensor::identity(1);
    FiniteLayer lay;
    lay.parity = BondParity::even;
    lay.gates = {id, id};
    const FiniteStepResult fr = tebd_step(ctx, f, {lay}, Scheme::qr, p);
    if (fr.reports.size() != 1 || fr.state.center_bond != 1) ++fails;
    ComplexTensor z({d, d});
    z.data()[0] = 1.0;
    z.data()[3] = -1.0;
    for (std::size_t site = 0; site < 3; ++site)
      if (std::abs(expectation_local(ctx, fr.state, z, site) - cplx(1.0)) > 1e-12) ++fails;
    const std::vector<double> sv = schmidt_values(ctx, fr.state, 2);
    if (sv.empty() || std::abs(sv[0] - 1.0) > 1e-12) ++fails;
    if (move_center(ctx, fr.state, 0).center_bond != 0) ++fails;
  }
  std::printf("%s: eps=%.3e defect=%.3e S=%.6f\n", fails ? "FAIL" : "OK", upd.report.eps_trunc, defect, s0);
  return fails ? 1 : 0;
}
