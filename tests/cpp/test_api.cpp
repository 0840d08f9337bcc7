// C++ drop-in check: the reference's own API signatures
// (include/qrtebd/qrtebd_api.hpp -> libqrtebd_api.so, the B200 path) driven
// the way proj/tests/test_gates.cc:271-309 drives the reference -- no
// context argument, value semantics, reference exception types.
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
  int fails = 0;
  // identity gate is an exact fixed point (test_gates.cc:271-287): eps <= 1e-14
  const std::size_t d = 2, chi = 2;
  ComplexTensor xi({chi, chi});
  xi.data()[0] = std::sqrt(0.8);
  xi.data()[3] = std::sqrt(0.2);
  // right-isometric site tensors from LQ of Gaussians through the device LQ
  auto right_iso = [&](unsigned seed) {  // test_gates.cc:19-23, device LQ
    return lq_reduced(random_tensor({chi, d * chi}, seed)).q.reshape({chi, d, chi}).transpose({1, 0, 2});
  };
  const ComplexTensor bm = right_iso(240), bn = right_iso(241);
  TwoSiteGate id{ComplexTensor::identity(d * d).reshape({d, d, d, d})};
  TruncationPolicy p;
  p.chi_max = 2;
  p.delta_chi_abs = 0;
  p.delta_chi_rel = 0.0;
  const GateUpdate upd = apply_gate_qr(xi, bm, bn, id, p);
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
    apply_gate_qr(ComplexTensor::identity(3), bm, bn, id, p);
    ++fails;
  } catch (const ShapeError&) {
  }
  // uniform step + observables
  UniformMPS st;
  st.phys_dim = d;
  st.site_tensors = {bm, bn};
  st.bond_matrices = {xi, xi};
  std::vector<std::pair<BondParity, TwoSiteGate>> sched = {{BondParity::even, id}, {BondParity::odd, id}};
  int observed = 0;  // UniformGateObserver fires after every gate (gates.hpp:120-123)
  const UniformStepResult r =
      tebd_step(st, sched, Scheme::qr, p, [&](const UniformMPS&, const BondReport&) { ++observed; });
  if (r.reports.size() != 2 || observed != 2) ++fails;
  // contract (tensor.cpp:172-233) on the device GEMM vs a loop
  {
    const ComplexTensor a = random_tensor({3, 4, 5}, 7), b = random_tensor({5, 4, 2}, 8);
    const ComplexTensor c = contract(a, b, {{1, 1}, {2, 0}});  // (3, 2)
    double err = 0;
    for (std::size_t i = 0; i < 3; ++i)
      for (std::size_t j = 0; j < 2; ++j) {
        cplx acc = 0;
        for (std::size_t x = 0; x < 4; ++x)
          for (std::size_t y = 0; y < 5; ++y) acc += a.at({i, x, y}) * b.at({y, x, j});
        err = std::max(err, std::abs(acc - c.at({i, j})));
      }
    if (c.shape() != std::vector<std::size_t>({3, 2}) || err > 1e-13) {
      std::printf("contract err %g\n", err);
      ++fails;
    }
  }
  const double s0 = entanglement_entropy(r.state, 0);
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
    const FiniteStepResult fr = tebd_step(f, {lay}, Scheme::qr, p);
    if (fr.reports.size() != 1 || fr.state.center_bond != 1) ++fails;
    ComplexTensor z({d, d});
    z.data()[0] = 1.0;
    z.data()[3] = -1.0;
    for (std::size_t site = 0; site < 3; ++site)
      if (std::abs(expectation_local(fr.state, z, site) - cplx(1.0)) > 1e-12) ++fails;
    const std::vector<double> sv = schmidt_values(fr.state, 2);
    if (sv.empty() || std::abs(sv[0] - 1.0) > 1e-12) ++fails;
    if (move_center(fr.state, 0).center_bond != 0) ++fails;
  }
  // the device-resident fast path gives the same step
  {
    b200::DeviceUniformMPS dev(st);
    dev.step(sched, Scheme::qr, p, false);
    const UniformMPS snap = dev.snapshot();
    for (std::size_t m = 0; m < 2; ++m)
      for (std::size_t k = 0; k < snap.site_tensors[m].size(); ++k)
        if (std::abs(snap.site_tensors[m].data()[k] - r.state.site_tensors[m].data()[k]) > 1e-12) {
          ++fails;
          break;
        }
  }
  std::printf("%s: eps=%.3e defect=%.3e S=%.6f\n", fails ? "FAIL" : "OK", upd.report.eps_trunc, defect, s0);
  return fails ? 1 : 0;
}
