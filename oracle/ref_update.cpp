// oracle/ref_update.cpp -- TEST INFRASTRUCTURE: one two-site update through
// the reference's own apply_gate (proj/src/gates.cpp:452-462) on inputs from
// a file, outputs to a file.  Used to pin the NumPy oracle and to generate
// golden fixtures (tests/golden/make_ref_golden.py).
//
//   ref_update IN OUT
// IN : int64[16] {scheme, d, chi_l, chi_m, chi_n, chi_r, chi_max, delta_chi_abs,
//                 chi_max_expansion, qr_sweeps, explicit, skip_renormalize, 0...}
//      double[4] {sv_cutoff, target_eps, delta_chi_rel, 0}
//      complex128 xi (chi_l, chi_m), b_m (d, chi_m, chi_n), b_n (d, chi_n, chi_r), u (d, d, d, d)
// OUT: int64[8] {kk, has_left_iso, chi_before, chi_expanded, chi_after, 0, 0, 0}
//      double[2] {eps_trunc, discarded_weight}
//      complex128 b_m (d, chi_m, kk), xi_n (kk, kk), b_n (d, kk, chi_r) [, left_iso (d, chi_l, kk)]
// Exit status: 0 ok; 1 ShapeError/InputError; 2 NumericError; 3 CapacityError.
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <vector>

#include "qrtebd/errors.hpp"
#include "qrtebd/gates.hpp"

using namespace qrtebd;

int main(int argc, char** argv) {
  if (argc != 3) {
    std::fprintf(stderr, "usage: ref_update IN OUT\n");
    return 4;
  }
  std::ifstream in(argv[1], std::ios::binary);
  int64_t h[16];
  double hd[4];
  in.read(reinterpret_cast<char*>(h), sizeof(h));
  in.read(reinterpret_cast<char*>(hd), sizeof(hd));
  const auto sz = [](int64_t v) { return static_cast<std::size_t>(v); };
  const std::size_t d = sz(h[1]), chi_l = sz(h[2]), chi_m = sz(h[3]), chi_n = sz(h[4]), chi_r = sz(h[5]);
  auto read = [&](std::vector<std::size_t> shape) {
    ComplexTensor t(shape);
    in.read(reinterpret_cast<char*>(t.data().data()), static_cast<std::streamsize>(t.size() * sizeof(cplx)));
    return t;
  };
  const ComplexTensor xi = read({chi_l, chi_m}), bm = read({d, chi_m, chi_n}), bn = read({d, chi_n, chi_r});
  TwoSiteGate u{read({d, d, d, d})};
  if (!in) {
    std::fprintf(stderr, "short input\n");
    return 4;
  }
  TruncationPolicy pol;
  pol.chi_max = sz(h[6]);
  pol.delta_chi_abs = sz(h[7]);
  pol.chi_max_expansion = sz(h[8]);
  pol.qr_sweeps = static_cast<int>(h[9]);
  pol.compute_explicit_error = h[10] != 0;
  pol.skip_renormalize = h[11] != 0;
  pol.sv_cutoff = hd[0];
  pol.target_eps = hd[1];
  pol.delta_chi_rel = hd[2];
  const Scheme scheme = static_cast<Scheme>(h[0]);
  try {
    const GateUpdate g = apply_gate(scheme, xi, bm, bn, u, pol);
    std::ofstream out(argv[2], std::ios::binary);
    const int64_t oh[8] = {static_cast<int64_t>(g.xi_n.dim(0)), g.left_iso ? 1 : 0,
                           static_cast<int64_t>(g.report.chi_before), static_cast<int64_t>(g.report.chi_expanded),
                           static_cast<int64_t>(g.report.chi_after), 0, 0, 0};
    const double od[2] = {g.report.eps_trunc, g.report.discarded_weight};
    out.write(reinterpret_cast<const char*>(oh), sizeof(oh));
    out.write(reinterpret_cast<const char*>(od), sizeof(od));
    auto write = [&](const ComplexTensor& t) {
      out.write(reinterpret_cast<const char*>(t.data().data()), static_cast<std::streamsize>(t.size() * sizeof(cplx)));
    };
    write(g.b_m);
    write(g.xi_n);
    write(g.b_n);
    if (g.left_iso) write(*g.left_iso);
  } catch (const ShapeError& e) {
    std::fprintf(stderr, "ShapeError: %s\n", e.what());
    return 1;
  } catch (const InputError& e) {
    std::fprintf(stderr, "InputError: %s\n", e.what());
    return 1;
  } catch (const NumericError& e) {
    std::fprintf(stderr, "NumericError: %s\n", e.what());
    return 2;
  } catch (const CapacityError& e) {
    std::fprintf(stderr, "CapacityError: %s\n", e.what());
    return 3;
  }
  return 0;
}
