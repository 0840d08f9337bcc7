// Times the reference's public pieces at a bench size (diagnostic for the
// CPU baseline; links oracle/_ref/libqrtebd_ref.so).
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <random>
#include "qrtebd/clock.hpp"
#include "qrtebd/gates.hpp"
#include "qrtebd/linalg.hpp"
using namespace qrtebd;
static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
int main(int argc, char** argv) {
  const size_t d = argc > 1 ? std::atoi(argv[1]) : 5, chi = argc > 2 ? std::atoi(argv[2]) : 1024;
  ComplexTensor th({chi, d, d, chi});
  for (auto& v : th.data()) v = {1e-3, 2e-3};
  double t = now();
  auto tt = th.transpose({2, 0, 1, 3});
  std::printf("transpose(2,0,1,3) of theta: %.3f s\n", now() - t);
  t = now();
  double n = th.norm();
  std::printf("norm: %.3f s (%g)\n", now() - t, n);
  ComplexTensor y({chi, d * chi});
  for (auto& v : y.data()) v = {1e-3, -2e-3};
  ComplexTensor x({chi * d, chi});
  std::mt19937 rng(1);
  std::normal_distribution<double> nd;
  for (auto& v : x.data()) v = {nd(rng), nd(rng)};
  auto thm = th.reshape({chi * d, d * chi});
  t = now();
  auto c = contract(thm, y, {{1, 1}});
  std::printf("contract theta y^T (GEMM %zux%zux%zu): %.3f s\n", chi * d, chi, d * chi, now() - t);
  t = now();
  auto q = qr_reduced(x);
  std::printf("qr_reduced %zux%zu: %.3f s\n", chi * d, chi, now() - t);
  t = now();
  auto l = lq_reduced(y);
  std::printf("lq_reduced %zux%zu: %.3f s\n", chi, d * chi, now() - t);
  t = now();
  double e = truncation_error_explicit(thm, q.q, l.l, l.q);
  std::printf("truncation_error_explicit: %.3f s (%g)\n", now() - t, e);
  // one full update
  auto riso = [&](unsigned s) {
    ComplexTensor g({chi, d * chi});
    std::mt19937 r2(s);
    for (auto& v : g.data()) v = {nd(r2), nd(r2)};
    return lq_reduced(g).q.reshape({chi, d, chi}).transpose({1, 0, 2});
  };
  auto bm = riso(2), bn = riso(3);
  ComplexTensor xi({chi, chi});
  for (auto& v : xi.data()) v = {nd(rng), nd(rng)};
  xi *= 1.0 / xi.norm();
  auto g = make_gate(bond_hamiltonian({d, 2.0}, BondKind::bulk), 0.05);
  TruncationPolicy p;
  p.chi_max = chi;
  p.delta_chi_abs = 0;
  p.delta_chi_rel = 0;
  t = now();
  auto u = apply_gate_qr(xi, bm, bn, g, p);
  std::printf("apply_gate_qr: %.3f s (eps %g)\n", now() - t, u.report.eps_trunc);
}
