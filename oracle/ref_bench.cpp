// oracle/ref_bench.cpp -- TEST INFRASTRUCTURE (the CPU baseline leg).
// Times the reference's own update path (apply_gate, proj/src/gates.cpp:
// 452-462, in the order tebd_step runs it for a uniform L=2 cell,
// gates.cpp:513-540: even dt/2, odd dt, even dt/2) on the state bench.py
// writes, with the reference's own gate construction (trotter_schedule of the
// clock bond hamiltonian, g = 2, dt = 0.05, order 2).
//
//   ref_bench STATE_FILE d chi scheme explicit dabs drel budget_s min_updates
//
// STATE_FILE: raw complex128, site0 (d,chi,chi), site1, bond0 (chi,chi), bond1.
// Prints one JSON object {"updates", "seconds", "threads", "last_eps"}.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <string>
#include <vector>

extern "C" int scipy_openblas_get_num_threads(void);  // the BLAS pool the shim's products run on

#include "qrtebd/clock.hpp"
#include "qrtebd/gates.hpp"
#include "qrtebd/mps.hpp"

using namespace qrtebd;

int main(int argc, char** argv) {
  if (argc < 10) {
    std::fprintf(stderr, "usage: ref_bench STATE d chi scheme explicit dabs drel budget_s min_updates\n");
    return 2;
  }
  const std::string path = argv[1];
  const std::size_t d = std::strtoull(argv[2], nullptr, 10), chi = std::strtoull(argv[3], nullptr, 10);
  const Scheme scheme = scheme_from_name(argv[4]);
  TruncationPolicy pol;
  pol.chi_max = chi;
  pol.compute_explicit_error = std::atoi(argv[5]) != 0;
  pol.delta_chi_abs = std::strtoull(argv[6], nullptr, 10);
  pol.delta_chi_rel = std::atof(argv[7]);
  const double budget = std::atof(argv[8]);
  const long min_updates = std::atol(argv[9]);

  std::ifstream in(path, std::ios::binary);
  auto read = [&](std::vector<std::size_t> shape) {
    ComplexTensor t(shape);
    in.read(reinterpret_cast<char*>(t.data().data()), static_cast<std::streamsize>(t.size() * sizeof(cplx)));
    return t;
  };
  std::vector<ComplexTensor> sites = {read({d, chi, chi}), read({d, chi, chi})};
  std::vector<ComplexTensor> bonds = {read({chi, chi}), read({chi, chi})};
  if (!in) {
    std::fprintf(stderr, "short state file\n");
    return 2;
  }
  const auto sched = trotter_schedule(bond_hamiltonian(ClockModel{d, 2.0}, BondKind::bulk), 0.05, 2);

  long k = 0, n = 0;
  double last_eps = 0.0;
  const auto t0 = std::chrono::steady_clock::now();
  auto elapsed = [&] { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); };
  for (;;) {
    const auto& [parity, gate] = sched[k % sched.size()];
    const std::size_t m = parity == BondParity::even ? 0 : 1, nn = 1 - m;
    GateUpdate upd = apply_gate(scheme, bonds[m], sites[m], sites[nn], gate, pol);
    sites[m] = std::move(upd.b_m);
    bonds[nn] = std::move(upd.xi_n);
    sites[nn] = std::move(upd.b_n);
    last_eps = upd.report.eps_trunc;
    ++k;
    ++n;
    if (std::getenv("REF_BENCH_VERBOSE")) std::fprintf(stderr, "update %ld at %.3f s\n", n, elapsed());
    if (n >= min_updates && elapsed() >= budget) break;
  }
  const int threads = scipy_openblas_get_num_threads();
  std::printf("{\"updates\": %ld, \"seconds\": %.6f, \"threads\": %d, \"last_eps\": %.17g}\n", n, elapsed(), threads,
              last_eps);
  return 0;
}
