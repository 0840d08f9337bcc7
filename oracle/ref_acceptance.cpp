// oracle/ref_acceptance.cpp -- TEST INFRASTRUCTURE.
// Compiles the reference's acceptance runner (proj/tests/acceptance.cc) in
// place and runs only the criteria named on the command line (default
// 2 4 5: the hot-path criteria -- 4-scheme agreement at d=5 chi=128,
// truncation-error semantics, CBE canonical form).  Linked against
// oracle/_ref/libqrtebd_ref.so (reference + Eigen shim) it validates the
// oracle; linked against the B200 library (oracle/Makefile.b200) it is the
// reference's own system-level contract run on the GPU path.
#define main qrtebd_acceptance_all_criteria
#include "acceptance.cc"
#undef main

#include <cstdlib>

int main(int argc, char** argv) {
  std::vector<int> ids;
  for (int i = 1; i < argc; ++i) ids.push_back(std::atoi(argv[i]));
  if (ids.empty()) ids = {2, 4, 5};
  bool all_pass = true;
  FiniteRunStats fin;
  UniformRunStats uni;
  for (int id : ids) {
    switch (id) {
      case 1: report(1, criterion1(fin), all_pass); break;
      case 2: report(2, criterion2(uni), all_pass); break;
      case 3: report(3, criterion3(), all_pass); break;
      case 4: report(4, criterion4(), all_pass); break;
      case 5: report(5, criterion5(), all_pass); break;
      case 6: report(6, criterion6(fin, uni), all_pass); break;
      case 7: report(7, criterion7(), all_pass); break;
      default: std::printf("unknown criterion %d\n", id); all_pass = false;
    }
  }
  std::printf("acceptance: %s\n", all_pass ? "ALL PASS" : "FAILURES PRESENT");
  return all_pass ? 0 : 1;
}
