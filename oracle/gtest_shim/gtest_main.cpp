// Runner of the gtest shim (TEST INFRASTRUCTURE, see gtest/gtest.h).
#include <chrono>
#include <cstdio>
#include <exception>
#include <string>
#include <vector>

#include "gtest/gtest.h"

namespace gtshim {

std::vector<TestInfo>& registry() {
  static std::vector<TestInfo> r;
  return r;
}

static int g_failures_in_test = 0;

void record_failure(const char* file, int line, const std::string& what, const std::string& msg) {
  ++g_failures_in_test;
  std::printf("%s:%d: Failure\n%s\n%s%s", file, line, what.c_str(), msg.c_str(), msg.empty() ? "" : "\n");
  std::fflush(stdout);
}

static bool glob(const char* p, const char* s) {
  if (*p == '\0') return *s == '\0';
  if (*p == '*') return glob(p + 1, s) || (*s && glob(p, s + 1));
  if (*p == '?') return *s && glob(p + 1, s + 1);
  return *p == *s && glob(p + 1, s + 1);
}

static std::vector<std::string> split(const std::string& s, char c) {
  std::vector<std::string> out;
  size_t b = 0;
  for (size_t i = 0; i <= s.size(); ++i)
    if (i == s.size() || s[i] == c) {
      if (i > b) out.push_back(s.substr(b, i - b));
      b = i + 1;
    }
  return out;
}

}  // namespace gtshim

int main(int argc, char** argv) {
  using namespace gtshim;
  std::string filter = "*";
  bool list = false;
  for (int i = 1; i < argc; ++i) {
    std::string a = argv[i];
    if (a.rfind("--gtest_filter=", 0) == 0) filter = a.substr(15);
    if (a == "--gtest_list_tests") list = true;
  }
  const size_t dash = filter.find('-');
  const auto pos = split(dash == std::string::npos ? filter : filter.substr(0, dash), ':');
  const auto neg = dash == std::string::npos ? std::vector<std::string>{} : split(filter.substr(dash + 1), ':');
  std::vector<TestInfo> run;
  for (const TestInfo& t : registry()) {
    const std::string full = t.suite + "." + t.name;
    bool in = pos.empty();
    for (const auto& p : pos) in = in || glob(p.c_str(), full.c_str());
    for (const auto& n : neg) in = in && !glob(n.c_str(), full.c_str());
    if (in) run.push_back(t);
  }
  if (list) {
    for (const TestInfo& t : run) std::printf("%s.%s\n", t.suite.c_str(), t.name.c_str());
    return 0;
  }
  std::printf("[==========] Running %zu tests.\n", run.size());
  std::vector<std::string> failed;
  const auto t_all = std::chrono::steady_clock::now();
  for (const TestInfo& t : run) {
    const std::string full = t.suite + "." + t.name;
    std::printf("[ RUN      ] %s\n", full.c_str());
    std::fflush(stdout);
    g_failures_in_test = 0;
    const auto t0 = std::chrono::steady_clock::now();
    try {
      t.fn();
    } catch (const std::exception& e) {
      record_failure("(test body)", 0, std::string("C++ exception with description \"") + e.what() + "\" thrown",
                     "");
    } catch (...) {
      record_failure("(test body)", 0, "unknown C++ exception thrown", "");
    }
    const double ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (g_failures_in_test == 0) {
      std::printf("[       OK ] %s (%.0f ms)\n", full.c_str(), ms);
    } else {
      std::printf("[  FAILED  ] %s (%.0f ms)\n", full.c_str(), ms);
      failed.push_back(full);
    }
    std::fflush(stdout);
  }
  const double ms_all =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_all).count();
  std::printf("[==========] %zu tests ran. (%.0f ms total)\n", run.size(), ms_all);
  std::printf("[  PASSED  ] %zu tests.\n", run.size() - failed.size());
  if (!failed.empty()) {
    std::printf("[  FAILED  ] %zu tests, listed below:\n", failed.size());
    for (const auto& f : failed) std::printf("[  FAILED  ] %s\n", f.c_str());
  }
  return failed.empty() ? 0 : 1;
}
