// Device-resident UniformMPS with a CUDA-graph step (the fast path of
// "a device-resident fast path keeps state on the GPU across
// steps"; tebd_step semantics of proj/src/gates.cpp:513-540).
//
// Every site tensor and bond matrix owns two HBM buffers; an update reads the
// live buffers and writes the spare ones, so a Trotter step is a fixed
// sequence of kernels over fixed addresses.  Once the bond dimensions are
// stationary (QR scheme, eta == chi on every bond) the step is captured once
// per buffer-parity pattern and replayed as one graph launch: no host work and
// no launch gaps inside the step.  The report scalars of every update are
// copied into pinned host memory inside the graph.
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "gate.cuh"

namespace qt {

struct UniformDev {
  Engine* e = nullptr;
  int L = 0;
  long long d = 0;
  std::vector<long long> chi;  // chi[m]: dimension of the bond left of site m
  std::vector<double2*> sbuf[2], bbuf[2];
  std::vector<size_t> scap[2], bcap[2];
  std::vector<int> sact, bact;
  double* rep_dev = nullptr;   // [updates][8]
  double* rep_host = nullptr;  // pinned mirror
  size_t rep_cap = 0;
  struct GraphEntry {
    cudaGraphExec_t exec = nullptr;
    std::vector<GemmProfRec> prof;
    unsigned long long kernels = 0;  // kernel nodes in the graph
    unsigned long long arena_gen = 0;  // workspace generation the graph's pointers belong to
  };
  std::map<std::string, GraphEntry> graphs;
  std::map<std::string, int> seen;
  // L >= 4: the L/2 updates of a layer are independent
  // (proj/tests/test_tebd.cc:139-175); update j of a layer runs on engine j
  // (0 = the context's own), each with its own stream and workspace; the
  // streams fork from and join into the main stream around every layer
  // (inside a captured graph the fork/join become graph dependencies)
  std::vector<Engine*> aux;
  std::vector<cudaEvent_t> ev;

  // sum of the workspace generations of every engine a step touches
  unsigned long long arena_gen() const {
    unsigned long long g = e->arena_gen;
    for (const Engine* a : aux) g += a->arena_gen;
    return g;
  }
  long long site_elems(int m) const { return d * chi[m] * chi[(m + 1) % L]; }
  long long bond_elems(int m) const { return chi[m] * chi[m]; }
};

namespace {

double2* ensure(double2*& p, size_t& cap, size_t elems) {
  if (cap < elems) {
    if (p) QT_CUDA(cudaFree(p));
    p = nullptr;
    cap = 0;
    QT_CUDA(cudaMalloc(&p, std::max<size_t>(elems, 1) * sizeof(double2)));
    cap = elems;
  }
  return p;
}

struct Upd {
  int m, n;
  const double2* u;
};

}  // namespace

UniformDev* uniform_create(Engine& e, int L, long long d, const std::vector<long long>& chi,
                           const std::vector<const double2*>& sites, const std::vector<const double2*>& bonds) {
  auto* s = new UniformDev;
  s->e = &e;
  s->L = L;
  s->d = d;
  s->chi = chi;
  for (int p = 0; p < 2; ++p) {
    s->sbuf[p].assign(L, nullptr);
    s->bbuf[p].assign(L, nullptr);
    s->scap[p].assign(L, 0);
    s->bcap[p].assign(L, 0);
  }
  s->sact.assign(L, 0);
  s->bact.assign(L, 0);
  for (int m = 0; m < L; ++m) {
    ensure(s->sbuf[0][m], s->scap[0][m], s->site_elems(m));
    ensure(s->bbuf[0][m], s->bcap[0][m], s->bond_elems(m));
    QT_CUDA(cudaMemcpyAsync(s->sbuf[0][m], sites[m], s->site_elems(m) * sizeof(double2), cudaMemcpyDeviceToDevice,
                            e.stream));
    QT_CUDA(cudaMemcpyAsync(s->bbuf[0][m], bonds[m], s->bond_elems(m) * sizeof(double2), cudaMemcpyDeviceToDevice,
                            e.stream));
  }
  QT_CUDA(cudaStreamSynchronize(e.stream));
  return s;
}

void uniform_destroy(UniformDev* s) {
  if (!s) return;
  cudaStreamSynchronize(s->e->stream);
  for (Engine* a : s->aux) {
    a->destroy();
    delete a;
  }
  for (cudaEvent_t x : s->ev) cudaEventDestroy(x);
  for (auto& kv : s->graphs) {
    cudaGraphExecDestroy(kv.second.exec);
    for (auto& r : kv.second.prof) {
      cudaEventDestroy(r.e0);
      cudaEventDestroy(r.e1);
    }
  }
  for (int p = 0; p < 2; ++p)
    for (int m = 0; m < s->L; ++m) {
      if (s->sbuf[p][m]) cudaFree(s->sbuf[p][m]);
      if (s->bbuf[p][m]) cudaFree(s->bbuf[p][m]);
    }
  if (s->rep_dev) cudaFree(s->rep_dev);
  if (s->rep_host) cudaFreeHost(s->rep_host);
  delete s;
}

double2* uniform_live(UniformDev* s, int which, int m, long long* shape) {
  if (m < 0 || m >= s->L) throw Error(Err::input, "site/bond index out of range");
  if (which == 0) {
    shape[0] = s->d;
    shape[1] = s->chi[m];
    shape[2] = s->chi[(m + 1) % s->L];
    return s->sbuf[s->sact[m]][m];
  }
  shape[0] = s->chi[m];
  shape[1] = s->chi[m];
  return s->bbuf[s->bact[m]][m];
}

// One Trotter step; one StepRecord per update.
std::vector<StepRecord> uniform_step(UniformDev* s, const std::vector<std::pair<int, const double2*>>& layers,
                                     int scheme_qr, const qt_policy& pol, bool use_graph) {
  Engine& e = *s->e;
  const int L = s->L;
  if (L % 2 != 0) throw Error(Err::input, "uniform TEBD needs an even unit cell");
  std::vector<Upd> ups;
  for (const auto& ly : layers)
    for (int m = ly.first; m < L; m += 2) ups.push_back({m, (m + 1) % L, ly.second});
  const size_t nup = ups.size();
  if (s->rep_cap < nup) {
    if (s->rep_dev) QT_CUDA(cudaFree(s->rep_dev));
    if (s->rep_host) QT_CUDA(cudaFreeHost(s->rep_host));
    QT_CUDA(cudaMalloc(&s->rep_dev, 8 * nup * sizeof(double)));
    QT_CUDA(cudaMallocHost(&s->rep_host, 8 * nup * sizeof(double)));
    s->rep_cap = nup;
  }

  // stationary dimensions: every QR update keeps eta == chi_n
  bool steady = scheme_qr != 0;
  {
    std::vector<long long> chi = s->chi;
    for (const Upd& u : ups) {
      Dims D{s->d, chi[u.m], chi[u.m], chi[u.n], chi[(u.n + 1) % L]};
      if (!scheme_qr) break;
      const long long eta = qr_eta(pol, D);
      if (eta != chi[u.n]) steady = false;
      chi[u.n] = eta;
    }
  }

  std::vector<StepRecord> out(nup);
  for (size_t k = 0; k < nup; ++k) {
    // static per-update fields (a replayed graph runs no host code)
    out[k].bond = ups[k].n;
    out[k].before = out[k].eta = out[k].after = s->chi[ups[k].n];
  }
  // layer boundaries in `ups` and the engine of every update
  std::vector<size_t> layer_start;
  {
    size_t k = 0;
    for (const auto& ly : layers) {
      layer_start.push_back(k);
      for (int m = ly.first; m < L; m += 2) ++k;
    }
    layer_start.push_back(k);
  }
  const bool concurrent = scheme_qr && L >= 4 && std::getenv("QT_UNIFORM_SERIAL") == nullptr;
  if (concurrent) {
    const size_t need = static_cast<size_t>(L / 2 - 1);
    while (s->aux.size() < need) {
      Engine* a = new Engine;
      a->init(e.device, nullptr);
      s->aux.push_back(a);
    }
    while (s->ev.size() < 2 * (need + 1)) {
      cudaEvent_t x;
      QT_CUDA(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
      s->ev.push_back(x);
    }
  }
  auto engine_of = [&](size_t k) -> Engine& {
    if (!concurrent) return e;
    size_t ly = 0;
    while (layer_start[ly + 1] <= k) ++ly;
    const size_t j = k - layer_start[ly];
    return j == 0 ? e : *s->aux[j - 1];
  };
  auto fork = [&](size_t nj) {  // aux streams 0..nj-2 wait for the main stream
    if (!concurrent || nj < 2) return;
    QT_CUDA(cudaEventRecord(s->ev[0], e.stream));
    for (size_t j = 1; j < nj; ++j) QT_CUDA(cudaStreamWaitEvent(s->aux[j - 1]->stream, s->ev[0], 0));
  };
  auto join = [&](size_t nj) {  // the main stream waits for the aux streams
    if (!concurrent || nj < 2) return;
    for (size_t j = 1; j < nj; ++j) {
      QT_CUDA(cudaEventRecord(s->ev[j], s->aux[j - 1]->stream));
      QT_CUDA(cudaStreamWaitEvent(e.stream, s->ev[j], 0));
    }
  };
  auto run_updates = [&](bool eager) {
    std::vector<int> sact = s->sact, bact = s->bact;
    size_t ly = 0;
    for (size_t k = 0; k < nup; ++k) {
      if (k == layer_start[ly]) fork(layer_start[ly + 1] - layer_start[ly]);
      const Upd& u = ups[k];
      Engine& eu = engine_of(k);
      const int m = u.m, n = u.n, nr = (n + 1) % L;
      Dims D{s->d, s->chi[m], s->chi[m], s->chi[n], s->chi[nr]};
      const double2* xi = s->bbuf[bact[m]][m];
      const double2* bm = s->sbuf[sact[m]][m];
      const double2* bn = s->sbuf[sact[n]][n];
      auto outputs = [&](long long w) {
        GateBuffers gb;
        gb.b_m = ensure(s->sbuf[sact[m] ^ 1][m], s->scap[sact[m] ^ 1][m], s->d * D.chi_m * w);
        gb.xi = ensure(s->bbuf[bact[n] ^ 1][n], s->bcap[bact[n] ^ 1][n], w * w);
        gb.b_n = ensure(s->sbuf[sact[n] ^ 1][n], s->scap[sact[n] ^ 1][n], s->d * w * D.chi_r);
        gb.left_iso = nullptr;
        return gb;
      };
      out[k].bond = n;
      out[k].before = D.chi_n;
      if (scheme_qr) {
        const long long eta = qr_eta(pol, D);
        gate_qr_async(eu, D, xi, bm, bn, u.u, pol, eta, outputs(eta));
        QT_CUDA(cudaMemcpyAsync(s->rep_dev + 8 * k, eu.dscal, 8 * sizeof(double), cudaMemcpyDeviceToDevice,
                                eu.stream));
        out[k].eta = out[k].after = eta;
        if (eager) s->chi[n] = eta;
      } else {
        const CbeResult r = gate_cbe(e, D, xi, bm, bn, u.u, pol, outputs);
        out[k].eta = r.eta;
        out[k].after = r.kk;
        out[k].rep = r.rep;
        s->chi[n] = r.kk;
      }
      sact[m] ^= 1;
      bact[n] ^= 1;
      sact[n] ^= 1;
      if (eager) {
        s->sact = sact;
        s->bact = bact;
      }
      if (k + 1 == layer_start[ly + 1]) {
        join(layer_start[ly + 1] - layer_start[ly]);
        ++ly;
      }
    }
    if (scheme_qr)
      QT_CUDA(cudaMemcpyAsync(s->rep_host, s->rep_dev, 8 * nup * sizeof(double), cudaMemcpyDeviceToHost, e.stream));
    return std::make_pair(sact, bact);
  };

  bool replayed = false;
  if (steady && use_graph) {
    // key: buffer parities, bond dimensions, gate pointers, policy bytes
    std::string key;
    auto put = [&](const void* p, size_t n) { key.append(static_cast<const char*>(p), n); };
    put(s->sact.data(), s->sact.size() * sizeof(int));
    put(s->bact.data(), s->bact.size() * sizeof(int));
    put(s->chi.data(), s->chi.size() * sizeof(long long));
    for (const Upd& u : ups) put(&u.u, sizeof(u.u));
    put(&pol, sizeof(pol));
    auto it = s->graphs.find(key);
    if (it != s->graphs.end() && it->second.arena_gen != s->arena_gen()) {
      // a workspace slot was reallocated since the capture (another call on
      // this context grew it): the graph's pointers are stale -- run this
      // step eagerly and recapture on the next one
      cudaGraphExecDestroy(it->second.exec);
      for (auto& r : it->second.prof) {
        cudaEventDestroy(r.e0);
        cudaEventDestroy(r.e1);
      }
      s->graphs.erase(it);
      it = s->graphs.end();
      s->seen[key] = 0;
    }
    if (it == s->graphs.end() && s->seen[key] >= 1) {
      // buffers are sized by an earlier eager step with the same key: capture
      cudaGraph_t g = nullptr;
      gemm_profile_take_captured();  // drop stale records
      const unsigned long long k0 = g_kernel_launches.load();
      QT_CUDA(cudaStreamBeginCapture(e.stream, cudaStreamCaptureModeThreadLocal));
      try {
        run_updates(false);
      } catch (...) {
        cudaStreamEndCapture(e.stream, &g);
        if (g) cudaGraphDestroy(g);
        throw;
      }
      QT_CUDA(cudaStreamEndCapture(e.stream, &g));
      UniformDev::GraphEntry ge;
      ge.arena_gen = s->arena_gen();
      // keep the captured stream priorities (latency-bound panel chains above
      // the side streams' GEMMs); by default a graph runs every kernel node at
      // the launch stream's priority
      QT_CUDA(cudaGraphInstantiateWithFlags(&ge.exec, g, cudaGraphInstantiateFlagUseNodePriority));
      QT_CUDA(cudaGraphDestroy(g));
      ge.prof = gemm_profile_take_captured();
      // captured launches are not executed: count them at replay instead
      ge.kernels = g_kernel_launches.load() - k0;
      g_kernel_launches.fetch_sub(ge.kernels, std::memory_order_relaxed);
      it = s->graphs.emplace(key, std::move(ge)).first;
    }
    if (it != s->graphs.end()) {
      QT_CUDA(cudaGraphLaunch(it->second.exec, e.stream));
      g_kernel_launches.fetch_add(it->second.kernels, std::memory_order_relaxed);
      // the same parity flips the captured sequence performed
      for (const Upd& u : ups) {
        s->sact[u.m] ^= 1;
        s->bact[u.n] ^= 1;
        s->sact[u.n] ^= 1;
      }
      replayed = true;
      QT_CUDA(cudaStreamSynchronize(e.stream));
      if (gemm_profile_active()) gemm_profile_add_replay(it->second.prof);
    } else {
      s->seen[key] += 1;
    }
  }
  if (!replayed) {
    run_updates(true);
    QT_CUDA(cudaStreamSynchronize(e.stream));
  }
  if (scheme_qr) {
    for (size_t k = 0; k < nup; ++k) {
      const double* r = s->rep_host + 8 * k;
      out[k].rep.theta2 = r[SC_THETA2];
      out[k].rep.kept2 = r[SC_L2];
      out[k].rep.resid = r[SC_RESID];
      int fl = 0;
      std::memcpy(&fl, &r[SC_TMP3], sizeof(int));
      out[k].rep.finite = fl == 0;
    }
  }
  return out;
}

}  // namespace qt
