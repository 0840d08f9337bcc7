// extern "C" boundary (include/qrtebd_c.h).  Thin: validates shapes with the
// reference's error taxonomy, allocates output handles, calls the engine.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "gate.cuh"

struct qt_ctx {
  qt::Engine eng;
};

struct qt_tensor {
  qt_ctx* ctx = nullptr;
  int rank = 0;
  uint64_t shape[4] = {1, 1, 1, 1};
  double2* data = nullptr;
  bool owning = false;
  size_t numel() const {
    size_t n = 1;
    for (int k = 0; k < rank; ++k) n *= shape[k];
    return n;
  }
};

namespace qt {
double fp64_peak_tflops(int kind, int reps, cudaStream_t st);
}

namespace {

thread_local std::string g_last_error;

qt_status to_status(qt::Err c) {
  switch (c) {
    case qt::Err::shape: return QT_ERR_SHAPE;
    case qt::Err::input: return QT_ERR_INPUT;
    case qt::Err::numeric: return QT_ERR_NUMERIC;
    case qt::Err::capacity: return QT_ERR_CAPACITY;
    case qt::Err::cuda: return QT_ERR_CUDA;
    case qt::Err::nccl: return QT_ERR_NCCL;
    default: return QT_ERR_INTERNAL;
  }
}

template <typename F>
qt_status guard(F&& f) {
  try {
    f();
    return QT_OK;
  } catch (const qt::Error& e) {
    g_last_error = e.what();
    return to_status(e.code);
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return QT_ERR_INTERNAL;
  } catch (...) {
    g_last_error = "unknown error";
    return QT_ERR_INTERNAL;
  }
}

void require(bool ok, qt::Err c, const char* msg) {
  if (!ok) throw qt::Error(c, msg);
}

qt_tensor* new_tensor(qt_ctx* ctx, std::initializer_list<uint64_t> shape) {
  auto* t = new qt_tensor;
  t->ctx = ctx;
  t->rank = static_cast<int>(shape.size());
  int k = 0;
  for (uint64_t s : shape) t->shape[k++] = s;
  t->owning = true;
  const size_t bytes = std::max<size_t>(t->numel(), 1) * sizeof(double2);
  cudaError_t err = cudaMallocAsync(reinterpret_cast<void**>(&t->data), bytes, ctx->eng.stream);
  if (err != cudaSuccess) {
    cudaGetLastError();
    delete t;
    throw qt::Error(qt::Err::capacity, "device allocation of an output tensor failed");
  }
  return t;
}

void free_tensor(qt_tensor* t) {
  if (!t) return;
  if (t->owning && t->data) cudaFreeAsync(t->data, t->ctx->eng.stream);
  delete t;
}

const qt_tensor* require_tensor(const qt_tensor* t, int rank, const char* what) {
  if (!t) throw qt::Error(qt::Err::input, std::string(what) + ": null tensor");
  if (t->rank != rank) throw qt::Error(qt::Err::shape, std::string(what) + ": wrong rank");
  return t;
}

// gate tensor: (d,d,d,d) or its (d^2 x d^2) matrix view (TwoSiteGate::matrix)
void require_gate(const qt_tensor* u, uint64_t d) {
  if (!u) throw qt::Error(qt::Err::input, "gate: null tensor");
  const bool r4 = u->rank == 4 && u->shape[0] == d && u->shape[1] == d && u->shape[2] == d && u->shape[3] == d;
  const bool r2 = u->rank == 2 && u->shape[0] == d * d && u->shape[1] == d * d;
  if (!r4 && !r2) throw qt::Error(qt::Err::shape, "physical dimensions disagree");
}

// build_theta shape checks, proj/src/gates.cpp:125-131
qt::Dims gate_dims(const qt_tensor* xi, const qt_tensor* bm, const qt_tensor* bn, const qt_tensor* u) {
  if (!xi || !bm || !bn || !u) throw qt::Error(qt::Err::input, "gate update: null tensor");
  if (bm->rank != 3 || bn->rank != 3 || xi->rank != 2)
    throw qt::Error(qt::Err::shape, "gate update expects rank-3 site tensors and a bond matrix");
  const uint64_t d = bm->shape[0];
  if (bn->shape[0] != d) throw qt::Error(qt::Err::shape, "physical dimensions disagree");
  require_gate(u, d);
  if (xi->shape[1] != bm->shape[1] || bm->shape[2] != bn->shape[1])
    throw qt::Error(qt::Err::shape, "bond dimensions disagree");
  qt::Dims D;
  D.d = static_cast<long long>(d);
  D.chi_l = static_cast<long long>(xi->shape[0]);
  D.chi_m = static_cast<long long>(bm->shape[1]);
  D.chi_n = static_cast<long long>(bm->shape[2]);
  D.chi_r = static_cast<long long>(bn->shape[2]);
  if (D.d == 0 || D.chi_l == 0 || D.chi_m == 0 || D.chi_n == 0 || D.chi_r == 0)
    throw qt::Error(qt::Err::shape, "gate update: empty dimension");
  return D;
}

void fill_report(qt_report* r, uint64_t before, uint64_t expanded, uint64_t after, double eps, double disc,
                 int scheme) {
  if (!r) return;
  r->chi_before = before;
  r->chi_expanded = expanded;
  r->chi_after = after;
  r->eps_trunc = eps;
  r->discarded_weight = disc;
  r->scheme = scheme;
  r->reserved = 0;
}

// report formulas of gates.cpp:375-384 / :434-447
void report_from(const qt::HostReport& h, const qt_policy& pol, double* eps, double* disc) {
  const double theta_norm = std::sqrt(h.theta2);
  const double total2 = theta_norm * theta_norm;
  const double kept_norm = std::sqrt(h.kept2);
  *disc = std::max(0.0, total2 - kept_norm * kept_norm);
  if (pol.compute_explicit_error)
    *eps = h.theta2 == 0.0 ? 0.0 : h.resid / h.theta2;
  else
    *eps = *disc / total2;
}

struct QrOut {
  qt_tensor *b_m = nullptr, *xi = nullptr, *b_n = nullptr, *left = nullptr;
  void release() {
    free_tensor(b_m);
    free_tensor(xi);
    free_tensor(b_n);
    free_tensor(left);
    b_m = xi = b_n = left = nullptr;
  }
};

// one QR update; returns the outputs and leaves the report scalars on device
QrOut launch_qr(qt_ctx* ctx, const qt::Dims& D, const qt_tensor* xi, const qt_tensor* bm, const qt_tensor* bn,
                const qt_tensor* u, const qt_policy& pol, long long eta, bool want_left) {
  QrOut o;
  try {
    const uint64_t d = D.d;
    o.b_m = new_tensor(ctx, {d, static_cast<uint64_t>(D.chi_m), static_cast<uint64_t>(eta)});
    o.xi = new_tensor(ctx, {static_cast<uint64_t>(eta), static_cast<uint64_t>(eta)});
    o.b_n = new_tensor(ctx, {d, static_cast<uint64_t>(eta), static_cast<uint64_t>(D.chi_r)});
    if (want_left) o.left = new_tensor(ctx, {d, static_cast<uint64_t>(D.chi_l), static_cast<uint64_t>(eta)});
    qt::GateBuffers gb{o.b_m->data, o.xi->data, o.b_n->data, o.left ? o.left->data : nullptr};
    qt::gate_qr_async(ctx->eng, D, xi->data, bm->data, bn->data, u->data, pol, eta, gb);
  } catch (...) {
    o.release();
    throw;
  }
  return o;
}

qt_policy policy_or_default(const qt_policy* p) {
  qt_policy q;
  qt_policy_default(&q);
  return p ? *p : q;
}

}  // namespace

extern "C" {

const char* qt_last_error(void) { return g_last_error.c_str(); }
// internal (not in the public header): other translation units of the library
// report errors through the same thread-local string
void qt_internal_set_last_error(const char* msg) { g_last_error = msg ? msg : ""; }
const char* qt_version(void) { return "qrtebd-b200 0.1.0 (sm_100a, complex128 DMMA)"; }

void qt_policy_default(qt_policy* p) {
  if (!p) return;
  p->chi_max = 1024;
  p->sv_cutoff = 1e-14;
  p->target_eps = 0.0;
  p->delta_chi_abs = 100;
  p->delta_chi_rel = 0.1;
  p->chi_max_expansion = 0;
  p->qr_sweeps = 1;
  p->compute_explicit_error = 1;
  p->skip_renormalize = 0;
  p->reserved = 0;
}

uint64_t qt_expanded_dim(const qt_policy* p, uint64_t chi, uint64_t d) {
  const qt_policy q = policy_or_default(p);
  return qt::expanded_dim(q, chi, d);
}

uint64_t qt_kernel_launches(void) { return qt::zgemm_launch_count(); }

qt_status qt_ctx_create(int device, void* stream, qt_ctx** out) {
  return guard([&] {
    require(out != nullptr, qt::Err::input, "qt_ctx_create: null out");
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
      cudaGetLastError();
      throw qt::Error(qt::Err::cuda, "no CUDA device available (this library has no CPU fallback)");
    }
    require(device >= 0 && device < n, qt::Err::input, "qt_ctx_create: device out of range");
    cudaDeviceProp prop;
    QT_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) throw qt::Error(qt::Err::cuda, "device is not sm_100 (B200); kernels are built for sm_100a");
    auto* c = new qt_ctx;
    try {
      c->eng.init(device, static_cast<cudaStream_t>(stream));
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
      }
    } catch (...) {
      delete c;
      throw;
    }
    *out = c;
  });
}

qt_status qt_ctx_destroy(qt_ctx* ctx) {
  return guard([&] {
    if (!ctx) return;
    ctx->eng.destroy();
    delete ctx;
  });
}

qt_status qt_ctx_synchronize(qt_ctx* ctx) {
  return guard([&] {
    require(ctx != nullptr, qt::Err::input, "null context");
    QT_CUDA(cudaStreamSynchronize(ctx->eng.stream));
  });
}

void* qt_ctx_stream(qt_ctx* ctx) { return ctx ? static_cast<void*>(ctx->eng.stream) : nullptr; }

qt_status qt_ctx_set_qr_pair_min_rows(qt_ctx* ctx, int64_t rows) {
  return guard([&] {
    require(ctx != nullptr, qt::Err::input, "qt_ctx_set_qr_pair_min_rows: null context");
    ctx->eng.qr_pair_min_rows = rows < 0 ? -1 : rows;
  });
}

qt_status qt_tensor_create(qt_ctx* ctx, int rank, const uint64_t* shape, qt_tensor** out) {
  return guard([&] {
    require(ctx && out && (rank == 0 || shape), qt::Err::input, "qt_tensor_create: null argument");
    require(rank >= 0 && rank <= 4, qt::Err::shape, "qt_tensor_create: rank must be 0..4");
    auto* t = new qt_tensor;
    t->ctx = ctx;
    t->rank = rank;
    for (int k = 0; k < rank; ++k) t->shape[k] = shape[k];
    t->owning = true;
    const size_t bytes = std::max<size_t>(t->numel(), 1) * sizeof(double2);
    cudaError_t err = cudaMallocAsync(reinterpret_cast<void**>(&t->data), bytes, ctx->eng.stream);
    if (err != cudaSuccess) {
      cudaGetLastError();
      delete t;
      throw qt::Error(qt::Err::capacity, "device allocation failed");
    }
    QT_CUDA(cudaMemsetAsync(t->data, 0, bytes, ctx->eng.stream));
    *out = t;
  });
}

qt_status qt_tensor_wrap(qt_ctx* ctx, int rank, const uint64_t* shape, void* device_ptr, qt_tensor** out) {
  return guard([&] {
    require(ctx && out && device_ptr && (rank == 0 || shape), qt::Err::input, "qt_tensor_wrap: null argument");
    require(rank >= 0 && rank <= 4, qt::Err::shape, "qt_tensor_wrap: rank must be 0..4");
    require((reinterpret_cast<uintptr_t>(device_ptr) & 15) == 0, qt::Err::input, "qt_tensor_wrap: 16-byte alignment");
    auto* t = new qt_tensor;
    t->ctx = ctx;
    t->rank = rank;
    for (int k = 0; k < rank; ++k) t->shape[k] = shape[k];
    t->data = static_cast<double2*>(device_ptr);
    t->owning = false;
    *out = t;
  });
}

qt_status qt_tensor_free(qt_tensor* t) {
  return guard([&] { free_tensor(t); });
}

qt_status qt_tensor_shape(const qt_tensor* t, int* rank, uint64_t* shape4) {
  return guard([&] {
    require(t && rank && shape4, qt::Err::input, "qt_tensor_shape: null argument");
    *rank = t->rank;
    for (int k = 0; k < 4; ++k) shape4[k] = k < t->rank ? t->shape[k] : 1;
  });
}

void* qt_tensor_data(const qt_tensor* t) { return t ? t->data : nullptr; }

qt_status qt_tensor_upload(qt_tensor* t, const double* host) {
  return guard([&] {
    require(t && (host || t->numel() == 0), qt::Err::input, "qt_tensor_upload: null argument");
    QT_CUDA(cudaMemcpyAsync(t->data, host, t->numel() * sizeof(double2), cudaMemcpyHostToDevice, t->ctx->eng.stream));
    QT_CUDA(cudaStreamSynchronize(t->ctx->eng.stream));
  });
}

qt_status qt_tensor_download(const qt_tensor* t, double* host) {
  return guard([&] {
    require(t && (host || t->numel() == 0), qt::Err::input, "qt_tensor_download: null argument");
    QT_CUDA(cudaMemcpyAsync(host, t->data, t->numel() * sizeof(double2), cudaMemcpyDeviceToHost, t->ctx->eng.stream));
    QT_CUDA(cudaStreamSynchronize(t->ctx->eng.stream));
  });
}

qt_status qt_tensor_upload_async(qt_tensor* t, const double* host) {
  return guard([&] {
    require(t && (host || t->numel() == 0), qt::Err::input, "qt_tensor_upload_async: null argument");
    QT_CUDA(cudaMemcpyAsync(t->data, host, t->numel() * sizeof(double2), cudaMemcpyHostToDevice, t->ctx->eng.stream));
  });
}

qt_status qt_tensor_download_async(const qt_tensor* t, double* host) {
  return guard([&] {
    require(t && (host || t->numel() == 0), qt::Err::input, "qt_tensor_download_async: null argument");
    QT_CUDA(cudaMemcpyAsync(host, t->data, t->numel() * sizeof(double2), cudaMemcpyDeviceToHost, t->ctx->eng.stream));
  });
}

qt_status qt_tensor_copy(qt_tensor* dst, const qt_tensor* src) {
  return guard([&] {
    require(dst && src, qt::Err::input, "qt_tensor_copy: null argument");
    if (dst->numel() != src->numel())
      throw qt::Error(qt::Err::shape, "qt_tensor_copy: element counts differ (" + std::to_string(dst->numel()) +
                                          " vs " + std::to_string(src->numel()) + ")");
    QT_CUDA(cudaMemcpyAsync(dst->data, src->data, src->numel() * sizeof(double2), cudaMemcpyDeviceToDevice,
                            dst->ctx->eng.stream));
  });
}

// ---------------------------------------------------------------- linalg
qt_status qt_qr_reduced(qt_ctx* ctx, const qt_tensor* m, qt_tensor** q_out, qt_tensor** r_out) {
  return guard([&] {
    require(ctx && q_out && r_out, qt::Err::input, "qt_qr_reduced: null argument");
    require_tensor(m, 2, "qr_reduced");
    qt::Engine& e = ctx->eng;
    const long long p = m->shape[0], q = m->shape[1], k = std::min(p, q);
    int* flag = reinterpret_cast<int*>(e.dscal + qt::SC_TMP3);
    QT_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), e.stream));
    qt::check_finite(e, m->data, p * q, flag);
    int hflag = 0;
    QT_CUDA(cudaMemcpyAsync(&hflag, flag, sizeof(int), cudaMemcpyDeviceToHost, e.stream));
    QT_CUDA(cudaStreamSynchronize(e.stream));
    if (hflag) throw qt::Error(qt::Err::input, "qr_reduced: non-finite entries");
    QrOut o;
    try {
      o.b_m = new_tensor(ctx, {static_cast<uint64_t>(p), static_cast<uint64_t>(k)});
      o.xi = new_tensor(ctx, {static_cast<uint64_t>(k), static_cast<uint64_t>(q)});
      if (k > 0) {
        double2* a = e.cbuf(qt::S_MISC2, p * q);
        qt::copy2d(e, m->data, q, a, q, p, q);
        qt::qr_inplace(e, a, p, q, q, o.b_m->data, k, o.xi->data, q);
      }
      QT_CUDA(cudaStreamSynchronize(e.stream));
    } catch (...) {
      o.release();
      throw;
    }
    *q_out = o.b_m;
    *r_out = o.xi;
  });
}

qt_status qt_lq_reduced(qt_ctx* ctx, const qt_tensor* m, qt_tensor** l_out, qt_tensor** q_out) {
  return guard([&] {
    require(ctx && q_out && l_out, qt::Err::input, "qt_lq_reduced: null argument");
    require_tensor(m, 2, "lq_reduced");
    qt::Engine& e = ctx->eng;
    const long long p = m->shape[0], q = m->shape[1], k = std::min(p, q);
    int* flag = reinterpret_cast<int*>(e.dscal + qt::SC_TMP3);
    QT_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), e.stream));
    qt::check_finite(e, m->data, p * q, flag);
    int hflag = 0;
    QT_CUDA(cudaMemcpyAsync(&hflag, flag, sizeof(int), cudaMemcpyDeviceToHost, e.stream));
    QT_CUDA(cudaStreamSynchronize(e.stream));
    if (hflag) throw qt::Error(qt::Err::input, "lq_reduced: non-finite entries");
    QrOut o;
    try {
      o.b_m = new_tensor(ctx, {static_cast<uint64_t>(p), static_cast<uint64_t>(k)});  // L
      o.xi = new_tensor(ctx, {static_cast<uint64_t>(k), static_cast<uint64_t>(q)});   // Q
      if (k > 0) {
        // m = L Q  <=>  m^H = Q^H L^H  (linalg.cpp:53-64)
        double2* a = e.cbuf(qt::S_MISC2, p * q + q * k + k * p);
        double2* qq = a + p * q;
        double2* rr = qq + q * k;
        const long long shp[2] = {p, q};
        const int perm[2] = {1, 0};
        qt::permute(e, m->data, 2, shp, perm, true, a);  // (q x p)
        qt::qr_inplace(e, a, q, p, p, qq, k, rr, p);   // qq (q x k), rr (k x p)
        const long long s1[2] = {k, p};
        qt::permute(e, rr, 2, s1, perm, true, o.b_m->data);  // L = rr^H (p x k)
        const long long s2[2] = {q, k};
        qt::permute(e, qq, 2, s2, perm, true, o.xi->data);  // Q = qq^H (k x q)
      }
      QT_CUDA(cudaStreamSynchronize(e.stream));
    } catch (...) {
      o.release();
      throw;
    }
    *l_out = o.b_m;
    *q_out = o.xi;
  });
}

qt_status qt_zgemm(qt_ctx* ctx, int op_a, int op_b, int64_t m, int64_t n, int64_t k, int batch, const void* a,
                   int64_t lda, int64_t stride_a, const void* b, int64_t ldb, int64_t stride_b, void* c,
                   int64_t ldc, int64_t stride_c, double alpha, double beta) {
  return guard([&] {
    require(ctx != nullptr, qt::Err::input, "qt_zgemm: null context");
    require((op_a == 0 || op_a == 1) && (op_b == 0 || op_b == 1), qt::Err::input, "qt_zgemm: op must be 0 or 1");
    qt::GemmDesc g;
    g.M = m;
    g.N = n;
    g.K = k;
    g.batch = batch;
    g.opA = static_cast<qt::Op>(op_a);
    g.opB = static_cast<qt::Op>(op_b);
    g.A = static_cast<const double2*>(a);
    g.lda = lda;
    g.strideA = stride_a;
    g.B = static_cast<const double2*>(b);
    g.ldb = ldb;
    g.strideB = stride_b;
    g.C = static_cast<double2*>(c);
    g.ldc = ldc;
    g.strideC = stride_c;
    g.alpha = alpha;
    g.beta = beta;
    qt::zgemm(g, ctx->eng.gemm_scratch(), ctx->eng.stream);
  });
}

// ---------------------------------------------------------------- updates
qt_status qt_apply_gate_qr(qt_ctx* ctx, const qt_tensor* xi, const qt_tensor* b_m, const qt_tensor* b_n,
                           const qt_tensor* u, const qt_policy* policy, qt_tensor** b_m_out, qt_tensor** xi_out,
                           qt_tensor** b_n_out, qt_tensor** left_iso_out, qt_report* report) {
  return guard([&] {
    require(ctx && b_m_out && xi_out && b_n_out, qt::Err::input, "qt_apply_gate_qr: null argument");
    const qt_policy pol = policy_or_default(policy);
    const qt::Dims D = gate_dims(xi, b_m, b_n, u);
    const long long eta = qt::qr_eta(pol, D);
    QrOut o = launch_qr(ctx, D, xi, b_m, b_n, u, pol, eta, left_iso_out != nullptr);
    qt::HostReport h;
    try {
      h = qt::read_report(ctx->eng);
    } catch (...) {
      o.release();
      throw;
    }
    if (!h.finite) {
      o.release();
      throw qt::Error(qt::Err::input, "qr_reduced: non-finite entries");
    }
    double eps = 0, disc = 0;
    report_from(h, pol, &eps, &disc);
    fill_report(report, D.chi_n, eta, eta, eps, disc, QT_SCHEME_QR);
    *b_m_out = o.b_m;
    *xi_out = o.xi;
    *b_n_out = o.b_n;
    if (left_iso_out) *left_iso_out = o.left;
  });
}

qt_status qt_apply_gate_qr_cbe(qt_ctx* ctx, const qt_tensor* xi, const qt_tensor* b_m, const qt_tensor* b_n,
                               const qt_tensor* u, const qt_policy* policy, qt_tensor** b_m_out,
                               qt_tensor** xi_out, qt_tensor** b_n_out, qt_report* report) {
  return guard([&] {
    require(ctx && b_m_out && xi_out && b_n_out, qt::Err::input, "qt_apply_gate_qr_cbe: null argument");
    const qt_policy pol = policy_or_default(policy);
    const qt::Dims D = gate_dims(xi, b_m, b_n, u);
    QrOut o;
    qt::CbeResult res;
    try {
      res = qt::gate_cbe(ctx->eng, D, xi->data, b_m->data, b_n->data, u->data, pol, [&](long long kk) {
        const uint64_t d = D.d, k = static_cast<uint64_t>(kk);
        o.b_m = new_tensor(ctx, {d, static_cast<uint64_t>(D.chi_m), k});
        o.xi = new_tensor(ctx, {k, k});
        o.b_n = new_tensor(ctx, {d, k, static_cast<uint64_t>(D.chi_r)});
        return qt::GateBuffers{o.b_m->data, o.xi->data, o.b_n->data, nullptr};
      });
    } catch (...) {
      o.release();
      throw;
    }
    double eps = 0, disc = 0;
    report_from(res.rep, pol, &eps, &disc);
    fill_report(report, D.chi_n, res.eta, res.kk, eps, disc, QT_SCHEME_QR_CBE);
    *b_m_out = o.b_m;
    *xi_out = o.xi;
    *b_n_out = o.b_n;
  });
}

qt_status qt_apply_gate(qt_ctx* ctx, qt_scheme scheme, const qt_tensor* xi, const qt_tensor* b_m,
                        const qt_tensor* b_n, const qt_tensor* u, const qt_policy* policy, qt_tensor** b_m_out,
                        qt_tensor** xi_out, qt_tensor** b_n_out, qt_tensor** left_iso_out, qt_report* report) {
  if (scheme == QT_SCHEME_QR)
    return qt_apply_gate_qr(ctx, xi, b_m, b_n, u, policy, b_m_out, xi_out, b_n_out, left_iso_out, report);
  if (scheme == QT_SCHEME_QR_CBE) {
    if (left_iso_out) *left_iso_out = nullptr;
    return qt_apply_gate_qr_cbe(ctx, xi, b_m, b_n, u, policy, b_m_out, xi_out, b_n_out, report);
  }
  g_last_error = "scheme not available on the device (svd/eig are CPU comparators of the reference)";
  return QT_ERR_INPUT;
}

qt_status qt_truncation_error_explicit(qt_ctx* ctx, const qt_tensor* theta, const qt_tensor* left,
                                       const qt_tensor* center, const qt_tensor* right, double* out) {
  return guard([&] {
    require(ctx && theta && left && center && right && out, qt::Err::input, "null argument");
    if (theta->rank != 4 && theta->rank != 2)
      throw qt::Error(qt::Err::shape, "truncation_error_explicit expects a matrix or a rank-4 block");
    if (left->rank != 2 || center->rank != 2 || right->rank != 2)
      throw qt::Error(qt::Err::shape, "truncation_error_explicit expects matrix factors");
    const long long rows = theta->rank == 4 ? theta->shape[0] * theta->shape[1] : theta->shape[0];
    const long long cols = theta->rank == 4 ? theta->shape[2] * theta->shape[3] : theta->shape[1];
    if (static_cast<long long>(left->shape[0]) != rows || left->shape[1] != center->shape[0] ||
        center->shape[1] != right->shape[0] || static_cast<long long>(right->shape[1]) != cols)
      throw qt::Error(qt::Err::shape, "factor shapes inconsistent with theta");
    *out = qt::explicit_error(ctx->eng, theta->data, rows, cols, left->data, left->shape[1], center->data,
                              center->shape[1], right->data);
  });
}

// ---------------------------------------------------------------- tebd step
qt_status qt_tebd_step_uniform(qt_ctx* ctx, uint64_t cell_length, qt_tensor* const* sites, qt_tensor* const* bonds,
                               uint64_t n_layers, const int32_t* parity, qt_tensor* const* gates, qt_scheme scheme,
                               const qt_policy* policy, qt_tensor** sites_out, qt_tensor** bonds_out,
                               qt_bond_report* reports, uint64_t* n_reports) {
  std::vector<qt_tensor*> cur_s, cur_b;
  std::vector<bool> own_s, own_b;
  auto cleanup = [&] {
    for (size_t m = 0; m < cur_s.size(); ++m)
      if (own_s[m]) free_tensor(cur_s[m]);
    for (size_t m = 0; m < cur_b.size(); ++m)
      if (own_b[m]) free_tensor(cur_b[m]);
  };
  qt_status st = guard([&] {
    require(ctx && sites && bonds && sites_out && bonds_out && (n_layers == 0 || (parity && gates)),
            qt::Err::input, "qt_tebd_step_uniform: null argument");
    const uint64_t L = cell_length;
    if (L % 2 != 0) throw qt::Error(qt::Err::input, "uniform TEBD needs an even unit cell");
    if (scheme != QT_SCHEME_QR && scheme != QT_SCHEME_QR_CBE)
      throw qt::Error(qt::Err::input, "scheme not available on the device");
    const qt_policy pol = policy_or_default(policy);
    const uint64_t cap = n_reports ? *n_reports : 0;
    cur_s.assign(sites, sites + L);
    cur_b.assign(bonds, bonds + L);
    own_s.assign(L, false);
    own_b.assign(L, false);
    const uint64_t d = L ? cur_s[0]->shape[0] : 0;
    struct Pending {
      uint64_t bond, before, eta;
    };
    std::vector<Pending> pend;
    std::vector<qt_report> reps;
    // 8 report doubles per update: the scalars and the SC_TMP3 finiteness flag
    double* rep_dev = ctx->eng.dbuf(qt::S_REPORTS, 8 * (n_layers * (L / 2 + 1) + 1));
    for (uint64_t l = 0; l < n_layers; ++l) {
      const qt_tensor* u = gates[l];
      require_gate(u, d);
      const uint64_t start = parity[l] == 0 ? 0 : 1;
      for (uint64_t m = start; m < L; m += 2) {
        const uint64_t n = (m + 1) % L;
        const qt::Dims D = gate_dims(cur_b[m], cur_s[m], cur_s[n], u);
        qt_tensor *nbm = nullptr, *nxi = nullptr, *nbn = nullptr;
        if (scheme == QT_SCHEME_QR) {
          const long long eta = qt::qr_eta(pol, D);
          QrOut o = launch_qr(ctx, D, cur_b[m], cur_s[m], cur_s[n], u, pol, eta, false);
          // stash the report scalars of this update (no host sync inside the step)
          QT_CUDA(cudaMemcpyAsync(rep_dev + 8 * pend.size(), ctx->eng.dscal, 8 * sizeof(double),
                                  cudaMemcpyDeviceToDevice, ctx->eng.stream));
          pend.push_back({n, static_cast<uint64_t>(D.chi_n), static_cast<uint64_t>(eta)});
          nbm = o.b_m;
          nxi = o.xi;
          nbn = o.b_n;
        } else {
          QrOut o;
          qt::CbeResult res;
          try {
            res = qt::gate_cbe(ctx->eng, D, cur_b[m]->data, cur_s[m]->data, cur_s[n]->data, u->data, pol,
                               [&](long long kk) {
                                 const uint64_t k = static_cast<uint64_t>(kk);
                                 o.b_m = new_tensor(ctx, {d, static_cast<uint64_t>(D.chi_m), k});
                                 o.xi = new_tensor(ctx, {k, k});
                                 o.b_n = new_tensor(ctx, {d, k, static_cast<uint64_t>(D.chi_r)});
                                 return qt::GateBuffers{o.b_m->data, o.xi->data, o.b_n->data, nullptr};
                               });
          } catch (...) {
            o.release();
            throw;
          }
          double eps = 0, disc = 0;
          report_from(res.rep, pol, &eps, &disc);
          qt_report r;
          fill_report(&r, D.chi_n, res.eta, res.kk, eps, disc, QT_SCHEME_QR_CBE);
          pend.push_back({n, static_cast<uint64_t>(D.chi_n), static_cast<uint64_t>(res.kk)});
          reps.push_back(r);
          nbm = o.b_m;
          nxi = o.xi;
          nbn = o.b_n;
        }
        if (own_s[m]) free_tensor(cur_s[m]);
        if (own_b[n]) free_tensor(cur_b[n]);
        if (own_s[n]) free_tensor(cur_s[n]);
        cur_s[m] = nbm;
        own_s[m] = true;
        cur_b[n] = nxi;
        own_b[n] = true;
        cur_s[n] = nbn;
        own_s[n] = true;
      }
    }
    if (scheme == QT_SCHEME_QR) {
      std::vector<double> h(8 * pend.size() + 8);
      if (!pend.empty())
        QT_CUDA(cudaMemcpyAsync(h.data(), rep_dev, 8 * pend.size() * sizeof(double), cudaMemcpyDeviceToHost,
                                ctx->eng.stream));
      QT_CUDA(cudaStreamSynchronize(ctx->eng.stream));
      for (size_t i = 0; i < pend.size(); ++i) {
        qt::HostReport hr;
        hr.theta2 = h[8 * i + qt::SC_THETA2];
        hr.kept2 = h[8 * i + qt::SC_L2];
        hr.resid = h[8 * i + qt::SC_RESID];
        int fl = 0;
        std::memcpy(&fl, &h[8 * i + qt::SC_TMP3], sizeof(int));
        // require_finite_matrix, proj/src/linalg.cpp:17-21
        if (fl != 0) throw qt::Error(qt::Err::input, "qr_reduced: non-finite entries");
        double eps = 0, disc = 0;
        report_from(hr, pol, &eps, &disc);
        qt_report r;
        fill_report(&r, pend[i].before, pend[i].eta, pend[i].eta, eps, disc, QT_SCHEME_QR);
        reps.push_back(r);
      }
    }
    for (size_t i = 0; i < reps.size() && i < cap; ++i) {
      reports[i].bond = pend[i].bond;
      reports[i].report = reps[i];
    }
    if (n_reports) *n_reports = reps.size();
    // sites/bonds never updated keep sharing the caller's handle: hand out
    // copies so every output handle is owned by the caller independently
    for (uint64_t m = 0; m < L; ++m) {
      if (!own_s[m]) {
        qt_tensor* t = new_tensor(ctx, {cur_s[m]->shape[0], cur_s[m]->shape[1], cur_s[m]->shape[2]});
        QT_CUDA(cudaMemcpyAsync(t->data, cur_s[m]->data, t->numel() * sizeof(double2), cudaMemcpyDeviceToDevice,
                                ctx->eng.stream));
        cur_s[m] = t;
        own_s[m] = true;
      }
      if (!own_b[m]) {
        qt_tensor* t = new_tensor(ctx, {cur_b[m]->shape[0], cur_b[m]->shape[1]});
        QT_CUDA(cudaMemcpyAsync(t->data, cur_b[m]->data, t->numel() * sizeof(double2), cudaMemcpyDeviceToDevice,
                                ctx->eng.stream));
        cur_b[m] = t;
        own_b[m] = true;
      }
      sites_out[m] = cur_s[m];
      bonds_out[m] = cur_b[m];
    }
    own_s.assign(L, false);
    own_b.assign(L, false);
  });
  if (st != QT_OK) cleanup();
  return st;
}

// ---------------------------------------------------------------- device-resident uniform state
struct qt_uniform {
  qt_ctx* ctx = nullptr;
  qt::UniformDev* dev = nullptr;
};

qt_status qt_uniform_create(qt_ctx* ctx, uint64_t cell_length, qt_tensor* const* sites, qt_tensor* const* bonds,
                            qt_uniform** out) {
  return guard([&] {
    require(ctx && sites && bonds && out, qt::Err::input, "qt_uniform_create: null argument");
    const uint64_t L = cell_length;
    if (L == 0 || L % 2 != 0) throw qt::Error(qt::Err::input, "uniform TEBD needs an even unit cell");
    std::vector<long long> chi(L);
    std::vector<const double2*> sp(L), bp(L);
    const uint64_t d = sites[0] ? sites[0]->shape[0] : 0;
    for (uint64_t m = 0; m < L; ++m) {
      require_tensor(sites[m], 3, "uniform site");
      require_tensor(bonds[m], 2, "uniform bond");
      if (bonds[m]->shape[0] != bonds[m]->shape[1]) throw qt::Error(qt::Err::shape, "bond matrices must be square");
      chi[m] = static_cast<long long>(bonds[m]->shape[0]);
      sp[m] = sites[m]->data;
      bp[m] = bonds[m]->data;
    }
    for (uint64_t m = 0; m < L; ++m)
      if (sites[m]->shape[0] != d || static_cast<long long>(sites[m]->shape[1]) != chi[m] ||
          static_cast<long long>(sites[m]->shape[2]) != chi[(m + 1) % L])
        throw qt::Error(qt::Err::shape, "site tensor shape disagrees with the bond dimensions");
    auto* u = new qt_uniform;
    u->ctx = ctx;
    try {
      u->dev = qt::uniform_create(ctx->eng, static_cast<int>(L), static_cast<long long>(d), chi, sp, bp);
    } catch (...) {
      delete u;
      throw;
    }
    *out = u;
  });
}

qt_status qt_uniform_destroy(qt_uniform* u) {
  return guard([&] {
    if (!u) return;
    qt::uniform_destroy(u->dev);
    delete u;
  });
}

qt_status qt_uniform_step(qt_uniform* u, uint64_t n_layers, const int32_t* parity, qt_tensor* const* gates,
                          qt_scheme scheme, const qt_policy* policy, int32_t use_graph, qt_bond_report* reports,
                          uint64_t* n_reports) {
  return guard([&] {
    require(u && (n_layers == 0 || (parity && gates)), qt::Err::input, "qt_uniform_step: null argument");
    if (scheme != QT_SCHEME_QR && scheme != QT_SCHEME_QR_CBE)
      throw qt::Error(qt::Err::input, "scheme not available on the device");
    const qt_policy pol = policy_or_default(policy);
    long long shp[3];
    qt::uniform_live(u->dev, 0, 0, shp);
    std::vector<std::pair<int, const double2*>> layers;
    for (uint64_t l = 0; l < n_layers; ++l) {
      require_gate(gates[l], static_cast<uint64_t>(shp[0]));
      layers.push_back({parity[l] == 0 ? 0 : 1, gates[l]->data});
    }
    const auto recs = qt::uniform_step(u->dev, layers, scheme == QT_SCHEME_QR ? 1 : 0, pol, use_graph != 0);
    for (const auto& r : recs)
      if (!r.rep.finite) throw qt::Error(qt::Err::input, "qr_reduced: non-finite entries");
    const uint64_t cap = n_reports ? *n_reports : 0;
    for (size_t i = 0; i < recs.size() && i < cap; ++i) {
      double eps = 0, disc = 0;
      report_from(recs[i].rep, pol, &eps, &disc);
      reports[i].bond = static_cast<uint64_t>(recs[i].bond);
      fill_report(&reports[i].report, recs[i].before, recs[i].eta, recs[i].after, eps, disc, scheme);
    }
    if (n_reports) *n_reports = recs.size();
  });
}

qt_status qt_uniform_view(qt_uniform* u, int which, uint64_t m, qt_tensor** out) {
  return guard([&] {
    require(u && out && (which == 0 || which == 1), qt::Err::input, "qt_uniform_view: bad argument");
    long long shp[3] = {1, 1, 1};
    double2* p = qt::uniform_live(u->dev, which, static_cast<int>(m), shp);
    auto* t = new qt_tensor;
    t->ctx = u->ctx;
    t->rank = which == 0 ? 3 : 2;
    for (int k = 0; k < t->rank; ++k) t->shape[k] = static_cast<uint64_t>(shp[k]);
    t->data = p;
    t->owning = false;
    *out = t;
  });
}

// ---------------------------------------------------------------- observables
qt_status qt_expectation_local(qt_ctx* ctx, const qt_tensor* xi_left, const qt_tensor* b, const qt_tensor* op,
                               double* out2) {
  return guard([&] {
    require(ctx && xi_left && b && op && out2, qt::Err::input, "qt_expectation_local: null argument");
    require_tensor(b, 3, "expectation_local");
    require_tensor(xi_left, 2, "expectation_local");
    const uint64_t d = b->shape[0];
    if (op->rank != 2 || op->shape[0] != d || op->shape[1] != d)
      throw qt::Error(qt::Err::shape, "operator must be d x d");
    if (xi_left->shape[1] != b->shape[1]) throw qt::Error(qt::Err::shape, "bond dimensions disagree");
    // lambda = Xi^T conj(Xi) is (chi x chi) over Xi's column index; Xi may be
    // rectangular (the reference finite path's center matrix)
    qt::expectation_local(ctx->eng, xi_left->data, static_cast<long long>(xi_left->shape[0]),
                          static_cast<long long>(xi_left->shape[1]), b->data, static_cast<long long>(d),
                          static_cast<long long>(b->shape[2]), op->data, out2);
  });
}

qt_status qt_schmidt_values(qt_ctx* ctx, const qt_tensor* xi, double* out, uint64_t* n) {
  return guard([&] {
    require(ctx && xi && out && n, qt::Err::input, "qt_schmidt_values: null argument");
    require_tensor(xi, 2, "schmidt_values");
    qt::Engine& e = ctx->eng;
    const long long p = xi->shape[0], q = xi->shape[1], k = std::min(p, q);
    require(static_cast<uint64_t>(k) <= *n, qt::Err::capacity, "qt_schmidt_values: output too small");
    const double* s = qt::singular_values_device(e, xi->data, p, q);
    QT_CUDA(cudaMemcpyAsync(out, s, k * sizeof(double), cudaMemcpyDeviceToHost, e.stream));
    QT_CUDA(cudaStreamSynchronize(e.stream));
    *n = k;
  });
}

qt_status qt_eigh(qt_ctx* ctx, const qt_tensor* h, double* w_host, qt_tensor** v_out) {
  return guard([&] {
    require(ctx && h && w_host && v_out, qt::Err::input, "qt_eigh: null argument");
    require_tensor(h, 2, "eigh");
    if (h->shape[0] != h->shape[1]) throw qt::Error(qt::Err::shape, "eigh: matrix not square");
    qt::Engine& e = ctx->eng;
    const long long n = h->shape[0];
    // require_finite_matrix + the hermiticity check of proj/src/linalg.cpp:80-86:
    // InputError when ||h - h^H||_F > 1e-10 max(||h||_F, 1e-300)
    {
      int* flag = reinterpret_cast<int*>(e.dscal + qt::SC_TMP3);
      QT_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), e.stream));
      qt::check_finite(e, h->data, n * n, flag);
      qt::hermitian_defect(e, h->data, n, e.dscal + qt::SC_TMP0);
      QT_CUDA(cudaMemcpyAsync(e.hscal, e.dscal, 8 * sizeof(double), cudaMemcpyDeviceToHost, e.stream));
      QT_CUDA(cudaStreamSynchronize(e.stream));
      int hflag = 0;
      std::memcpy(&hflag, &e.hscal[qt::SC_TMP3], sizeof(int));
      if (hflag) throw qt::Error(qt::Err::input, "eigh: non-finite entries");
      const double defect = std::sqrt(e.hscal[qt::SC_TMP0]), nrm = std::sqrt(e.hscal[qt::SC_TMP1]);
      if (defect > 1e-10 * std::max(nrm, 1e-300))
        throw qt::Error(qt::Err::input, "eigh: matrix not hermitian within tolerance");
    }
    qt_tensor* v = new_tensor(ctx, {static_cast<uint64_t>(n), static_cast<uint64_t>(n)});
    try {
      double* w = e.dbuf(qt::S_EIG_W, n + 8);
      const qt::EighStatus* esw = qt::eigh_device(e, h->data, n, w, v->data);
      qt::EighStatus status{1, 0, 0.0, 0.0};
      QT_CUDA(cudaMemcpyAsync(w_host, w, n * sizeof(double), cudaMemcpyDeviceToHost, e.stream));
      if (esw) QT_CUDA(cudaMemcpyAsync(&status, esw, sizeof(status), cudaMemcpyDeviceToHost, e.stream));
      QT_CUDA(cudaStreamSynchronize(e.stream));
      qt::require_eigh_converged(status, n);
    } catch (...) {
      free_tensor(v);
      throw;
    }
    *v_out = v;
  });
}

qt_status qt_right_defect(qt_ctx* ctx, const qt_tensor* b, double* out) {
  return guard([&] {
    require(ctx && b && out, qt::Err::input, "qt_right_defect: null argument");
    require_tensor(b, 3, "right_defect");
    *out = qt::right_defect(ctx->eng, b->data, b->shape[0], b->shape[1], b->shape[2]);
  });
}

qt_status qt_check_isometric_uniform(qt_ctx* ctx, uint64_t cell_length, qt_tensor* const* sites,
                                     qt_tensor* const* bonds, double tol, double* right_defects,
                                     double* left_defects, double* translation_defects, double* norm_defects,
                                     qt_isometry_report* out) {
  return guard([&] {
    require(ctx && sites && bonds && out && cell_length > 0, qt::Err::input,
            "qt_check_isometric_uniform: null argument");
    const uint64_t L = cell_length;
    std::vector<const double2*> s(L), b(L);
    std::vector<long long> chi(L);
    long long d = 0;
    for (uint64_t m = 0; m < L; ++m) {
      require_tensor(sites[m], 3, "check_isometric");
      require_tensor(bonds[m], 2, "check_isometric");
      chi[m] = static_cast<long long>(bonds[m]->shape[0]);
      if (m == 0) d = static_cast<long long>(sites[0]->shape[0]);
    }
    for (uint64_t m = 0; m < L; ++m) {
      const uint64_t n = (m + 1) % L;
      if (bonds[m]->shape[1] != bonds[m]->shape[0] || static_cast<long long>(sites[m]->shape[0]) != d ||
          static_cast<long long>(sites[m]->shape[1]) != chi[m] ||
          static_cast<long long>(sites[m]->shape[2]) != chi[n])
        throw qt::Error(qt::Err::shape, "check_isometric: site/bond dimensions do not chain");
      s[m] = sites[m]->data;
      b[m] = bonds[m]->data;
    }
    const qt::IsometryParts r = qt::check_isometric_uniform(ctx->eng, d, chi, s, b);
    auto mx = [](const std::vector<double>& v) { return v.empty() ? 0.0 : *std::max_element(v.begin(), v.end()); };
    out->max_right_defect = mx(r.right);
    out->max_left_defect = mx(r.left);
    out->max_translation_defect = mx(r.translation);
    out->max_norm_defect = mx(r.norm);
    const double m = std::max(std::max(out->max_right_defect, out->max_left_defect),
                              std::max(out->max_translation_defect, out->max_norm_defect));
    out->pass = m <= tol ? 1 : 0;
    out->reserved = 0;
    for (uint64_t k = 0; k < L; ++k) {
      if (right_defects) right_defects[k] = r.right[k];
      if (left_defects) left_defects[k] = r.left[k];
      if (translation_defects) translation_defects[k] = r.translation[k];
      if (norm_defects) norm_defects[k] = r.norm[k];
    }
  });
}

qt_status qt_bond_energy(qt_ctx* ctx, const qt_tensor* xi, const qt_tensor* b_m, const qt_tensor* b_n,
                         const qt_tensor* h_bond, double* out) {
  return guard([&] {
    require(ctx && out, qt::Err::input, "qt_bond_energy: null argument");
    const qt::Dims D = gate_dims(xi, b_m, b_n, h_bond);
    *out = qt::bond_energy(ctx->eng, D, xi->data, b_m->data, b_n->data, h_bond->data);
  });
}

qt_status qt_profile_begin(qt_ctx* ctx, double min_flops) {
  return guard([&] {
    require(ctx != nullptr, qt::Err::input, "null context");
    qt::gemm_profile_begin(min_flops);
  });
}

qt_status qt_profile_end(qt_ctx* ctx, double* gemm_flops, double* gemm_ms, uint64_t* gemm_launches) {
  return guard([&] {
    require(ctx && gemm_flops && gemm_ms && gemm_launches, qt::Err::input, "null argument");
    const qt::GemmProfile p = qt::gemm_profile_end();
    *gemm_flops = p.flops;
    *gemm_ms = p.ms;
    *gemm_launches = p.launches;
  });
}

qt_status qt_fp64_peak(qt_ctx* ctx, int kind, double* tflops) {
  return guard([&] {
    require(ctx && tflops, qt::Err::input, "qt_fp64_peak: null argument");
    *tflops = qt::fp64_peak_tflops(kind, 5, ctx->eng.stream);
  });
}

}  // extern "C"

// ---------------------------------------------------------------- finite chain, reference semantics
// FiniteMPS (proj/include/qrtebd/mps.hpp:31-38) resident in HBM: site tensors
// (d, chi_l, chi_r) and the (possibly rectangular) center matrix on
// center_bond.  move_center (proj/src/mps.cpp:226-257) and the sequential
// tebd_step(FiniteMPS) (proj/src/gates.cpp:542-578) run on the device, every
// contraction on the DMMA GEMM, every QR/LQ on the blocked Householder engine.
struct qt_finite {
  qt_ctx* ctx = nullptr;
  uint64_t d = 0;
  std::vector<qt_tensor*> sites;
  qt_tensor* center = nullptr;
  uint64_t center_bond = 0;
  ~qt_finite() {
    for (qt_tensor* t : sites) free_tensor(t);
    free_tensor(center);
  }
};

namespace {

// one gauge move to the right, mps.cpp:231-240:
// M(a,i,b) = sum_q C(a,q) B(i,q,b);  QR of M ((a i) x b);  B <- Q (d,a,k);  C <- R
void finite_shift_right(qt_finite* f) {
  qt::Engine& e = f->ctx->eng;
  const uint64_t c = f->center_bond;
  qt_tensor* C = f->center;
  qt_tensor* B = f->sites[c];
  const long long p = C->shape[0], q = C->shape[1], d = B->shape[0], r = B->shape[2];
  if (static_cast<long long>(B->shape[1]) != q) throw qt::Error(qt::Err::shape, "center matrix disagrees with site");
  const long long rows = p * d, k = std::min(rows, r);
  double2* M = e.cbuf(qt::S_X, rows * r);
  {
    qt::GemmDesc g;
    g.M = p; g.N = r; g.K = q; g.batch = static_cast<int>(d);
    g.A = C->data; g.lda = q; g.strideA = 0;
    g.B = B->data; g.ldb = r; g.strideB = q * r;
    g.C = M; g.ldc = d * r; g.strideC = r;
    qt::zgemm(g, e.gemm_scratch(), e.stream);
  }
  qt_tensor* R = new_tensor(f->ctx, {static_cast<uint64_t>(k), static_cast<uint64_t>(r)});
  qt_tensor* S = nullptr;
  try {
    S = new_tensor(f->ctx, {static_cast<uint64_t>(d), static_cast<uint64_t>(p), static_cast<uint64_t>(k)});
    double2* Q = e.cbuf(qt::S_QM, rows * k);
    qt::qr_inplace(e, M, rows, r, r, Q, k, R->data, r);
    const long long shp[3] = {p, d, k};
    const int perm[3] = {1, 0, 2};
    qt::permute(e, Q, 3, shp, perm, false, S->data);  // (a,i,k) -> (i,a,k), mps.cpp:237-238
  } catch (...) {
    free_tensor(R);
    free_tensor(S);
    throw;
  }
  free_tensor(B);
  free_tensor(C);
  f->sites[c] = S;
  f->center = R;
  f->center_bond = c + 1;
}

// one gauge move to the left, mps.cpp:242-254:
// M(i,a,g) = sum_b B(i,a,b) C(b,g);  LQ of M as a x (i g);  B <- Q (d,k,g);  C <- L.
// LQ(m) = QR(m^H)^H (linalg.cpp:53-64): m^H[(i g), a] = (C^H B[i]^H)[g, a] is formed
// directly by the batched GEMM, so no transpose of M is materialized.
void finite_shift_left(qt_finite* f) {
  qt::Engine& e = f->ctx->eng;
  const uint64_t c = f->center_bond;
  qt_tensor* C = f->center;
  qt_tensor* B = f->sites[c - 1];
  const long long d = B->shape[0], a = B->shape[1], b = B->shape[2], gdim = C->shape[1];
  if (static_cast<long long>(C->shape[0]) != b) throw qt::Error(qt::Err::shape, "center matrix disagrees with site");
  const long long rows = d * gdim, k = std::min(rows, a);
  double2* MH = e.cbuf(qt::S_X, rows * a);
  {
    qt::GemmDesc g;
    g.M = gdim; g.N = a; g.K = b; g.batch = static_cast<int>(d);
    g.opA = qt::Op::H; g.A = C->data; g.lda = gdim; g.strideA = 0;
    g.opB = qt::Op::H; g.B = B->data; g.ldb = b; g.strideB = a * b;
    g.C = MH; g.ldc = a; g.strideC = gdim * a;
    qt::zgemm(g, e.gemm_scratch(), e.stream);
  }
  qt_tensor* Lt = new_tensor(f->ctx, {static_cast<uint64_t>(a), static_cast<uint64_t>(k)});
  qt_tensor* S = nullptr;
  try {
    S = new_tensor(f->ctx, {static_cast<uint64_t>(d), static_cast<uint64_t>(k), static_cast<uint64_t>(gdim)});
    double2* Qh = e.cbuf(qt::S_QM, rows * k);
    double2* Rh = e.cbuf(qt::S_RM, k * a);
    qt::qr_inplace(e, MH, rows, a, a, Qh, k, Rh, a);
    const long long s1[2] = {k, a};
    const int t2[2] = {1, 0};
    qt::permute(e, Rh, 2, s1, t2, true, Lt->data);  // L = Rh^H (a x k)
    // site[i,kk,g] = Q[kk,(i g)] = conj(Qh[(i g),kk])   (mps.cpp:251-252)
    const long long s3[3] = {d, gdim, k};
    const int p3[3] = {0, 2, 1};
    qt::permute(e, Qh, 3, s3, p3, true, S->data);
  } catch (...) {
    free_tensor(Lt);
    free_tensor(S);
    throw;
  }
  free_tensor(B);
  free_tensor(C);
  f->sites[c - 1] = S;
  f->center = Lt;
  f->center_bond = c - 1;
}

void finite_move_center(qt_finite* f, uint64_t target) {
  if (target > f->sites.size()) throw qt::Error(qt::Err::input, "center bond out of range");
  while (f->center_bond < target) finite_shift_right(f);
  while (f->center_bond > target) finite_shift_left(f);
}

qt_tensor* clone_tensor(qt_ctx* ctx, const qt_tensor* src) {
  qt_tensor* t = src->rank == 3 ? new_tensor(ctx, {src->shape[0], src->shape[1], src->shape[2]})
                                : new_tensor(ctx, {src->shape[0], src->shape[1]});
  QT_CUDA(cudaMemcpyAsync(t->data, src->data, src->numel() * sizeof(double2), cudaMemcpyDeviceToDevice,
                          ctx->eng.stream));
  return t;
}

}  // namespace

extern "C" {

qt_status qt_finite_create(qt_ctx* ctx, uint64_t n_sites, qt_tensor* const* sites, uint64_t center_bond,
                           const qt_tensor* center, qt_finite** out) {
  return guard([&] {
    require(ctx && sites && center && out, qt::Err::input, "qt_finite_create: null argument");
    if (n_sites == 0) throw qt::Error(qt::Err::input, "chain length must be positive");
    if (center_bond > n_sites) throw qt::Error(qt::Err::input, "center bond out of range");
    require_tensor(center, 2, "finite center matrix");
    const uint64_t d = sites[0] ? sites[0]->shape[0] : 0;
    for (uint64_t m = 0; m < n_sites; ++m) {
      require_tensor(sites[m], 3, "finite site");
      if (sites[m]->shape[0] != d) throw qt::Error(qt::Err::shape, "physical dimensions disagree");
      if (m + 1 < n_sites && sites[m]->shape[2] != sites[m + 1]->shape[1])
        throw qt::Error(qt::Err::shape, "bond dimensions disagree");
    }
    auto* f = new qt_finite;
    f->ctx = ctx;
    f->d = d;
    f->center_bond = center_bond;
    try {
      for (uint64_t m = 0; m < n_sites; ++m) f->sites.push_back(clone_tensor(ctx, sites[m]));
      f->center = clone_tensor(ctx, center);
    } catch (...) {
      delete f;
      throw;
    }
    *out = f;
  });
}

qt_status qt_finite_destroy(qt_finite* f) {
  return guard([&] { delete f; });
}

qt_status qt_finite_clone(const qt_finite* f, qt_finite** out) {
  return guard([&] {
    require(f && out, qt::Err::input, "qt_finite_clone: null argument");
    auto* g = new qt_finite;
    g->ctx = f->ctx;
    g->d = f->d;
    g->center_bond = f->center_bond;
    try {
      for (const qt_tensor* t : f->sites) g->sites.push_back(clone_tensor(f->ctx, t));
      g->center = clone_tensor(f->ctx, f->center);
    } catch (...) {
      delete g;
      throw;
    }
    *out = g;
  });
}

qt_status qt_finite_center_bond(const qt_finite* f, uint64_t* out) {
  return guard([&] {
    require(f && out, qt::Err::input, "qt_finite_center_bond: null argument");
    *out = f->center_bond;
  });
}

qt_status qt_finite_view(qt_finite* f, int which, uint64_t m, qt_tensor** out) {
  return guard([&] {
    require(f && out && (which == 0 || which == 1), qt::Err::input, "qt_finite_view: bad argument");
    if (which == 0 && m >= f->sites.size()) throw qt::Error(qt::Err::input, "site out of range");
    const qt_tensor* src = which == 0 ? f->sites[m] : f->center;
    auto* t = new qt_tensor;
    *t = *src;
    t->owning = false;
    *out = t;
  });
}

qt_status qt_finite_move_center(qt_finite* f, uint64_t new_center) {
  return guard([&] {
    require(f != nullptr, qt::Err::input, "qt_finite_move_center: null argument");
    finite_move_center(f, new_center);
  });
}

qt_status qt_finite_step(qt_finite* f, uint64_t n_layers, const int32_t* parity, qt_tensor* const* gates,
                         qt_scheme scheme, const qt_policy* policy, qt_bond_report* reports, uint64_t* n_reports) {
  return qt_finite_step_observed(f, n_layers, parity, gates, scheme, policy, reports, n_reports, nullptr, nullptr);
}

qt_status qt_finite_step_observed(qt_finite* f, uint64_t n_layers, const int32_t* parity, qt_tensor* const* gates,
                                  qt_scheme scheme, const qt_policy* policy, qt_bond_report* reports,
                                  uint64_t* n_reports, qt_gate_observer observer, void* user) {
  return guard([&] {
    require(f && (n_layers == 0 || (parity && gates)), qt::Err::input, "qt_finite_step: null argument");
    if (scheme != QT_SCHEME_QR && scheme != QT_SCHEME_QR_CBE)
      throw qt::Error(qt::Err::input, "scheme not available on the device");
    const qt_policy pol = policy_or_default(policy);
    qt_ctx* ctx = f->ctx;
    qt::Engine& e = ctx->eng;
    const uint64_t n = f->sites.size();
    const uint64_t nb = n > 0 ? n - 1 : 0;
    const uint64_t cap = n_reports ? *n_reports : 0;
    std::vector<qt_bond_report> out;
    struct Pending {
      uint64_t bond, before, eta;
    };
    std::vector<Pending> pend;  // QR reports whose scalars are still on the device
    constexpr int kRep = 8;  // dscal[0..7]: theta2, L2, resid, tmp0..tmp3 (the finiteness flag is SC_TMP3)
    double* rep_dev = e.dbuf(qt::S_REPORTS, kRep * (n_layers * (nb / 2 + 1) + 1));
    auto flush_qr = [&] {
      if (pend.empty()) return;
      std::vector<double> h(kRep * pend.size());
      QT_CUDA(cudaMemcpyAsync(h.data(), rep_dev, h.size() * sizeof(double), cudaMemcpyDeviceToHost, e.stream));
      QT_CUDA(cudaStreamSynchronize(e.stream));
      for (size_t i = 0; i < pend.size(); ++i) {
        qt::HostReport hr;
        hr.theta2 = h[kRep * i + qt::SC_THETA2];
        hr.kept2 = h[kRep * i + qt::SC_L2];
        hr.resid = h[kRep * i + qt::SC_RESID];
        int flag = 0;
        std::memcpy(&flag, &h[kRep * i + qt::SC_TMP3], sizeof(int));
        if (flag) throw qt::Error(qt::Err::input, "qr_reduced: non-finite entries");
        double eps = 0, disc = 0;
        report_from(hr, pol, &eps, &disc);
        qt_bond_report br;
        br.bond = pend[i].bond;
        fill_report(&br.report, pend[i].before, pend[i].eta, pend[i].eta, eps, disc, QT_SCHEME_QR);
        out.push_back(br);
      }
      pend.clear();
    };
    for (uint64_t l = 0; l < n_layers; ++l) {
      const uint64_t start = parity[l] == 0 ? 0 : 1;
      for (uint64_t m = start; m + 1 < n; m += 2) {
        const qt_tensor* u = gates[l * nb + m];
        finite_move_center(f, m);  // gates.cpp:556
        const qt::Dims D = gate_dims(f->center, f->sites[m], f->sites[m + 1], u);
        if (scheme == QT_SCHEME_QR) {
          // left_iso present: the center moves onto bond m+1 (gates.cpp:559-563)
          const long long eta = qt::qr_eta(pol, D);
          const uint64_t d = D.d;
          qt_tensor* xi = new_tensor(ctx, {static_cast<uint64_t>(eta), static_cast<uint64_t>(eta)});
          qt_tensor *bn = nullptr, *left = nullptr;
          try {
            bn = new_tensor(ctx, {d, static_cast<uint64_t>(eta), static_cast<uint64_t>(D.chi_r)});
            left = new_tensor(ctx, {d, static_cast<uint64_t>(D.chi_l), static_cast<uint64_t>(eta)});
            qt::GateBuffers gb{nullptr, xi->data, bn->data, left->data};
            qt::gate_qr_async(e, D, f->center->data, f->sites[m]->data, f->sites[m + 1]->data, u->data, pol, eta,
                              gb);
          } catch (...) {
            free_tensor(xi);
            free_tensor(bn);
            free_tensor(left);
            throw;
          }
          QT_CUDA(cudaMemcpyAsync(rep_dev + kRep * pend.size(), e.dscal, kRep * sizeof(double), cudaMemcpyDeviceToDevice,
                                  e.stream));
          pend.push_back({m + 1, static_cast<uint64_t>(D.chi_n), static_cast<uint64_t>(eta)});
          free_tensor(f->sites[m]);
          free_tensor(f->sites[m + 1]);
          free_tensor(f->center);
          f->sites[m] = left;
          f->sites[m + 1] = bn;
          f->center = xi;
          f->center_bond = m + 1;
          if (observer) flush_qr();  // the observer sees this gate's report
        } else {
          // Hastings-only scheme: the center matrix stays put; b_m is renormalized
          // by 1/sqrt(1 - eps) unless skip_renormalize (gates.cpp:564-571)
          flush_qr();
          QrOut o;
          qt::CbeResult res;
          try {
            res = qt::gate_cbe(e, D, f->center->data, f->sites[m]->data, f->sites[m + 1]->data, u->data, pol,
                               [&](long long kk) {
                                 const uint64_t k = static_cast<uint64_t>(kk), d = D.d;
                                 o.b_m = new_tensor(ctx, {d, static_cast<uint64_t>(D.chi_m), k});
                                 o.xi = new_tensor(ctx, {k, k});
                                 o.b_n = new_tensor(ctx, {d, k, static_cast<uint64_t>(D.chi_r)});
                                 return qt::GateBuffers{o.b_m->data, o.xi->data, o.b_n->data, nullptr};
                               });
          } catch (...) {
            o.release();
            throw;
          }
          double eps = 0, disc = 0;
          report_from(res.rep, pol, &eps, &disc);
          if (!pol.skip_renormalize && eps > 0.0 && eps < 1.0) {
            qt_tensor* scaled = clone_tensor(ctx, o.b_m);
            const long long cnt = static_cast<long long>(o.b_m->numel());
            const int idp[1] = {0};
            qt::permute(e, o.b_m->data, 1, &cnt, idp, false, scaled->data, 1.0 / std::sqrt(1.0 - eps));
            free_tensor(o.b_m);
            o.b_m = scaled;
          }
          qt_bond_report br;
          br.bond = m + 1;
          fill_report(&br.report, D.chi_n, res.eta, res.kk, eps, disc, QT_SCHEME_QR_CBE);
          out.push_back(br);
          free_tensor(f->sites[m]);
          free_tensor(f->sites[m + 1]);
          free_tensor(o.xi);
          o.xi = nullptr;
          f->sites[m] = o.b_m;
          f->sites[m + 1] = o.b_n;
        }
        // FiniteGateObserver, proj/include/qrtebd/gates.hpp:120-123: after
        // every gate, with the state as it stands
        if (observer && observer(user, &out.back()) != 0)
          throw qt::Error(qt::Err::internal, "gate observer failed");
      }
    }
    flush_qr();
    for (size_t i = 0; i < out.size() && i < cap; ++i) reports[i] = out[i];
    if (n_reports) *n_reports = out.size();
  });
}

/* Observables of a FiniteMPS in one left-to-right gauge sweep over a copy of
 * the state: <op> on every site (expectation_local(FiniteMPS), mps.cpp:188-196)
 * and the Schmidt values of every bond 0..n (schmidt_values(FiniteMPS),
 * mps.cpp:203-207).  z_out: 2n doubles (re, im) or NULL; schmidt_out: values of
 * bond b at offsets[b] (offsets has n+2 entries; the values are written only
 * when the capacity cap suffices, the offsets always). */
qt_status qt_finite_observables(const qt_finite* f, const qt_tensor* op, double* z_out, double* schmidt_out,
                                uint64_t cap, uint64_t* offsets) {
  qt_finite* w = nullptr;
  qt_status st = guard([&] {
    require(f != nullptr, qt::Err::input, "qt_finite_observables: null argument");
    if (op && (op->rank != 2 || op->shape[0] != f->d || op->shape[1] != f->d))
      throw qt::Error(qt::Err::shape, "operator must be d x d");
    qt_status cs = qt_finite_clone(f, &w);
    if (cs != QT_OK) throw qt::Error(qt::Err::internal, qt_last_error());
    qt::Engine& e = w->ctx->eng;
    const uint64_t n = w->sites.size();
    finite_move_center(w, 0);
    uint64_t off = 0;
    for (uint64_t b = 0; b <= n; ++b) {
      if (b > 0) finite_shift_right(w);
      const long long p = w->center->shape[0], q = w->center->shape[1], k = std::min(p, q);
      if (offsets) offsets[b] = off;
      if (schmidt_out && off + k <= cap) {
        const double* s = qt::singular_values_device(e, w->center->data, p, q);
        QT_CUDA(cudaMemcpyAsync(schmidt_out + off, s, k * sizeof(double), cudaMemcpyDeviceToHost, e.stream));
        QT_CUDA(cudaStreamSynchronize(e.stream));
      }
      off += k;
      if (b < n && op && z_out) {
        const qt_tensor* B = w->sites[b];
        qt::expectation_local(e, w->center->data, p, q, B->data, static_cast<long long>(f->d),
                              static_cast<long long>(B->shape[2]), op->data, z_out + 2 * b);
      }
    }
    if (offsets) offsets[n + 1] = off;
  });
  delete w;
  return st;
}

qt_status qt_left_defect(qt_ctx* ctx, const qt_tensor* b, double* out) {
  return guard([&] {
    require(ctx && b && out, qt::Err::input, "qt_left_defect: null argument");
    require_tensor(b, 3, "left_defect");
    *out = qt::left_defect(ctx->eng, b->data, b->shape[0], b->shape[1], b->shape[2]);
  });
}

qt_status qt_check_isometric_finite(const qt_finite* f, double tol, double* right_defects, double* left_defects,
                                    double* norm_defect, qt_isometry_report* out) {
  return guard([&] {
    require(f && out, qt::Err::input, "qt_check_isometric_finite: null argument");
    qt::Engine& e = f->ctx->eng;
    const uint64_t n = f->sites.size();
    double mr = 0.0, ml = 0.0;
    for (uint64_t s = 0; s < n; ++s) {
      const qt_tensor* b = f->sites[s];
      double r = 0.0, l = 0.0;
      if (s < f->center_bond)
        l = qt::left_defect(e, b->data, b->shape[0], b->shape[1], b->shape[2]);
      else
        r = qt::right_defect(e, b->data, b->shape[0], b->shape[1], b->shape[2]);
      if (right_defects) right_defects[s] = r;
      if (left_defects) left_defects[s] = l;
      mr = std::max(mr, r);
      ml = std::max(ml, l);
    }
    qt::norm2(e, f->center->data, f->center->shape[0], f->center->shape[1], f->center->shape[1],
              e.dscal + qt::SC_TMP2);
    double n2 = 0.0;
    QT_CUDA(cudaMemcpyAsync(&n2, e.dscal + qt::SC_TMP2, sizeof(double), cudaMemcpyDeviceToHost, e.stream));
    QT_CUDA(cudaStreamSynchronize(e.stream));
    const double nd = std::abs(std::sqrt(n2) - 1.0);
    if (norm_defect) *norm_defect = nd;
    out->max_right_defect = mr;
    out->max_left_defect = ml;
    out->max_translation_defect = 0.0;
    out->max_norm_defect = nd;
    out->pass = std::max(std::max(mr, ml), nd) <= tol ? 1 : 0;
    out->reserved = 0;
  });
}

}  // extern "C"
