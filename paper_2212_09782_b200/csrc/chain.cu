// Sharded finite chain in Hastings form behind
// the C-ABI: qt_chain_* and qt_tebd_step_finite_sharded (include/qrtebd_c.h).
//
// The chain of n sites is cut into contiguous, even-aligned site blocks, one
// per rank (process, one GPU each).  A layer of parity P updates the bonds
// (m, m+1) with m = P (mod 2) -- all independent (proj/tests/test_tebd.cc:
// 139-175), so each rank updates its interior bonds concurrently on worker
// contexts (own stream + workspace each, one host thread each) and only the
// bond that straddles a block boundary needs its neighbour: the right rank
// sends its first site tensor B[e] to the left rank, which runs the update
// and returns Xi[e] and B[e].  Everything else stays in HBM.
// The exchange is ncclSend / ncclRecv of raw device buffers inside
// ncclGroupStart / ncclGroupEnd on a dedicated stream, posted before the
// interior bonds are enqueued; shapes travel first in an 8-word header.
//
// The transport is an interface: NCCL across processes, or an in-process
// loopback (qt_loopback_*: device copies and events between chains of one
// process, one host thread per rank) that runs the same orchestration on one
// GPU for the multi-rank tests.  Results are committed in bond order, so a
// sharded step is bitwise the single-rank step.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/qrtebd_c.h"
#include "common.cuh"

struct qt_loopback;

// the C-ABI's thread-local last-error string (capi.cu)
extern "C" void qt_internal_set_last_error(const char* msg);

namespace {

struct ChainError : std::runtime_error {
  qt_status code;
  ChainError(qt_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void ok(qt_status s) {
  if (s != QT_OK) throw ChainError(s, qt_last_error());
}
void cuda_ok(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw ChainError(QT_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
// NCCL is resolved at first use (dlopen of libnccl.so.2), not at load time:
// a process that imports torch after this library must still get torch's own
// NCCL build, and when torch is already loaded the same soname resolves to
// its copy -- one NCCL per process either way
struct Nccl {
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
};

const Nccl& nccl() {
  static const Nccl n = [] {
    Nccl x;
    // 1. an NCCL already in the process (torch's), 2. QRTEBD_NCCL_LIB (the
    // Python binding points it at torch's bundled build, so that a later
    // `import torch` finds the same soname satisfied), 3. the system library
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    const char* env = std::getenv("QRTEBD_NCCL_LIB");
    if (!h && env && *env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) throw ChainError(QT_ERR_NCCL, std::string("cannot load libnccl.so.2: ") + dlerror());
    auto sym = [&](const char* name) {
      void* p = dlsym(h, name);
      if (!p) throw ChainError(QT_ERR_NCCL, std::string("libnccl.so.2 lacks ") + name);
      return p;
    };
    x.get_unique_id = reinterpret_cast<decltype(x.get_unique_id)>(sym("ncclGetUniqueId"));
    x.comm_init_rank = reinterpret_cast<decltype(x.comm_init_rank)>(sym("ncclCommInitRank"));
    x.comm_destroy = reinterpret_cast<decltype(x.comm_destroy)>(sym("ncclCommDestroy"));
    x.group_start = reinterpret_cast<decltype(x.group_start)>(sym("ncclGroupStart"));
    x.group_end = reinterpret_cast<decltype(x.group_end)>(sym("ncclGroupEnd"));
    x.send = reinterpret_cast<decltype(x.send)>(sym("ncclSend"));
    x.recv = reinterpret_cast<decltype(x.recv)>(sym("ncclRecv"));
    x.error_string = reinterpret_cast<decltype(x.error_string)>(sym("ncclGetErrorString"));
    return x;
  }();
  return n;
}

void nccl_ok(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw ChainError(QT_ERR_NCCL, std::string(what) + ": " + nccl().error_string(r));
}

// ---------------------------------------------------------------- transports
struct Transport {
  virtual ~Transport() = default;
  virtual void group_start() = 0;
  virtual void send(const void* buf, size_t bytes, int peer) = 0;
  virtual void recv(void* buf, size_t bytes, int peer) = 0;
  virtual void group_end(cudaStream_t st) = 0;
};

struct NcclTransport : Transport {
  ncclComm_t comm = nullptr;
  cudaStream_t st_ = nullptr;
  struct Op {
    bool is_send;
    void* buf;
    size_t bytes;
    int peer;
  };
  std::vector<Op> ops;
  ~NcclTransport() override {
    if (comm) nccl().comm_destroy(comm);
  }
  void group_start() override { ops.clear(); }
  void send(const void* buf, size_t bytes, int peer) override { ops.push_back({true, const_cast<void*>(buf), bytes, peer}); }
  void recv(void* buf, size_t bytes, int peer) override { ops.push_back({false, buf, bytes, peer}); }
  void group_end(cudaStream_t st) override {
    nccl_ok(nccl().group_start(), "ncclGroupStart");
    for (const Op& o : ops) {
      if (o.is_send)
        nccl_ok(nccl().send(o.buf, o.bytes, ncclUint8, o.peer, comm, st), "ncclSend");
      else
        nccl_ok(nccl().recv(o.buf, o.bytes, ncclUint8, o.peer, comm, st), "ncclRecv");
    }
    nccl_ok(nccl().group_end(), "ncclGroupEnd");
    ops.clear();
  }
};

}  // namespace

// In-process loopback: FIFO mailboxes per (src, dst); a send publishes the
// buffer with a ready event, the receiver's stream waits for it and copies,
// and publishes a done event that the sender's stream waits on (so the send
// buffer stays valid until the copy completed, as with NCCL)
struct qt_loopback {
  int world = 0;
  struct Msg {
    const void* buf;
    size_t bytes;
    cudaEvent_t ready;
    cudaEvent_t done;
    bool done_set = false;
  };
  std::mutex mu;
  std::condition_variable cv;
  std::map<std::pair<int, int>, std::deque<std::shared_ptr<Msg>>> box;
};

namespace {

struct LoopbackTransport : Transport {
  qt_loopback* lb;
  int rank;
  struct Op {
    bool is_send;
    void* buf;
    size_t bytes;
    int peer;
  };
  std::vector<Op> ops;
  LoopbackTransport(qt_loopback* l, int r) : lb(l), rank(r) {}
  void group_start() override { ops.clear(); }
  void send(const void* buf, size_t bytes, int peer) override { ops.push_back({true, const_cast<void*>(buf), bytes, peer}); }
  void recv(void* buf, size_t bytes, int peer) override { ops.push_back({false, buf, bytes, peer}); }
  void group_end(cudaStream_t st) override {
    std::vector<std::shared_ptr<qt_loopback::Msg>> mine;
    // 1. publish every send (non-blocking)
    for (const Op& o : ops) {
      if (!o.is_send) continue;
      auto m = std::make_shared<qt_loopback::Msg>();
      m->buf = o.buf;
      m->bytes = o.bytes;
      cuda_ok(cudaEventCreateWithFlags(&m->ready, cudaEventDisableTiming), "cudaEventCreate");
      cuda_ok(cudaEventCreateWithFlags(&m->done, cudaEventDisableTiming), "cudaEventCreate");
      cuda_ok(cudaEventRecord(m->ready, st), "cudaEventRecord");
      {
        std::lock_guard<std::mutex> g(lb->mu);
        lb->box[{rank, o.peer}].push_back(m);
      }
      mine.push_back(m);
    }
    lb->cv.notify_all();
    // 2. receive: wait for the matching send, copy behind its ready event
    for (const Op& o : ops) {
      if (o.is_send) continue;
      std::shared_ptr<qt_loopback::Msg> m;
      {
        std::unique_lock<std::mutex> g(lb->mu);
        auto& q = lb->box[{o.peer, rank}];
        lb->cv.wait(g, [&] { return !q.empty(); });
        m = q.front();
        q.pop_front();
      }
      if (m->bytes != o.bytes) throw ChainError(QT_ERR_INTERNAL, "loopback: message size mismatch");
      cuda_ok(cudaStreamWaitEvent(st, m->ready, 0), "cudaStreamWaitEvent");
      cuda_ok(cudaMemcpyAsync(o.buf, m->buf, o.bytes, cudaMemcpyDeviceToDevice, st), "cudaMemcpyAsync");
      cuda_ok(cudaEventRecord(m->done, st), "cudaEventRecord");
      {
        std::lock_guard<std::mutex> g(lb->mu);
        m->done_set = true;
      }
      lb->cv.notify_all();
    }
    // 3. the sender's stream waits until its buffers have been copied
    for (auto& m : mine) {
      {
        std::unique_lock<std::mutex> g(lb->mu);
        lb->cv.wait(g, [&] { return m->done_set; });
      }
      cuda_ok(cudaStreamWaitEvent(st, m->done, 0), "cudaStreamWaitEvent");
    }
    cuda_ok(cudaStreamSynchronize(st), "cudaStreamSynchronize");
    for (auto& m : mine) {
      cudaEventDestroy(m->ready);
      cudaEventDestroy(m->done);
    }
    ops.clear();
  }
};

// contiguous even-aligned blocks of whole (even, odd) site pairs
void partition(uint64_t n, int world, int rank, uint64_t* b, uint64_t* e) {
  const uint64_t pairs = n / 2;
  const uint64_t w = std::max<uint64_t>(1, std::min<uint64_t>(static_cast<uint64_t>(world), std::max<uint64_t>(pairs, 1)));
  const uint64_t base = pairs / w, extra = pairs % w;
  uint64_t start = 0;
  for (uint64_t r = 0; r < static_cast<uint64_t>(rank); ++r) start += 2 * (base + (r < extra ? 1 : 0));
  uint64_t len = 2 * (base + (static_cast<uint64_t>(rank) < extra ? 1 : 0));
  if (static_cast<uint64_t>(rank) >= w) {
    start = n;
    len = 0;
  }
  uint64_t end = start + len;
  if (static_cast<uint64_t>(rank) + 1 == w) end = n;  // an odd last site joins the last block
  *b = start;
  *e = end;
}

}  // namespace

struct qt_chain {
  qt_ctx* ctx = nullptr;
  int rank = 0, world = 1;
  uint64_t n = 0, begin = 0, end = 0;
  std::vector<qt_tensor*> sites;  // sites[m - begin]
  std::vector<qt_tensor*> bonds;  // bonds[m - begin]: the bond matrix left of site m
  std::vector<qt_ctx*> workers;
  // the straddling bond's context: configured like the workers, so that every
  // bond runs the same code path on every rank (bitwise the one-rank chain)
  qt_ctx* edge = nullptr;
  cudaStream_t comm_stream = nullptr;
  std::unique_ptr<Transport> tr;
  // device scratch: headers (8 int64 each: out / in)
  int64_t* hdr = nullptr;
  ~qt_chain() {
    for (qt_tensor* t : sites) qt_tensor_free(t);
    for (qt_tensor* t : bonds) qt_tensor_free(t);
    for (qt_ctx* w : workers) qt_ctx_destroy(w);
    if (edge) qt_ctx_destroy(edge);
    if (hdr) cudaFree(hdr);
    tr.reset();
    if (comm_stream) cudaStreamDestroy(comm_stream);
  }
};

namespace {

qt_status guard_chain(const std::function<void()>& f) {
  try {
    f();
    return QT_OK;
  } catch (const ChainError& e) {
    qt_internal_set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    qt_internal_set_last_error(e.what());
    return QT_ERR_INTERNAL;
  }
}

std::vector<uint64_t> shape_of(const qt_tensor* t) {
  int r = 0;
  uint64_t s4[4];
  ok(qt_tensor_shape(t, &r, s4));
  return std::vector<uint64_t>(s4, s4 + r);
}

size_t bytes_of(const std::vector<uint64_t>& s) {
  size_t n = 16;
  for (uint64_t x : s) n *= x;
  return n;
}

qt_tensor* empty_like_shape(qt_ctx* ctx, const std::vector<uint64_t>& s) {
  qt_tensor* t = nullptr;
  ok(qt_tensor_create(ctx, static_cast<int>(s.size()), s.data(), &t));
  return t;
}

qt_tensor* clone(qt_ctx* ctx, const qt_tensor* src) {
  qt_tensor* t = empty_like_shape(ctx, shape_of(src));
  ok(qt_tensor_copy(t, src));
  return t;
}

struct Upd {
  qt_tensor *bm = nullptr, *xi = nullptr, *bn = nullptr;
  qt_report rep{};
};

Upd update_on(qt_ctx* c, qt_scheme scheme, const qt_tensor* xi, const qt_tensor* bm, const qt_tensor* bn,
              const qt_tensor* u, const qt_policy* pol) {
  Upd r;
  ok(qt_apply_gate(c, scheme, xi, bm, bn, u, pol, &r.bm, &r.xi, &r.bn, nullptr, &r.rep));
  return r;
}

// header exchange (8 int64 words) + host synchronization: the payload sizes
void exchange_headers(qt_chain* c, int send_peer, const int64_t* out8, int recv_peer, int64_t* in8) {
  int64_t* dout = c->hdr;
  int64_t* din = c->hdr + 8;
  if (send_peer >= 0)
    cuda_ok(cudaMemcpyAsync(dout, out8, 8 * sizeof(int64_t), cudaMemcpyHostToDevice, c->comm_stream), "hdr h2d");
  c->tr->group_start();
  if (send_peer >= 0) c->tr->send(dout, 8 * sizeof(int64_t), send_peer);
  if (recv_peer >= 0) c->tr->recv(din, 8 * sizeof(int64_t), recv_peer);
  c->tr->group_end(c->comm_stream);
  if (recv_peer >= 0)
    cuda_ok(cudaMemcpyAsync(in8, din, 8 * sizeof(int64_t), cudaMemcpyDeviceToHost, c->comm_stream), "hdr d2h");
  cuda_ok(cudaStreamSynchronize(c->comm_stream), "comm sync");
}

void put_shape(int64_t* h, int slot, const std::vector<uint64_t>& s) {
  for (int k = 0; k < 3; ++k) h[4 * slot + k] = k < static_cast<int>(s.size()) ? static_cast<int64_t>(s[k]) : 0;
  h[4 * slot + 3] = static_cast<int64_t>(s.size());
}
std::vector<uint64_t> get_shape(const int64_t* h, int slot) {
  std::vector<uint64_t> s;
  for (int k = 0; k < h[4 * slot + 3]; ++k) s.push_back(static_cast<uint64_t>(h[4 * slot + k]));
  return s;
}

}  // namespace

extern "C" {

qt_status qt_nccl_get_unique_id(uint8_t* id128) {
  return guard_chain([&] {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    ncclUniqueId id;
    nccl_ok(nccl().get_unique_id(&id), "ncclGetUniqueId");
    std::memcpy(id128, &id, 128);
  });
}

qt_status qt_nccl_selftest(int device, uint64_t bytes, int* ok_out) {
  // one-rank NCCL communicator, a grouped send + recv to itself on a stream,
  // byte-compared: exercises the runtime-resolved NCCL (dlopen), communicator
  // setup and the grouped point-to-point path the chain uses, on one GPU
  return guard_chain([&] {
    if (!ok_out) throw ChainError(QT_ERR_INPUT, "null argument");
    cuda_ok(cudaSetDevice(device), "cudaSetDevice");
    ncclUniqueId id;
    nccl_ok(nccl().get_unique_id(&id), "ncclGetUniqueId");
    NcclTransport t;
    nccl_ok(nccl().comm_init_rank(&t.comm, 1, id, 0), "ncclCommInitRank");
    cudaStream_t st = nullptr;
    cuda_ok(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "cudaStreamCreate");
    uint8_t *src = nullptr, *dst = nullptr;
    cuda_ok(cudaMalloc(&src, bytes), "cudaMalloc");
    cuda_ok(cudaMalloc(&dst, bytes), "cudaMalloc");
    std::vector<uint8_t> h(bytes), back(bytes, 0);
    for (uint64_t i = 0; i < bytes; ++i) h[i] = static_cast<uint8_t>((i * 131 + 7) & 0xff);
    cuda_ok(cudaMemcpy(src, h.data(), bytes, cudaMemcpyHostToDevice), "h2d");
    cuda_ok(cudaMemset(dst, 0, bytes), "memset");
    t.group_start();
    t.send(src, bytes, 0);
    t.recv(dst, bytes, 0);
    t.group_end(st);
    cuda_ok(cudaStreamSynchronize(st), "sync");
    cuda_ok(cudaMemcpy(back.data(), dst, bytes, cudaMemcpyDeviceToHost), "d2h");
    *ok_out = std::memcmp(h.data(), back.data(), bytes) == 0 ? 1 : 0;
    cudaFree(src);
    cudaFree(dst);
    cudaStreamDestroy(st);
  });
}

qt_status qt_loopback_create(int world, qt_loopback** out) {
  return guard_chain([&] {
    auto* l = new qt_loopback;
    l->world = world;
    *out = l;
  });
}

qt_status qt_loopback_destroy(qt_loopback* l) {
  delete l;
  return QT_OK;
}

qt_status qt_chain_partition(uint64_t n_sites, int world, int rank, uint64_t* begin, uint64_t* end) {
  return guard_chain([&] {
    if (world < 1 || rank < 0 || rank >= world) throw ChainError(QT_ERR_INPUT, "bad rank / world");
    partition(n_sites, world, rank, begin, end);
  });
}

qt_status qt_chain_create(qt_ctx* ctx, uint64_t n_sites, int rank, int world, const uint8_t* nccl_id,
                          qt_loopback* loopback, qt_tensor* const* sites, qt_tensor* const* bonds, int n_workers,
                          qt_chain** out) {
  return guard_chain([&] {
    if (!ctx || !out || !sites || !bonds) throw ChainError(QT_ERR_INPUT, "qt_chain_create: null argument");
    if (world < 1 || rank < 0 || rank >= world) throw ChainError(QT_ERR_INPUT, "bad rank / world");
    cuda_ok(cudaDeviceSynchronize(), "cudaDeviceSynchronize");  // the caller's tensors may come from any stream
    auto c = std::make_unique<qt_chain>();
    c->ctx = ctx;
    c->rank = rank;
    c->world = world;
    c->n = n_sites;
    partition(n_sites, world, rank, &c->begin, &c->end);
    for (uint64_t m = c->begin; m < c->end; ++m) {
      c->sites.push_back(clone(ctx, sites[m - c->begin]));
      c->bonds.push_back(clone(ctx, bonds[m - c->begin]));
    }
    int dev = 0;
    cuda_ok(cudaGetDevice(&dev), "cudaGetDevice");
    for (int w = 0; w < std::max(0, n_workers); ++w) {
      qt_ctx* wc = nullptr;
      ok(qt_ctx_create(dev, nullptr, &wc));
      // bond updates side by side: the pair's side streams cost more than they hide
      ok(qt_ctx_set_qr_pair_min_rows(wc, 256));
      c->workers.push_back(wc);
    }
    if (n_workers > 0) {
      ok(qt_ctx_create(dev, nullptr, &c->edge));
      ok(qt_ctx_set_qr_pair_min_rows(c->edge, 256));
    }
    cuda_ok(cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking), "cudaStreamCreate");
    cuda_ok(cudaMalloc(&c->hdr, 16 * sizeof(int64_t)), "cudaMalloc");
    if (world > 1) {
      if (loopback) {
        c->tr = std::make_unique<LoopbackTransport>(loopback, rank);
      } else {
        if (!nccl_id) throw ChainError(QT_ERR_INPUT, "qt_chain_create: world > 1 needs an NCCL id or a loopback");
        auto t = std::make_unique<NcclTransport>();
        ncclUniqueId id;
        std::memcpy(&id, nccl_id, 128);
        nccl_ok(nccl().comm_init_rank(&t->comm, world, id, rank), "ncclCommInitRank");
        c->tr = std::move(t);
      }
    }
    ok(qt_ctx_synchronize(ctx));
    *out = c.release();
  });
}

qt_status qt_chain_destroy(qt_chain* c) {
  if (c) {
    qt_ctx_synchronize(c->ctx);
    delete c;
  }
  return QT_OK;
}

qt_status qt_chain_range(const qt_chain* c, uint64_t* begin, uint64_t* end) {
  if (!c) return QT_ERR_INPUT;
  *begin = c->begin;
  *end = c->end;
  return QT_OK;
}

qt_status qt_chain_view(qt_chain* c, int which, uint64_t m, qt_tensor** out) {
  return guard_chain([&] {
    if (!c || !out || m < c->begin || m >= c->end) throw ChainError(QT_ERR_INPUT, "qt_chain_view: site not owned");
    const qt_tensor* src = which == 0 ? c->sites[m - c->begin] : c->bonds[m - c->begin];
    const std::vector<uint64_t> s = shape_of(src);
    ok(qt_tensor_wrap(c->ctx, static_cast<int>(s.size()), s.data(), qt_tensor_data(src), out));
  });
}

qt_status qt_tebd_step_finite_sharded(qt_chain* c, uint64_t n_layers, const int32_t* parity, qt_tensor* const* gates,
                                      qt_scheme scheme, const qt_policy* policy, qt_bond_report* reports,
                                      uint64_t* n_reports) {
  return guard_chain([&] {
    if (!c || (n_layers > 0 && (!parity || !gates))) throw ChainError(QT_ERR_INPUT, "null argument");
    const uint64_t n = c->n, b = c->begin, e = c->end, nb = n > 0 ? n - 1 : 0;
    const uint64_t cap = n_reports ? *n_reports : 0;
    std::vector<qt_bond_report> out;
    auto site = [&](uint64_t m) -> qt_tensor*& { return c->sites[m - b]; };
    auto bond = [&](uint64_t m) -> qt_tensor*& { return c->bonds[m - b]; };
    for (uint64_t l = 0; l < n_layers; ++l) {
      const uint64_t P = parity[l] == 0 ? 0 : 1;
      const auto gate = [&](uint64_t m) { return gates[l * nb + m]; };
      // straddling bonds of this parity: (b-1, b) on the left, (e-1, e) on the right
      const bool left = c->world > 1 && b > 0 && b < e && (b - 1) % 2 == P;
      const bool right = c->world > 1 && e < n && e > b && (e - 1) % 2 == P;
      const int lpeer = c->rank - 1, rpeer = c->rank + 1;
      // 1. headers, then payload: B[b] -> left, B[e] <- right (posted first)
      qt_tensor* rsite = nullptr;
      if (left || right) {
        int64_t ho[8] = {0}, hi[8] = {0};
        if (left) put_shape(ho, 0, shape_of(site(b)));
        exchange_headers(c, left ? lpeer : -1, ho, right ? rpeer : -1, hi);
        if (right) {
          rsite = empty_like_shape(c->ctx, get_shape(hi, 0));
          ok(qt_ctx_synchronize(c->ctx));  // stream-ordered allocation complete before the comm stream writes it
        }
        c->tr->group_start();
        if (left) c->tr->send(qt_tensor_data(site(b)), bytes_of(shape_of(site(b))), lpeer);
        if (right) c->tr->recv(qt_tensor_data(rsite), bytes_of(shape_of(rsite)), rpeer);
        c->tr->group_end(c->comm_stream);
      }
      // 2. interior bonds, concurrently on the workers (committed in bond order)
      std::vector<uint64_t> inner;
      for (uint64_t m = b + ((b % 2 == P) ? 0 : 1); m + 1 < e; m += 2) inner.push_back(m);
      std::vector<Upd> res(inner.size());
      const size_t K = std::min(c->workers.size(), inner.size());
      if (K > 1) {
        std::vector<std::thread> th;
        std::vector<std::exception_ptr> err(K);
        for (size_t t = 0; t < K; ++t)
          th.emplace_back([&, t] {
            try {
              for (size_t i = t; i < inner.size(); i += K) {
                const uint64_t m = inner[i];
                res[i] = update_on(c->workers[t], scheme, bond(m), site(m), site(m + 1), gate(m), policy);
              }
            } catch (...) {
              err[t] = std::current_exception();
            }
          });
        for (auto& x : th) x.join();
        for (auto& x : err)
          if (x) std::rethrow_exception(x);
      } else {
        qt_ctx* ic = c->workers.empty() ? c->ctx : c->workers[0];
        for (size_t i = 0; i < inner.size(); ++i) {
          const uint64_t m = inner[i];
          res[i] = update_on(ic, scheme, bond(m), site(m), site(m + 1), gate(m), policy);
        }
      }
      for (size_t i = 0; i < inner.size(); ++i) {
        const uint64_t m = inner[i];
        qt_tensor_free(site(m));
        qt_tensor_free(bond(m + 1));
        qt_tensor_free(site(m + 1));
        site(m) = res[i].bm;
        bond(m + 1) = res[i].xi;
        site(m + 1) = res[i].bn;
        out.push_back({m + 1, res[i].rep});
      }
      // 3. the right straddling bond (e-1, e): updated here, Xi[e], B[e] returned
      qt_tensor *rxi = nullptr, *rbn = nullptr;
      if (right) {
        cuda_ok(cudaStreamSynchronize(c->comm_stream), "comm sync");  // B[e] arrived
        ok(qt_ctx_synchronize(c->ctx));
        qt_ctx* ec = c->edge ? c->edge : c->ctx;
        Upd u = update_on(ec, scheme, bond(e - 1), site(e - 1), rsite, gate(e - 1), policy);
        qt_tensor_free(site(e - 1));
        site(e - 1) = u.bm;
        rxi = u.xi;
        rbn = u.bn;
        out.push_back({e, u.rep});
        ok(qt_ctx_synchronize(c->ctx));
      }
      if (left || right) {
        int64_t ho[8] = {0}, hi[8] = {0};
        if (right) {
          put_shape(ho, 0, shape_of(rxi));
          put_shape(ho, 1, shape_of(rbn));
        }
        exchange_headers(c, right ? rpeer : -1, ho, left ? lpeer : -1, hi);
        qt_tensor *lxi = nullptr, *lbn = nullptr;
        if (left) {
          lxi = empty_like_shape(c->ctx, get_shape(hi, 0));
          lbn = empty_like_shape(c->ctx, get_shape(hi, 1));
          ok(qt_ctx_synchronize(c->ctx));
        }
        c->tr->group_start();
        if (right) {
          c->tr->send(qt_tensor_data(rxi), bytes_of(shape_of(rxi)), rpeer);
          c->tr->send(qt_tensor_data(rbn), bytes_of(shape_of(rbn)), rpeer);
        }
        if (left) {
          c->tr->recv(qt_tensor_data(lxi), bytes_of(shape_of(lxi)), lpeer);
          c->tr->recv(qt_tensor_data(lbn), bytes_of(shape_of(lbn)), lpeer);
        }
        c->tr->group_end(c->comm_stream);
        cuda_ok(cudaStreamSynchronize(c->comm_stream), "comm sync");
        if (left) {
          qt_tensor_free(bond(b));
          qt_tensor_free(site(b));
          bond(b) = lxi;
          site(b) = lbn;
        }
        qt_tensor_free(rxi);
        qt_tensor_free(rbn);
        qt_tensor_free(rsite);
      }
    }
    ok(qt_ctx_synchronize(c->ctx));
    for (size_t i = 0; i < out.size() && i < cap; ++i) reports[i] = out[i];
    if (n_reports) *n_reports = out.size();
  });
}

}  // extern "C"
