// Device-resident engine state: stream, grow-only scratch arena, device
// scalars and the host-visible pinned mirror used for reports.
#pragma once

#include <cuda_runtime.h>

#include <functional>
#include <vector>

#include "common.cuh"
#include "zgemm.cuh"

namespace qt {

enum Slot : int {
  S_PHI = 0,
  S_PHIEV,
  S_THETA,
  S_Y0,
  S_X,
  S_QM,
  S_RM,
  S_YH,
  S_QP,
  S_RP,
  S_W,
  S_QR_V,
  S_QR_T,
  S_QR_W,
  S_QR_W2,
  S_QR_PART,
  S_GEMM_PART,
  S_TILE_SUMS,
  S_NORM_PART,
  S_GRAM,
  S_EIG_V,
  S_EIG_W,
  S_MISC,
  S_MISC2,
  S_REPORTS,
  S_QA_W,        // W = V^H C of the reflector application to a second matrix (QrOpts::capply)
  S_QA_W2,
  S_GEMM_PART2,  // split-K partials of GEMMs on the second side stream
  S_TILE_SUMS2,
  S_QT_PART,     // partial sums of the Q^H theta residual
  S_QR_V2,       // reflectors / T factors of the second QR of a pipelined pair
  S_QR_T2,
  S_GEMM_PART3,  // split-K scratch of GEMMs on side4 (consumers of the pair's Q blocks)
  S_QR_WS,       // W / W2 of the QR look-ahead's wide updates on e.side (GEMM path)
  S_QR_WS2,
  S_GEMM_PARTS,  // split-K scratch of GEMMs on e.side
  S_TILE_SUMSS,
  S_TILE_SUMS3,
  S_QR_TOB,      // combined T factors of the outer (multi-panel) blocks of a tall QR
  S_QR_GRAM,     // V_ob^H V_ob of one outer block, and the Z scratch of the T combination
  S_QN,          // Q_n = Qp^H (eta x cols): the Hastings GEMM's B operand read K-major
  S_QR_TOB2,     // the tall pair's Y^H chain: combined T per outer block,
  S_QR_GRAM2,    //   Gram / Z scratch,
  S_QR_YW,       //   W / W2 of its block reflectors,
  S_QR_YW2,
  S_QR_TALL,     //   T of all finished Y^H blocks (k x k, left-looking updates),
  S_QR_TALLZ,    //   the V^H V / Z scratch of its growth,
  S_QR_PART2,    //   panel scratch,
  S_QR_QYM,      //   T_all V_b^H, forming Q of Y^H block by block
  S_GEMM_PART4,  // split-K scratch of GEMMs on side5 (the tall pair's Q blocks and their consumers)
  S_TILE_SUMS4,
  S_COUNT
};

// device scalar indices (doubles)
enum Scal : int {
  SC_THETA2 = 0,  // ||theta||^2
  SC_L2,          // ||L||^2 (or ||kept||^2 for CBE)
  SC_RESID,       // explicit residual ||theta - approx||^2
  SC_TMP0,
  SC_TMP1,
  SC_TMP2,
  SC_TMP3,
  SC_COUNT = 64
};

struct Engine {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  std::vector<void*> slot_ptr = std::vector<void*>(S_COUNT, nullptr);
  std::vector<size_t> slot_bytes = std::vector<size_t>(S_COUNT, 0);
  double* dscal = nullptr;   // device scalars
  double* hscal = nullptr;   // pinned host mirror
  unsigned* barrier = nullptr;  // grid-barrier words (count, generation)
  int num_sms = kNumSMs;
  // second stream for work that overlaps the main stream inside one call
  // (the QR trailing update behind the next panel); forks and joins through
  // events, so it is captured into CUDA graphs with the main stream
  cudaStream_t side = nullptr;
  // third stream: applies each finished panel's block reflector to a second
  // matrix (Q^H theta) behind the panel chain (QrOpts::capply)
  cudaStream_t side2 = nullptr;
  // fourth stream: the second QR of a pipelined pair (qr_pair_pipelined)
  cudaStream_t side3 = nullptr;
  // fifth stream: column blocks of the pair's explicit Q, formed as soon as
  // their reflectors exist
  cudaStream_t side4 = nullptr;
  // sixth stream: left-looking updates of the pair's Y^H blocks, concurrent
  // with the Y panel before them
  cudaStream_t side5 = nullptr;
  std::vector<cudaEvent_t> events;
  cudaEvent_t event(size_t i);
  // smallest two-site block height that takes the pipelined QR pair on this
  // engine (-1: the library default); contexts that run side by side with
  // other contexts (sharded chains) raise it (qt_ctx_set_qr_pair_min_rows)
  long long qr_pair_min_rows = -1;
  // bumped whenever raw() frees and reallocates a slot: captured CUDA graphs
  // hold raw slot pointers and must be recaptured after a regrowth
  unsigned long long arena_gen = 0;

  void init(int dev, cudaStream_t st);
  void destroy();
  // grow-only scratch; contents are not preserved across growth
  void* raw(int slot, size_t bytes);
  double2* cbuf(int slot, size_t elems) { return static_cast<double2*>(raw(slot, elems * sizeof(double2))); }
  double* dbuf(int slot, size_t elems) { return static_cast<double*>(raw(slot, elems * sizeof(double))); }
  GemmScratch gemm_scratch();
  GemmScratch gemm_scratch2();  // separate split-K buffers for GEMMs on side2
  GemmScratch gemm_scratch3();  // ... and on side4
  GemmScratch gemm_scratch4();  // ... and on side5
};

// ---- kernels shared by the modules (aux.cu) -------------------------------
// out = scale * [conj](permute(in)); rank <= 4, perm[k] = input axis of output axis k
void permute(Engine& e, const double2* in, int rank, const long long* shape, const int* perm, bool conj,
             double2* out, double scale = 1.0, const double* dscale = nullptr, cudaStream_t st = nullptr);
// out[0] = sum |x|^2 over a (rows x cols, ld) matrix, deterministic
void norm2(Engine& e, const double2* x, long long rows, long long cols, long long ld, double* out);
// dst = src over rows x cols blocks with leading dimensions
void copy2d(Engine& e, const double2* src, long long lds, double2* dst, long long ldd, long long rows,
            long long cols, cudaStream_t st = nullptr);
void set_identity(Engine& e, double2* q, long long rows, long long cols, long long ld, cudaStream_t st = nullptr);
void check_finite(Engine& e, const double2* x, long long n, int* dflag);
// the same over a (rows x cols, ld) block, on `st` (nullptr: e.stream)
void check_finite_2d(Engine& e, const double2* x, long long rows, long long cols, long long ld, int* dflag,
                     cudaStream_t st = nullptr);

// ---- Householder QR (householder.cu) ----------------------------------------
// Blocked Householder QR of the m x n row-major matrix a (ld lda), factored
// in place (a is destroyed).  Writes the explicit thin Q (m x k, ld ldq) and
// R (k x n, ld ldr), k = min(m, n), gauge-fixed so that diag(R) is real and
// non-negative (proj/src/linalg.cpp:25-51).
struct QrOpts {
  // when set: C (m x nc, ld ldc) <- Q^H C, applied panel by panel on e.side2
  // while the later panels factor (the reflectors are complete when qr_inplace
  // returns; the caller's stream has joined side2)
  double2* capply = nullptr;
  long long ldc = 0, nc = 0;
  bool want_q = true;  // form the explicit thin Q (gauge-fixed)
  bool want_r = true;  // write the gauge-fixed R
};
void qr_inplace(Engine& e, double2* a, long long m, long long n, long long lda, double2* q, long long ldq,
                double2* r, long long ldr, const QrOpts& opts = QrOpts());

// The two QRs of one alternating sweep (proj/src/gates.cpp:293-308), pipelined:
//   QR(X), X (m x k) -- every finished panel p is applied to C (m x nc) on
//   e.side2, so C <- Q_full^H C, and rows [32p, 32p + 32) of C, final once
//   panel p is applied, are published as columns of Y^H (nc x k, ld k):
//   yh[c, i] = ph_i conj(C[i, c]) with ph_i the phase of X's R_ii (the gauge
//   of Q_m), i.e. Y = Q_m^H C;
//   QR(Y^H) on e.side3 runs one panel behind: panel p of Y^H starts once block
//   p is extracted and has received the reflectors of Y^H panels < p
//   (left-looking block update).
// Only the explicit thin Q of Y^H (qy, nc x k) and its R (ry, k x k) are
// formed, gauge-fixed; X keeps its factored form (R on the upper triangle,
// the gauge phases on the diagonal).  Requires k <= m, k <= nc and both
// heights within one block-reflector cluster (qr_pair_fits).  Everything is
// joined into e.stream on return.
bool qr_pair_fits(long long m, long long nc);
// The same sweep for tall blocks (m, nc > 2048, both panels within one
// cluster): two-level QR(X) with each outer block applied to C (= theta) on
// e.side2 and its rows of Q_full^H C published through `extract` as columns of
// Y^H; QR(Y^H) runs on e.side3 one outer block behind, each block first
// receiving the combined reflector of the finished Y^H blocks (left-looking,
// one K = J GEMM triple).  Forms Q (nc x k) and R (k x k) of Y^H gauge-fixed,
// and, with qx != nullptr, X's thin Q (m x k) too.  Joined into e.stream.
bool qr_pair_tall_fits(long long m, long long nc, long long k);
void qr_pair_tall(Engine& e, double2* x, long long m, long long k, double2* c, long long nc, double2* yh,
                  double2* qy, double2* ry, double2* qx,
                  const std::function<void(long long, long long, cudaStream_t)>& extract);
// After qr_pair_pipelined: the explicit, gauge-fixed thin Q of X (m x k, ld
// ldq) from the reflectors the pair left in S_QR_V / S_QR_T, on stream st
// (left_iso of apply_gate_qr, proj/src/gates.cpp:373)
void pair_form_q(Engine& e, const double2* x, long long m, long long k, double2* q, long long ldq, cudaStream_t st);
// Callers may leave work in flight on e.side (the X look-ahead stream: X's
// columns past the first two panels, first touched there by the wide update)
// and have e.side2 wait for anything that still reads C (C is first written
// on e.side2).
void qr_pair_pipelined(Engine& e, double2* x, long long m, long long k, double2* c, long long nc, double2* yh,
                       double2* qy, double2* ry);

}  // namespace qt
