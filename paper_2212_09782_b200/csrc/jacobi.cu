// K5/K9: Hermitian eigensolver on the device (block two-sided Jacobi).
//
// Replaces eigh (proj/src/linalg.cpp:79-101: Eigen SelfAdjointEigenSolver on
// the symmetrized matrix, eigenpairs re-sorted descending) for the CBE Gram
// matrix G = L^H L (proj/src/gates.cpp:408-413) and for the Schmidt spectra of
// the bond matrices (singular values via the Gram matrix).
//
// One persistent cooperative kernel per solve.  The matrix is scaled by an
// exact power of two and padded to N = JB * nb (nb even, JB = 16 for n <= 512,
// else 32) with decoupled diagonal entries below every eigenvalue.  Each sweep
// runs nb-1 rounds of a round-robin pairing of JB-wide blocks; a round is
//   A. one CTA per block pair (I,J): load the 2JB x 2JB Hermitian subproblem
//      G[X,X], X = I u J, into shared memory and run an inner sweep: JB
//      "cross" rounds of JB disjoint complex rotations pairing I with J, plus
//      (first round of a sweep only, when every block meets its pair partner)
//      JB-1 rounds inside I and J; each inner round forms the rotations once
//      and applies them two-sidedly in one pass over 2x2 blocks; store J_X;
//   B. every pair tile G[X,Y] <- J_X^H G[X,Y] J_Y with X <= Y (the tile
//      (Y,X) is written as its conjugate transpose) and every row chunk
//      V[r,Y] <- V[r,Y] J_Y, as m8n8k4 DMMA products in shared memory.
// Rounds are separated by a grid barrier on a monotonic arrival counter.
// Sweeps stop when, after a sweep, no off-diagonal entry meets the criterion
// of make_rot (a grid-wide scan: a further sweep would rotate nothing), at
// most 30 sweeps.  Every reduction has a fixed order: results are bitwise
// reproducible run to run.
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "gate.cuh"

namespace qt {
namespace {

constexpr int MAX_SWEEPS = 30;

// grid barrier on a monotonic arrival counter (zeroed by the setup kernel):
// release-add by every CTA, acquire-poll until epoch * nblocks arrivals
__device__ __forceinline__ void jgrid_sync(unsigned* bar, unsigned nblocks, unsigned& epoch) {
  __syncthreads();
  if (threadIdx.x == 0) {
    ++epoch;
    const unsigned target = epoch * nblocks;
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

// block (or local index) at position j of round r of a round-robin over n slots
__device__ __forceinline__ int rr_slot(int j, int r, int n) { return j == 0 ? 0 : 1 + (j - 1 + r) % (n - 1); }

struct JacobiArgs {
  double2* G;     // N x N, row-major
  double2* V;     // N x N
  double2* Jbuf;  // [2 round parities][npairs][JX][JX]
  double* flags;  // [MAX_SWEEPS] per-sweep max |offdiag| (reduced per CTA into slots below)
  double* cta_max;  // [2][gridDim]: per-CTA "an entry still meets the criterion" of the end-of-sweep scan
  unsigned* bar;
  int N, nb;
  int full_inner;  // 1: full inner sweep in every outer round (QT_JACOBI_FULL)
  double tol;
  double abs_floor;  // rotations skipped below abs_floor * ||G||_F
  int* sweeps_out;
  long long* prof;  // optional: cycles of CTA 0 in phase A / flag waits / phase B / first wave + barrier
  unsigned* tflag;  // [P(P+1)/2][2] round counter of the last update of every critical pair tile half
  const double* fro2;  // ||G||_F^2 (device)
};

// complex Jacobi rotation for [[a, c], [c*, b]] (a, b real): U = [[cs, sn],
// [-sn e^{-i phi}, cs e^{-i phi}]] zeroes the off-diagonal of U^H A U
struct Rot {
  double cs, sn;
  double2 e;  // e^{-i phi}
  bool active;
};

// power-of-two scale bringing ||G||_F into [1, 2): exact, so the eigenvalues
// are recovered bit-exactly and the squared magnitudes below cannot underflow
// above the absolute threshold
__device__ __forceinline__ double jscale(const double* fro2) {
  const double nrm = sqrt(*fro2);
  return nrm > 0.0 && isfinite(nrm) ? ldexp(1.0, -ilogb(nrm)) : 1.0;
}

// Rotation criterion (squared, on the scaled matrix):
//  * relative (Demmel-Veselic): |c| > eps sqrt(|a b|) keeps the small
//    eigenvalues of graded PSD Gram matrices (the CBE spectrum) accurate to
//    high relative precision;
//  * absolute: |c| > 1e-22 ||G||_F -- below it an off-diagonal element cannot
//    move any eigenvalue the truncation or the spectra can resolve (the
//    reference's own eigh is accurate to ~1e-16 ||G||).
__device__ __forceinline__ Rot make_rot(double a, double b, double2 c, double tol2, double abs_tol2) {
  Rot r;
  const double ac2 = fma(c.x, c.x, c.y * c.y);
  r.active = ac2 > tol2 * fabs(a * b) && ac2 > abs_tol2;
  if (!r.active) {
    r.cs = 1.0;
    r.sn = 0.0;
    r.e = make_double2(1.0, 0.0);
    return r;
  }
  // t = tan = sign(d) 2|c| / (|d| + sqrt(d^2 + 4|c|^2)), d = b - a, written so
  // that only two transcendental steps are dependent: with s = |d| + sqrt(..),
  // cs = s / sqrt(s^2 + 4|c|^2) and sn = sign(d) 2|c| / sqrt(s^2 + 4|c|^2);
  // |c| and the phase come from rsqrt(|c|^2) alongside
  const double d = b - a;
  const double inv_ac = rsqrt(ac2);
  const double s = fabs(d) + sqrt(fma(d, d, 4.0 * ac2));
  const double inv = rsqrt(fma(s, s, 4.0 * ac2));
  r.e = make_double2(c.x * inv_ac, -c.y * inv_ac);
  r.cs = s * inv;
  r.sn = copysign(2.0 * ac2 * inv_ac * inv, d);
  return r;
}

// pair k (< jb) of inner round ir over the 2 jb local indices, p < q:
// rounds ir < jb pair block I with block J, (k, jb + (k + ir) mod jb); rounds
// jb <= ir < 2 jb - 1 run a round-robin inside I (k < jb/2) and inside J
__device__ __forceinline__ void inner_pair(int k, int ir, int jb, int& p, int& q) {
  if (ir < jb) {
    int t = k + ir;
    if (t >= jb) t -= jb;
    p = k;
    q = jb + t;
  } else {
    const int h = jb / 2, t = ir - jb, kk = k < h ? k : k - h, base = k < h ? 0 : jb;
    int a = kk - 1 + t, b = jb - 2 - kk + t;  // round-robin slots, modulo jb - 1
    if (a >= jb - 1) a -= jb - 1;
    if (b >= jb - 1) b -= jb - 1;
    const int x = kk == 0 ? 0 : 1 + a, y = 1 + b;
    p = base + min(x, y);
    q = base + max(x, y);
  }
}

// rows (p,q) of a 2x2 block <- U^H (rows)
__device__ __forceinline__ void rot_rows(double2& s00, double2& s01, double2& s10, double2& s11, const Rot& r) {
  const double2 ce = cconj(r.e);
  const double2 u0 = cmul(ce, s10), u1 = cmul(ce, s11);
  const double2 t00 = csub(cscale(s00, r.cs), cscale(u0, r.sn));
  const double2 t01 = csub(cscale(s01, r.cs), cscale(u1, r.sn));
  s10 = cadd(cscale(s00, r.sn), cscale(u0, r.cs));
  s11 = cadd(cscale(s01, r.sn), cscale(u1, r.cs));
  s00 = t00;
  s01 = t01;
}

// columns (p,q) of a 2x2 block <- (cols) U
__device__ __forceinline__ void rot_cols(double2& s00, double2& s01, double2& s10, double2& s11, const Rot& r) {
  const double2 v0 = cmul(r.e, s01), v1 = cmul(r.e, s11);
  const double2 t00 = csub(cscale(s00, r.cs), cscale(v0, r.sn));
  const double2 t10 = csub(cscale(s10, r.cs), cscale(v1, r.sn));
  s01 = cadd(cscale(s00, r.sn), cscale(v0, r.cs));
  s11 = cadd(cscale(s10, r.sn), cscale(v1, r.cs));
  s00 = t00;
  s10 = t10;
}

// one m8n8k4 FP64 MMA: c += a b (A row-major 8x4, B column-major 4x8)
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// C = op(A) B for JX x JX complex tiles in shared memory (row stride JX+1),
// op(A) = A or A^H, on NW warps with DMMA: each warp owns one 8-row block and
// BPW 8-column blocks; a complex product is three real MMAs (3M, as in
// zgemm.cu: P1 = Re a Re b, P2 = Im a Im b, P3 = (Re a + Im a)(Re b + Im b))
// HALF: only the output columns [hc JX/2, (hc + 1) JX/2) (one column block
// of the pair), on all warps
template <int JX, int NW, bool HALF = false>
__device__ __forceinline__ void tile_mm(double2 (*A)[JX + 1], bool conj_t, double2 (*B)[JX + 1],
                                        double2 (*C)[JX + 1], int hc = 0) {
  constexpr int NBLK = JX / 8;                  // 8x8 blocks per dimension
  constexpr int NBC = HALF ? NBLK / 2 : NBLK;   // output column blocks
  constexpr int BPW = NBLK * NBC / NW;          // blocks per warp
  constexpr int WPR = NBC / BPW;                // warps per block row
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int rb = w / WPR, cb0 = (w % WPR) * BPW + (HALF ? hc * NBC : 0);
  double p1[BPW][2], p2[BPW][2], p3[BPW][2];
#pragma unroll
  for (int b = 0; b < BPW; ++b) p1[b][0] = p1[b][1] = p2[b][0] = p2[b][1] = p3[b][0] = p3[b][1] = 0.0;
#pragma unroll 4
  for (int k0 = 0; k0 < JX; k0 += 4) {
    const double2 av = conj_t ? cconj(A[k0 + t][rb * 8 + g]) : A[rb * 8 + g][k0 + t];
    const double sa = av.x + av.y;
#pragma unroll
    for (int b = 0; b < BPW; ++b) {
      const double2 bv = B[k0 + t][(cb0 + b) * 8 + g];
      dmma(p1[b], av.x, bv.x);
      dmma(p2[b], av.y, bv.y);
      dmma(p3[b], sa, bv.x + bv.y);
    }
  }
#pragma unroll
  for (int b = 0; b < BPW; ++b)
#pragma unroll
    for (int h = 0; h < 2; ++h)
      C[rb * 8 + g][(cb0 + b) * 8 + 2 * t + h] = make_double2(p1[b][h] - p2[b][h], p3[b][h] - (p1[b][h] + p2[b][h]));
}

template <int JB>
__global__ void __launch_bounds__(JB * 16) jacobi_kernel(JacobiArgs a) {
  constexpr int JX = 2 * JB;   // subproblem size
  constexpr int JT = JB * 16;  // threads
  extern __shared__ double2 jdyn[];
  __shared__ Rot rots[JB];
  __shared__ int rp[JB], rq[JB];
  double2(*S)[JX + 1] = reinterpret_cast<double2(*)[JX + 1]>(jdyn);
  double2(*Jm)[JX + 1] = reinterpret_cast<double2(*)[JX + 1]>(jdyn + JX * (JX + 1));
  double2(*T1)[JX + 1] = reinterpret_cast<double2(*)[JX + 1]>(jdyn + 2 * JX * (JX + 1));
  __shared__ double red[JT];
  __shared__ int done_flag;

  const int tid = threadIdx.x;
  const int G = static_cast<int>(gridDim.x);
  const int cta = static_cast<int>(blockIdx.x);
  const int nb = a.nb, P = nb / 2, R1 = nb - 1;  // pairs per round, rounds per sweep
  const int N = a.N;
  const int ngt = P * (P + 1) / 2, nvt = (N / JX) * P;
  const double sc = jscale(a.fro2);
  const double abs_tol = a.abs_floor * sqrt(*a.fro2) * sc;
  const double abs_tol2 = abs_tol * abs_tol, tol2 = a.tol * a.tol;
  const bool stamp = a.prof && tid == 0 && cta == 0;
  long long pa = 0, pw = 0, pb = 0, ps = 0;
  unsigned epoch = 0;

  // ---- round-robin bookkeeping: block at position j of round r; pair of a
  // block in round r; the block paired with b in round r
  auto pos_of = [&](int b, int r) {
    if (b == 0) return 0;
    int j = (b - 1 - r) % R1;
    if (j < 0) j += R1;
    return j + 1;
  };
  auto pair_of = [&](int b, int r) {
    const int j = pos_of(b, r);
    return j < P ? j : nb - 1 - j;
  };
  auto partner = [&](int b, int r) { return rr_slot(nb - 1 - pos_of(b, r), r, nb); };
  auto tidx = [&](int x, int y) { return x * P - x * (x - 1) / 2 + (y - x); };  // x <= y

  // ---- phase A: one 2JB x 2JB subproblem of round `round`, pair p -> Jbuf[p]
  auto jslot = [&](long long g, int p) { return a.Jbuf + ((g & 1) * P + p) * static_cast<long long>(JX * JX); };
  auto phase_a = [&](long long g, int round, int p) {
    const int bI = rr_slot(p, round, nb), bJ = rr_slot(nb - 1 - p, round, nb);
    {
      constexpr int PER = JX * JX / JT;
      double2 rs[PER];
#pragma unroll
      for (int k = 0; k < PER; ++k) {  // all loads in flight at once
        const int e = tid + k * JT, i = e / JX, j = e % JX;
        const int gi = (i < JB ? bI * JB + i : bJ * JB + i - JB);
        const int gj = (j < JB ? bI * JB + j : bJ * JB + j - JB);
        rs[k] = a.G[static_cast<long long>(gi) * N + gj];
      }
#pragma unroll
      for (int k = 0; k < PER; ++k) {
        const int e = tid + k * JT, i = e / JX, j = e % JX;
        S[i][j] = rs[k];
        Jm[i][j] = make_double2(i == j ? 1.0 : 0.0, 0.0);
      }
    }
    __syncthreads();
    // inner sweep over the 2JB local indices: JB "cross" rounds pairing I
    // with J (i, JB + (i + s) mod JB), then JB-1 rounds inside I and J.  The
    // within-block rounds run only in the first outer round of a sweep (every
    // block is paired there); later rounds rotate the cross pairs only --
    // every pair is still rotated once per sweep.  Per inner round: JB
    // threads form the rotations once, then the thread owning the 2x2 block
    // (k,l) writes U_k^H S_kl U_l and J_kl U_l in place.  (Forming the
    // rotations redundantly in every thread to save the first barrier loses:
    // the FP64 pipe, not the barrier, is the limit.)
    const int n_inner = (round == 0 || a.full_inner) ? JX - 1 : JB;
    for (int ir = 0; ir < n_inner; ++ir) {
      if (tid < JB) {
        int p0, q0;
        inner_pair(tid, ir, JB, p0, q0);
        rots[tid] = make_rot(S[p0][p0].x, S[q0][q0].x, S[p0][q0], tol2, abs_tol2);
        rp[tid] = p0;
        rq[tid] = q0;
      }
      __syncthreads();
      for (int b = tid; b < JB * JB; b += JT) {
        const int k = b / JB, l = b % JB;
        const Rot rk = rots[k], rl = rots[l];
        if (!rk.active && !rl.active) continue;
        const int pk = rp[k], qk = rq[k], pl = rp[l], ql = rq[l];
        double2 s00 = S[pk][pl], s01 = S[pk][ql], s10 = S[qk][pl], s11 = S[qk][ql];
        if (rk.active) rot_rows(s00, s01, s10, s11, rk);
        if (rl.active) {
          rot_cols(s00, s01, s10, s11, rl);
          double2 j00 = Jm[pk][pl], j01 = Jm[pk][ql], j10 = Jm[qk][pl], j11 = Jm[qk][ql];
          rot_cols(j00, j01, j10, j11, rl);
          Jm[pk][pl] = j00;
          Jm[pk][ql] = j01;
          Jm[qk][pl] = j10;
          Jm[qk][ql] = j11;
        }
        if (k == l) {  // the rotated pivot block is diagonal and real
          s00.y = 0.0;
          s11.y = 0.0;
          if (rk.active) {
            s01 = make_double2(0.0, 0.0);
            s10 = make_double2(0.0, 0.0);
          }
        }
        S[pk][pl] = s00;
        S[pk][ql] = s01;
        S[qk][pl] = s10;
        S[qk][ql] = s11;
      }
      __syncthreads();
    }
    double2* jo = jslot(g, p);  // double-buffered: round g+1's solves overlap round g's tile updates
    for (int e = tid; e < JX * JX; e += JT) jo[e] = Jm[e / JX][e % JX];
    __syncthreads();
  };

  // ---- phase B work item: G pair tile (xa <= yb) or V row chunk rc
  // hc >= 0 (G tiles): only the columns of block hc of pair yb (and their
  // mirrored rows) -- a critical tile split over two CTAs
  auto tile = [&](long long g, int round, bool isG, int xa, int yb, int rc, int hc = -1) {
    const double2* jy = jslot(g, yb);
    const double2* jx = jslot(g, xa < 0 ? 0 : xa);
    const int yI = rr_slot(yb, round, nb), yJ = rr_slot(nb - 1 - yb, round, nb);
    int xI = 0, xJ = 0;
    if (isG) {
      xI = rr_slot(xa, round, nb);
      xJ = rr_slot(nb - 1 - xa, round, nb);
    }
    double2* M = isG ? a.G : a.V;
    // the item's global loads issue at once (tile, Jy and, for JB = 16, Jx
    // staged in registers): one L2 round trip instead of a dependent chain per
    // loop iteration (JB = 32 fetches Jx after the first product: 24 staged
    // values per thread would spill at 128 registers)
    constexpr int PER = JX * JX / JT;
    constexpr bool STAGE_JX = PER <= 4;
    double2 rs[PER], rj[PER], rx[STAGE_JX ? PER : 1];
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int e = tid + k * JT, i = e / JX, j = e % JX;
      const int gi = isG ? (i < JB ? xI * JB + i : xJ * JB + i - JB) : rc * JX + i;
      const int gj = j < JB ? yI * JB + j : yJ * JB + j - JB;
      rs[k] = M[static_cast<long long>(gi) * N + gj];
      rj[k] = jy[e];
      if (STAGE_JX) rx[STAGE_JX ? k : 0] = isG ? jx[e] : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int e = tid + k * JT;
      S[e / JX][e % JX] = rs[k];
      Jm[e / JX][e % JX] = rj[k];
    }
    __syncthreads();
    // T1 = S Jy, then (G tiles) out = Jx^H T1, on the FP64 tensor pipe
    if (hc >= 0)
      tile_mm<JX, JT / 32, true>(S, false, Jm, T1, hc);
    else
      tile_mm<JX, JT / 32>(S, false, Jm, T1);
    __syncthreads();
    if (isG) {
#pragma unroll
      for (int k = 0; k < PER; ++k) {
        const int e = tid + k * JT;
        Jm[e / JX][e % JX] = STAGE_JX ? rx[STAGE_JX ? k : 0] : jx[e];
      }
      __syncthreads();
      if (hc >= 0)
        tile_mm<JX, JT / 32, true>(Jm, true, T1, S, hc);
      else
        tile_mm<JX, JT / 32>(Jm, true, T1, S);
      __syncthreads();
    }
    double2(*O)[JX + 1] = isG ? S : T1;
    const int jlo = hc >= 0 ? hc * JB : 0, jw = hc >= 0 ? JB : JX;
    for (int e = tid; e < JX * jw; e += JT) {
      const int i = e / jw, j = jlo + e % jw;
      const int gi = isG ? (i < JB ? xI * JB + i : xJ * JB + i - JB) : rc * JX + i;
      const int gj = j < JB ? yI * JB + j : yJ * JB + j - JB;
      M[static_cast<long long>(gi) * N + gj] = O[i][j];
    }
    if (isG && xa != yb)
      for (int e = tid; e < JX * jw; e += JT) {  // mirror, coalesced along i
        const int j = jlo + e / JX, i = e % JX;
        const int gi = i < JB ? xI * JB + i : xJ * JB + i - JB;
        const int gj = j < JB ? yI * JB + j : yJ * JB + j - JB;
        M[static_cast<long long>(gj) * N + gi] = cconj(O[i][j]);
      }
    __syncthreads();
  };
  // the diagonal pair tile (x, x) of round g IS the rotated subproblem phase
  // A(g) leaves in shared memory (J^H G[X,X] J up to rounding): written back
  // by the solving CTA itself -- no other item of round g - 1 or g touches
  // those three block pairs -- so round g needs no diagonal tile update
  auto store_diag = [&](int round, int p) {
    const int bI = rr_slot(p, round, nb), bJ = rr_slot(nb - 1 - p, round, nb);
    for (int e = tid; e < JX * JX; e += JT) {
      const int i = e / JX, j = e % JX;
      const int gi = (i < JB ? bI * JB + i : bJ * JB + i - JB);
      const int gj = (j < JB ? bI * JB + j : bJ * JB + j - JB);
      a.G[static_cast<long long>(gi) * N + gj] = S[i][j];
    }
    __syncthreads();
  };
  // publish a G tile of global round rg (release after the CTA's stores)
  // (one flag per column half of a critical tile: the halves run on two CTAs)
  auto flag_tile = [&](int x, int y, int hc, unsigned rg) {
    if (tid == 0) {
      __threadfence();
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a.tflag + 2 * tidx(x, y) + hc), "r"(rg) : "memory");
    }
  };
  auto wait_tile = [&](int x, int y, unsigned rg) {
    if (tid == 0)
      for (int hc = 0; hc < 2; ++hc) {
        const unsigned* f = a.tflag + 2 * tidx(min(x, y), max(x, y)) + hc;
        unsigned v;
        do {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
        } while (v < rg);
      }
  };
  // ---- schedule: phase A of round 0, barrier; then every iteration runs
  // phase B of round (sw, rd) and, overlapped with it, phase A of the next
  // round: the 2P pair tiles the next subproblems read (the diagonal tiles,
  // CTA x, and one off-diagonal tile per next pair, CTAs P..) go first and are
  // flagged; the CTAs < P wait for their three tiles and solve; the other
  // CTAs finish the remaining tiles; one grid barrier per round.
  if (cta < P) {
    phase_a(0, 0, cta);
    store_diag(0, cta);
  }
  jgrid_sync(a.bar, G, epoch);
  int sw = 0, rd = 0;
  bool conv = false;
  for (;;) {
    long long t0 = stamp ? clock64() : 0;
    const int ns = rd == R1 - 1 ? sw + 1 : sw, nr = rd == R1 - 1 ? 0 : rd + 1;
    const bool doA = ns < MAX_SWEEPS;
    const long long gcur = static_cast<long long>(sw) * R1 + rd;  // global round index
    const unsigned rg = static_cast<unsigned>(gcur + 1);
    // critical off-diagonal tile of next pair q: the pairs (round rd) of its blocks
    auto crit = [&](int q, int& x, int& y) {
      const int u = pair_of(rr_slot(q, nr, nb), rd), v = pair_of(rr_slot(nb - 1 - q, nr, nb), rd);
      x = min(u, v);
      y = max(u, v);
    };
    auto is_crit = [&](int x, int y) {  // x < y
      const int y1 = pair_of(partner(rr_slot(x, rd, nb), nr), rd);
      const int y2 = pair_of(partner(rr_slot(nb - 1 - x, rd, nb), nr), rd);
      return y == y1 || y == y2;
    };
    if (doA && cta >= P)
      for (int u = cta - P; u < 2 * P; u += G - P) {  // (next pair, column half)
        const int q = u >> 1, hc = u & 1;
        int x, y;
        crit(q, x, y);
        if (x == y) continue;
        // two next pairs can read the same tile (blocks of pairs x and y
        // pair up crosswise): the lower next pair owns it
        const int b1 = rr_slot(q, nr, nb), b2 = rr_slot(nb - 1 - q, nr, nb);
        const int o1 = b1 == rr_slot(pair_of(b1, rd), rd, nb) ? rr_slot(nb - 1 - pair_of(b1, rd), rd, nb)
                                                                : rr_slot(pair_of(b1, rd), rd, nb);
        const int o2 = partner(o1, nr);  // the other block of pair(b1) meets o2 in the next round
        if (o2 != b2 && pair_of(o2, rd) == pair_of(b2, rd) && pair_of(o1, nr) < q) continue;
        tile(gcur, rd, true, x, y, 0, hc);
        flag_tile(x, y, hc, rg);
      }
    long long t1 = stamp ? clock64() : 0;
    if (doA && cta < P) {
      int x, y;
      crit(cta, x, y);
      // the diagonal tiles (x, x) and (y, y) of round gcur were written by
      // the solves of the previous iteration (before the grid barrier)
      if (x != y) wait_tile(x, y, rg);
      __syncthreads();
      long long t2 = stamp ? clock64() : 0;
      phase_a(gcur + 1, nr, cta);
      // at a sweep end the solve is speculative: its diagonal tile is
      // written only once the convergence scan (which must see the end of
      // this sweep) has decided to go on
      if (rd != R1 - 1) store_diag(nr, cta);
      if (stamp) {
        pw += t2 - t1;
        pa += clock64() - t2;
      }
    }
    // remaining work: off-diagonal G tiles that are not critical, then V chunks
    const int c0 = doA ? P : 0, nw = doA ? G - P : G;
    if (cta >= c0)
      for (int u = cta - c0; u < ngt + nvt; u += nw) {
        if (u < ngt) {
          int v = u, x = 0;
          while (v >= P - x) {
            v -= P - x;
            ++x;
          }
          const int y = x + v;
          if (y == x || (doA && is_crit(x, y))) continue;
          tile(gcur, rd, true, x, y, 0);
        } else {
          const int w2 = u - ngt;
          tile(gcur, rd, false, -1, w2 % P, w2 / P);
        }
      }
    if (stamp) pb += clock64() - t1;
    long long t3 = stamp ? clock64() : 0;
    jgrid_sync(a.bar, G, epoch);
    if (rd == R1 - 1) {
      // sweep sw is complete and G holds its result: a further sweep rotates
      // iff some off-diagonal entry meets make_rot's criterion (the phase A
      // solves of the next round, run speculatively above, then rotated
      // nothing).  This scan replaces a whole verification sweep.
      double any = 0.0;
      const long long NN = static_cast<long long>(N) * N;
      for (long long e = static_cast<long long>(cta) * JT + tid; e < NN; e += static_cast<long long>(G) * JT) {
        const int i = static_cast<int>(e / N), j = static_cast<int>(e % N);
        if (j <= i) continue;
        const double2 c = __ldcg(&a.G[e]);
        const double ac2 = fma(c.x, c.x, c.y * c.y);
        if (ac2 > abs_tol2 &&
            ac2 > tol2 * fabs(__ldcg(&a.G[static_cast<long long>(i) * (N + 1)].x) *
                              __ldcg(&a.G[static_cast<long long>(j) * (N + 1)].x)))
          any = 1.0;
      }
      red[tid] = any;
      __syncthreads();
      for (int w = JT / 2; w > 0; w >>= 1) {
        if (tid < w) red[tid] = fmax(red[tid], red[tid + w]);
        __syncthreads();
      }
      if (tid == 0) a.cta_max[(sw & 1) * G + cta] = red[0];
      jgrid_sync(a.bar, G, epoch);
      if (tid == 0) {
        double m = 0.0;
        for (int b = 0; b < G; ++b) m = fmax(m, __ldcg(&a.cta_max[(sw & 1) * G + b]));
        done_flag = m == 0.0;
      }
      __syncthreads();
      if (done_flag || !doA) {
        conv = done_flag != 0;
        sw = ns;
        break;
      }
      // going on: the deferred diagonal tiles, visible to every solve of the
      // next round (which reads them without a flag) after one more barrier
      if (cta < P) store_diag(nr, cta);
      jgrid_sync(a.bar, G, epoch);
    }
    if (stamp) ps += clock64() - t3 + (t1 - t0);
    sw = ns;
    rd = nr;
  }
  // > 0: sweeps to convergence; < 0: stopped at MAX_SWEEPS without converging
  if (cta == 0 && tid == 0) *a.sweeps_out = conv ? max(sw, 1) : -max(sw, 1);
  if (stamp) {
    a.prof[0] = pa;
    a.prof[1] = pw;
    a.prof[2] = pb;
    a.prof[3] = ps;
  }
}

// pad: G_pad = [[G, 0], [0, diag(-(|G|+1) - i)]], V = I
__global__ void jacobi_setup_kernel(const double2* __restrict__ h, int n, int N, const double* fro, double2* G,
                                    double2* V, unsigned* bar, unsigned* tflag, int ntflag) {
  if (blockIdx.x == 0 && threadIdx.x == 0) bar[0] = 0;
  if (blockIdx.x == 0)
    for (int i = threadIdx.x; i < ntflag; i += blockDim.x) tflag[i] = 0;
  const double sc = jscale(fro);
  const double shift = -(sqrt(*fro) * sc + 1.0);
  const long long total = static_cast<long long>(N) * N;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(e / N), j = static_cast<int>(e % N);
    double2 g = make_double2(0.0, 0.0);
    if (i < n && j < n) {
      // symmetrize (proj/src/linalg.cpp:87): 0.5 (h + h^H)
      const double2 x = h[static_cast<long long>(i) * n + j], y = h[static_cast<long long>(j) * n + i];
      g = make_double2((0.5 * sc) * (x.x + y.x), (0.5 * sc) * (x.y - y.y));
      if (i == j) g.y = 0.0;
    } else if (i == j) {
      g = make_double2(shift - i, 0.0);
    }
    G[e] = g;
    V[e] = make_double2(i == j ? 1.0 : 0.0, 0.0);
  }
}

// sort the N diagonal entries descending (ties: lower index first), write the
// first n eigenvalues and the matching eigenvector columns (n x n, ld n)
__global__ void jacobi_sort_kernel(const double2* __restrict__ G, int n, int N, const double* fro, double* w,
                                   int* idx_out) {
  extern __shared__ unsigned char jsm[];
  int P = 1;
  while (P < N) P <<= 1;
  double* k2 = reinterpret_cast<double*>(jsm);  // capacity P
  int* idx = reinterpret_cast<int*>(k2 + P);
  for (int i = threadIdx.x; i < P; i += blockDim.x) {
    k2[i] = i < N ? G[static_cast<long long>(i) * N + i].x : -INFINITY;
    idx[i] = i;
  }
  __syncthreads();
  // bitonic sort, descending by key, ascending by index on ties
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < P; i += blockDim.x) {
        const int j = i ^ stride;
        if (j > i) {
          const bool desc = (i & size) == 0;
          const bool i_first = (k2[i] > k2[j]) || (k2[i] == k2[j] && idx[i] < idx[j]);
          if (desc != i_first) {
            const double tk = k2[i];
            k2[i] = k2[j];
            k2[j] = tk;
            const int ti = idx[i];
            idx[i] = idx[j];
            idx[j] = ti;
          }
        }
      }
      __syncthreads();
    }
  }
  const double inv_sc = 1.0 / jscale(fro);  // exact (power of two)
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    w[i] = k2[i] * inv_sc;
    idx_out[i] = idx[i];
  }
}

// eigenvectors in the sorted order: vout[r, c] = V[r, idx[c]] (grid-wide; one
// CTA per row block, the permuted reads stay inside a 16 N-byte row)
__global__ void jacobi_gather_kernel(const double2* __restrict__ V, int n, int N, const int* __restrict__ idx,
                                     double2* __restrict__ vout) {
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < static_cast<long long>(n) * n;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(e / n), c = static_cast<int>(e % n);
    vout[e] = V[static_cast<long long>(r) * N + idx[c]];
  }
}

// s = sqrt(max(w, 0)) (Gram eigenvalues) or max(w, 0) (Jordan-Wielandt)
__global__ void sqrt_clip_kernel(const double* __restrict__ w, int n, double* s, bool no_sqrt = false) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    s[i] = w[i] > 0.0 ? (no_sqrt ? w[i] : sqrt(w[i])) : 0.0;
}

// H = [[0, m], [m^H, 0]] ((p+q) x (p+q), row-major) for the p x q matrix m
__global__ void jw_build_kernel(const double2* __restrict__ m, long long p, long long q, double2* __restrict__ h) {
  const long long n = p + q, total = n * n;
  for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long i = t / n, j = t % n;
    double2 v = make_double2(0.0, 0.0);
    if (i < p && j >= p) {
      v = m[i * q + (j - p)];
    } else if (i >= p && j < p) {
      const double2 a = m[j * q + (i - p)];
      v = make_double2(a.x, -a.y);
    }
    h[t] = v;
  }
}

}  // namespace

namespace {
__global__ void offdiag_rows_kernel(const double2* __restrict__ g, int n, double* rows) {
  __shared__ double sd[256];
  const int i = blockIdx.x;
  double acc = 0.0;
  for (int j = threadIdx.x; j < n; j += blockDim.x)
    if (j != i) {
      const double2 a = g[static_cast<long long>(i) * n + j];
      acc = fma(a.x, a.x, fma(a.y, a.y, acc));
    }
  sd[threadIdx.x] = acc;
  __syncthreads();
  for (int st = blockDim.x / 2; st > 0; st >>= 1) {
    if (threadIdx.x < st) sd[threadIdx.x] += sd[threadIdx.x + st];
    __syncthreads();
  }
  if (threadIdx.x == 0) rows[i] = sd[0];
}

__global__ void offdiag_sum_kernel(const double* __restrict__ rows, int n, const double* fro2, EighStatus* st) {
  __shared__ double sd[256];
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc += rows[i];
  sd[threadIdx.x] = acc;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sd[threadIdx.x] += sd[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    // G was scaled by a power of two s.t. ||G||_F ~ 1 (jscale); compare in
    // the scaled frame
    const double sc = jscale(fro2);  // G is held in the scaled frame
    st->offdiag2 = sd[0];
    st->fro2 = *fro2 * sc * sc;
  }
}
}  // namespace

const EighStatus* eigh_device(Engine& e, const double2* h, long long n, double* w, double2* v) {
  if (n <= 0) return nullptr;
  // 16-wide blocks (32x32 subproblems) below n = 512, 32-wide above: the
  // subproblem sweep is the critical path for small n, the tile updates for large n
  static const int jb_env = std::getenv("QT_JACOBI_JB") ? std::atoi(std::getenv("QT_JACOBI_JB")) : 0;
  const int JB = jb_env == 16 || jb_env == 32 ? jb_env : (n <= 512 ? 16 : 32), JX = 2 * JB, JT = 16 * JB;
  int nb = static_cast<int>(ceil_div(n, JB));
  if (nb < 2) nb = 2;
  if (nb & 1) ++nb;
  const int N = nb * JB;
  const int npairs = nb / 2;
  double2* G = e.cbuf(S_EIG_V, static_cast<size_t>(2) * N * N + static_cast<size_t>(2) * npairs * JX * JX);
  double2* V = G + static_cast<size_t>(N) * N;
  double2* Jbuf = V + static_cast<size_t>(N) * N;
  double* fro = e.dscal + SC_TMP2;
  norm2(e, h, n, n, n, fro);
  // at least P + 1 CTAs: CTAs < P solve the next round's subproblems while
  // the others finish the tile updates
  const int ngt = npairs * (npairs + 1) / 2;
  const int grid = std::min(e.num_sms, std::max(2 * npairs, std::min(ngt + (N / JX) * npairs, e.num_sms)));
  if (grid <= npairs) throw Error(Err::capacity, "eigh: matrix too large for the cooperative Jacobi kernel");
  // [cta_max 2 grid][sweeps 8][tflag: 2 halves x ngt -> ngt+1][sorted index n/2+1] (doubles)
  double* cta_max = e.dbuf(S_MISC, 2 * static_cast<size_t>(grid) + 8 + ngt + 1 + static_cast<size_t>(n) / 2 + 2);
  int* sweeps = reinterpret_cast<int*>(cta_max + 2 * grid);
  unsigned* tflag = reinterpret_cast<unsigned*>(cta_max + 2 * grid + 8);
  jacobi_setup_kernel<<<static_cast<int>(std::min<long long>(ceil_div(static_cast<long long>(N) * N, 256), 2048)), 256,
                        0, e.stream>>>(h, static_cast<int>(n), N, fro, G, V, e.barrier + 8, tflag, 2 * ngt);
  QT_LAUNCHED();
  JacobiArgs a;
  a.G = G;
  a.V = V;
  a.Jbuf = Jbuf;
  a.flags = nullptr;
  a.cta_max = cta_max;
  a.bar = e.barrier + 8;
  a.N = N;
  a.nb = nb;
  a.tol = 2.220446049250313e-16;  // relative off-diagonal threshold (unit roundoff)
  static const double abs_floor = std::getenv("QT_JACOBI_ABS") ? std::atof(std::getenv("QT_JACOBI_ABS")) : 1e-22;
  a.abs_floor = abs_floor;
  static const bool full_inner = std::getenv("QT_JACOBI_FULL") != nullptr;
  a.full_inner = full_inner ? 1 : 0;
  a.sweeps_out = sweeps;
  a.tflag = tflag;
  static long long* prof = nullptr;
  if (std::getenv("QT_EIGH_DEBUG") && !prof) QT_CUDA(cudaMalloc(&prof, 8 * sizeof(long long)));
  a.prof = prof;
  a.fro2 = fro;
  const size_t jsmem = 3 * JX * (JX + 1) * sizeof(double2);
  auto kern = JB == 16 ? jacobi_kernel<16> : jacobi_kernel<32>;
  static std::once_flag jattr[2];
  std::call_once(jattr[JB == 32], [&] {
    QT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(jsmem)));
  });
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(JT);
  cfg.dynamicSmemBytes = jsmem;
  cfg.stream = e.stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  static const bool dbg = std::getenv("QT_EIGH_DEBUG") != nullptr;
  cudaEvent_t d0 = nullptr, d1 = nullptr;
  if (dbg) {
    QT_CUDA(cudaEventCreate(&d0));
    QT_CUDA(cudaEventCreate(&d1));
    QT_CUDA(cudaEventRecord(d0, e.stream));
  }
  QT_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
  QT_LAUNCHED();
  if (dbg) {
    QT_CUDA(cudaEventRecord(d1, e.stream));
    int sw = 0;
    QT_CUDA(cudaMemcpyAsync(&sw, sweeps, sizeof(int), cudaMemcpyDeviceToHost, e.stream));
    QT_CUDA(cudaStreamSynchronize(e.stream));
    float ms = 0.f;
    QT_CUDA(cudaEventElapsedTime(&ms, d0, d1));
    long long pc[4] = {0, 0, 0, 0};
    QT_CUDA(cudaMemcpy(pc, prof, sizeof(pc), cudaMemcpyDeviceToHost));
    const double rounds = static_cast<double>(sw) * (nb - 1);
    std::fprintf(stderr,
                 "eigh n=%lld N=%d grid=%d sweeps=%d rounds/sweep=%d time=%.3f ms | CTA 0 cycles/round: phase A %.0f "
                 "flag wait %.0f phase B %.0f first wave + barrier %.0f\n",
                 n, N, grid, sw, nb - 1, ms, pc[0] / rounds, pc[1] / rounds, pc[2] / rounds, pc[3] / rounds);
    cudaEventDestroy(d0);
    cudaEventDestroy(d1);
  }
  int P = 1;
  while (P < N) P <<= 1;
  const size_t smem = static_cast<size_t>(P) * (sizeof(double) + sizeof(int));
  if (smem > 200 * 1024) throw Error(Err::capacity, "eigh: matrix too large for the device sort");
  static std::once_flag attr_once;  // set once to the cap checked above (no lost updates across threads)
  std::call_once(attr_once, [] {
    QT_CUDA(cudaFuncSetAttribute(jacobi_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  });
  int* idx = reinterpret_cast<int*>(cta_max + 2 * grid + 8 + ngt + 1);
  jacobi_sort_kernel<<<1, 1024, smem, e.stream>>>(G, static_cast<int>(n), N, fro, w, idx);
  QT_LAUNCHED();
  const long long nn = static_cast<long long>(n) * n;
  jacobi_gather_kernel<<<static_cast<int>(std::min<long long>(ceil_div(nn, 256), 4 * e.num_sms)), 256, 0, e.stream>>>(
      V, static_cast<int>(n), N, idx, v);
  QT_LAUNCHED();
  // residual off-diagonal mass of the rotated matrix (deterministic), for the
  // convergence verdict: rank-deficient Gram matrices keep rotating rounding
  // noise under the relative criterion until the sweep cap, yet are diagonal
  // to working precision
  auto* st = reinterpret_cast<EighStatus*>(sweeps);
  offdiag_rows_kernel<<<N, 256, 0, e.stream>>>(G, N, reinterpret_cast<double*>(Jbuf));
  QT_LAUNCHED();
  offdiag_sum_kernel<<<1, 256, 0, e.stream>>>(reinterpret_cast<const double*>(Jbuf), N, fro, st);
  QT_LAUNCHED();
  return st;
}

void require_eigh_converged(const EighStatus& st, long long n) {
  // Eigen's SelfAdjointEigenSolver info() != Success -> NumericError
  // (proj/src/linalg.cpp:88-90): converged when a full sweep rotated nothing,
  // or when the off-diagonal mass left at the sweep cap is at the rounding
  // level of a backward-stable solver (n u ||G||_F)
  if (st.sweeps > 0) return;
  const double u = 2.220446049250313e-16;
  const double lim = 32.0 * static_cast<double>(n) * u;  // Jacobi's rounding floor, with margin
  if (st.offdiag2 <= lim * lim * st.fro2) return;
  char buf[160];
  std::snprintf(buf, sizeof(buf), "eigh: factorization did not converge (n=%lld, %d sweeps, offdiag %.3e of %.3e)", n,
                -st.sweeps, std::sqrt(st.offdiag2), std::sqrt(st.fro2));
  throw Error(Err::numeric, buf);
}

namespace {
// per-row partial sums of |h_ij - conj(h_ji)|^2 and |h_ij|^2 (one CTA per row,
// fixed-order tree: deterministic)
__global__ void herm_defect_rows_kernel(const double2* __restrict__ h, int n, double* rows) {
  __shared__ double sd[256], sn[256];
  const int i = blockIdx.x;
  double acc_d = 0.0, acc_n = 0.0;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const double2 a = h[static_cast<long long>(i) * n + j], b = h[static_cast<long long>(j) * n + i];
    const double dr = a.x - b.x, di = a.y + b.y;
    acc_d += dr * dr + di * di;
    acc_n += a.x * a.x + a.y * a.y;
  }
  sd[threadIdx.x] = acc_d;
  sn[threadIdx.x] = acc_n;
  __syncthreads();
  for (int st = blockDim.x / 2; st > 0; st >>= 1) {
    if (threadIdx.x < st) {
      sd[threadIdx.x] += sd[threadIdx.x + st];
      sn[threadIdx.x] += sn[threadIdx.x + st];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    rows[2 * i] = sd[0];
    rows[2 * i + 1] = sn[0];
  }
}

__global__ void herm_defect_sum_kernel(const double* __restrict__ rows, int n, double* out2) {
  __shared__ double sd[256], sn[256];
  double acc_d = 0.0, acc_n = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    acc_d += rows[2 * i];
    acc_n += rows[2 * i + 1];
  }
  sd[threadIdx.x] = acc_d;
  sn[threadIdx.x] = acc_n;
  __syncthreads();
  for (int st = blockDim.x / 2; st > 0; st >>= 1) {
    if (threadIdx.x < st) {
      sd[threadIdx.x] += sd[threadIdx.x + st];
      sn[threadIdx.x] += sn[threadIdx.x + st];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out2[0] = sd[0];
    out2[1] = sn[0];
  }
}

}  // namespace


void hermitian_defect(Engine& e, const double2* h, long long n, double* out2) {
  double* rows = e.dbuf(S_QR_PART, 2 * n + 8);
  herm_defect_rows_kernel<<<static_cast<int>(n), 256, 0, e.stream>>>(h, static_cast<int>(n), rows);
  QT_LAUNCHED();
  herm_defect_sum_kernel<<<1, 256, 0, e.stream>>>(rows, static_cast<int>(n), out2);
  QT_LAUNCHED();
}

namespace {
// any nonzero off-diagonal element of the p x q matrix -> flag = 1
__global__ void offdiag_any_kernel(const double2* __restrict__ m, long long p, long long q, int* flag) {
  const long long total = p * q;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long i = e / q, j = e % q;
    if (i != j) {
      const double2 v = m[e];
      if (v.x != 0.0 || v.y != 0.0) {
        *flag = 1;
        return;
      }
    }
  }
}

// s = |diag(m)| sorted descending (ties: lower index first), one CTA bitonic
__global__ void diag_sv_kernel(const double2* __restrict__ m, long long q, int k, double* s) {
  extern __shared__ unsigned char dsm[];
  int P = 1;
  while (P < k) P <<= 1;
  double* key = reinterpret_cast<double*>(dsm);
  int* idx = reinterpret_cast<int*>(key + P);
  for (int i = threadIdx.x; i < P; i += blockDim.x) {
    key[i] = i < k ? hypot(m[static_cast<long long>(i) * q + i].x, m[static_cast<long long>(i) * q + i].y) : -1.0;
    idx[i] = i;
  }
  __syncthreads();
  for (int size = 2; size <= P; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < P; i += blockDim.x) {
        const int j = i ^ stride;
        if (j > i) {
          const bool desc = (i & size) == 0;
          const bool i_first = (key[i] > key[j]) || (key[i] == key[j] && idx[i] < idx[j]);
          if (desc != i_first) {
            const double tk = key[i];
            key[i] = key[j];
            key[j] = tk;
            const int ti = idx[i];
            idx[i] = idx[j];
            idx[j] = ti;
          }
        }
      }
      __syncthreads();
    }
  for (int i = threadIdx.x; i < k; i += blockDim.x) s[i] = key[i];
}
}  // namespace

bool diagonal_singular_values(Engine& e, const double2* m, long long p, long long q, double* s) {
  // CBE bond matrices are diagonal (gates.cpp:430, diagonal_bond_matrix): their
  // Schmidt values are the sorted |diagonal| -- exact, no Gram route
  const long long k = std::min(p, q);
  if (k <= 0 || k > 16384) return false;
  int* flag = reinterpret_cast<int*>(e.dscal + SC_TMP3);
  QT_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), e.stream));
  offdiag_any_kernel<<<static_cast<int>(std::min<long long>(ceil_div(p * q, 256), 4 * e.num_sms)), 256, 0,
                       e.stream>>>(m, p, q, flag);
  QT_LAUNCHED();
  int h = 1;
  QT_CUDA(cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, e.stream));
  QT_CUDA(cudaStreamSynchronize(e.stream));
  if (h != 0) return false;
  int P = 1;
  while (P < k) P <<= 1;
  const size_t smem = static_cast<size_t>(P) * (sizeof(double) + sizeof(int));
  if (smem > 200 * 1024) return false;
  static std::once_flag attr_once;
  std::call_once(attr_once, [] {
    QT_CUDA(cudaFuncSetAttribute(diag_sv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  });
  diag_sv_kernel<<<1, 1024, smem, e.stream>>>(m, q, static_cast<int>(k), s);
  QT_LAUNCHED();
  return true;
}

double* singular_values_device(Engine& e, const double2* m, long long p, long long q) {
  // Singular values of Xi, descending (svd(Xi).s, proj/src/mps.cpp:198-207).
  //  1. Gram route: s = sqrt(max(eig(m^H m), 0)).  Its absolute error is
  //     ~u s_0^2 / s_k: exact enough (<= 1e-13 s_0) when the spectrum spans
  //     less than 3 decades (s_min >= 1e-3 s_0) -- the common case.
  //  2. Otherwise the Jordan-Wielandt matrix H = [[0, m], [m^H, 0]], whose
  //     eigenvalues are +-s_k (and |p - q| zeros), goes through the same
  //     backward-stable Jacobi eigensolver: every s_k to ~u s_0 absolute,
  //     no squaring (|ds_k| <= 1e-10 s_0).
  const long long k = std::min(p, q);
  if (k == 0) return e.dbuf(S_EIG_W, 8);
  double* wd = e.dbuf(S_EIG_W, std::max(k, p + q) + 8);
  if (diagonal_singular_values(e, m, p, q, wd)) return wd;
  const bool wide = q > p;  // Gram on the smaller side
  const long long g = wide ? p : q;
  double2* gm = e.cbuf(S_GRAM, std::max(g * g, (p + q) * (p + q)));
  GemmDesc d;
  d.M = g;
  d.N = g;
  d.K = wide ? q : p;
  if (wide) {
    d.opA = Op::N;  // m m^H
    d.A = m;
    d.lda = q;
    d.opB = Op::H;
    d.B = m;
    d.ldb = q;
  } else {
    d.opA = Op::H;  // m^H m
    d.A = m;
    d.lda = q;
    d.opB = Op::N;
    d.B = m;
    d.ldb = q;
  }
  d.C = gm;
  d.ldc = g;
  zgemm(d, e.gemm_scratch(), e.stream);
  double2* v = e.cbuf(S_MISC2, std::max(g * g, (p + q) * (p + q)));
  const EighStatus* st = eigh_device(e, gm, g, wd, v);
  EighStatus hs{1, 0, 0.0, 0.0};
  double ends[2] = {0.0, 0.0};
  QT_CUDA(cudaMemcpyAsync(&hs, st, sizeof(hs), cudaMemcpyDeviceToHost, e.stream));
  QT_CUDA(cudaMemcpyAsync(&ends[0], wd, sizeof(double), cudaMemcpyDeviceToHost, e.stream));
  QT_CUDA(cudaMemcpyAsync(&ends[1], wd + (k - 1), sizeof(double), cudaMemcpyDeviceToHost, e.stream));
  QT_CUDA(cudaStreamSynchronize(e.stream));
  require_eigh_converged(hs, g);
  const long long n2 = p + q;
  if (ends[1] >= 1e-6 * ends[0] || n2 > 8192) {
    sqrt_clip_kernel<<<1, 256, 0, e.stream>>>(wd, static_cast<int>(k), wd);
    QT_LAUNCHED();
    return wd;
  }
  jw_build_kernel<<<static_cast<int>(std::min<long long>(ceil_div(n2 * n2, 256), 8 * e.num_sms)), 256, 0,
                    e.stream>>>(m, p, q, gm);
  QT_LAUNCHED();
  st = eigh_device(e, gm, n2, wd, v);
  QT_CUDA(cudaMemcpyAsync(&hs, st, sizeof(hs), cudaMemcpyDeviceToHost, e.stream));
  QT_CUDA(cudaStreamSynchronize(e.stream));
  require_eigh_converged(hs, n2);
  // the k largest eigenvalues are s_1 >= ... >= s_k >= 0 (rounding noise of
  // exact zeros clipped)
  sqrt_clip_kernel<<<1, 256, 0, e.stream>>>(wd, static_cast<int>(k), wd, true);
  QT_LAUNCHED();
  return wd;
}

}  // namespace qt
