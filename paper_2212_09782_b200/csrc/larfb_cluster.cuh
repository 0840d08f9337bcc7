// Fused block-reflector application for short panels (included by
// householder.cu inside its anonymous namespace; uses qr_panel.cuh helpers).
//
//   A <- (I - V T' V^H) A,   T' = T^H (trailing update of zgeqrf, zlarfb 'C')
//                            T' = T   (explicit Q, zungqr / zlarfb 'N')
//
// replaces the four launches W = V^H A (split-K + reduce), W2 = T' W,
// A -= V W2 when the panel is short (m <= 16 x 128 rows): one thread-block
// cluster per 32-column block of A, the cluster's CTAs split the rows.  Each
// CTA forms its partial W = V_r^H A_r in shared memory; the partials are
// reduce-scattered (row i of W summed on CTA i % CS in a fixed source order)
// and all-gathered through distributed shared memory with st.async +
// mbarrier complete_tx; every CTA then applies A_r -= V_r (T' W) to its rows.
// One launch, no global scratch, bitwise deterministic.
constexpr int LB_THREADS = 256;
constexpr int LB_MAX_RPC = 128;

__device__ __forceinline__ void lb_cp16(void* smem, const void* gmem, bool pred) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
               "l"(gmem), "r"(pred ? 16 : 0)
               : "memory");
}

// XOR swizzle of the 16-byte column slot inside each 8-column group: the
// m8n8k4 fragment loads (rows r..r+3 x 8 columns, and 8 rows x 4 columns) hit
// distinct bank groups in every quarter warp
__device__ __forceinline__ int lb_sw(int row, int col) { return col ^ (((row & 1) << 2) | (row & 2)); }

// one m8n8k4 FP64 MMA: c += a b (A row-major 8x4, B column-major 4x8)
__device__ __forceinline__ void lb_dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}
// complex 8x8x4 block product: (cre + i cim) += a b, four real MMAs
__device__ __forceinline__ void cmma(double (&cre)[2], double (&cim)[2], double2 a, double2 b) {
  lb_dmma(cre, a.x, b.x);
  lb_dmma(cre, -a.y, b.y);
  lb_dmma(cim, a.x, b.y);
  lb_dmma(cim, a.y, b.x);
}

// One cluster per CW-column block of A (CW = 32, 16 or 8: narrow blocks put
// more SMs on short updates); the cluster's CTAs split the rows (rpc each).
// The products run on the FP64 tensor pipe (m8n8k4 DMMA, four real MMAs per
// complex block) over XOR-swizzled shared-memory tiles.
template <int CW>
__global__ void __launch_bounds__(LB_THREADS, 1)
    larfb_cluster_kernel(const double2* __restrict__ V, long long ldv, const double2* __restrict__ T, double2* A,
                         long long lda, int mp, int ncols, int nbp, int rpc, int use_th, long long* dbg) {
  const bool stamp = dbg && threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0;
  if (stamp) dbg[0] = clock64();
  extern __shared__ __align__(16) double2 lsm[];
  double2* Vs = lsm;                 // [rpc][32]
  double2* As = Vs + rpc * NB;       // [rpc][CW]
  double2* Wp = As + rpc * CW;       // [32][CW] W2 = T' W
  double2* Wf = Wp + NB * CW;        // [32][CW] reduced W (all-gathered)
  double2* Tp = Wf + NB * CW;        // [32][32] T'
  double2* rs = Tp + NB * NB;        // [CS][rows_owned][CW] reduce-scatter inbox
  __shared__ uint64_t bars[2];       // reduce-scatter, all-gather

  const int tid = threadIdx.x;
  const unsigned rank = cluster_rank();
  const int CS = static_cast<int>(gridDim.x);
  const int rows_owned = (NB + CS - 1) / CS;  // W rows i with i % CS == rank
  const int my_rows = (NB - static_cast<int>(rank) + CS - 1) / CS;
  const long long c0 = static_cast<long long>(blockIdx.y) * CW;
  const int nc = static_cast<int>(min(static_cast<long long>(CW), ncols - c0));
  const int r0 = static_cast<int>(rank) * rpc;
  const int nloc = max(0, min(rpc, mp - r0));

  if (tid == 0) {
    pmbar_init(&bars[0], 1);
    pmbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    pmbar_arm(&bars[0], static_cast<unsigned>(CS * my_rows * CW * sizeof(double2)));
    pmbar_arm(&bars[1], static_cast<unsigned>(NB * CW * sizeof(double2)));
  }
  // stage V rows (full 32-wide, zero-padded by the panel) and the A row
  // slices with asynchronous 16-byte copies, all in flight at once; zero-fill
  // past the panel and past A's edge
  for (int e = tid; e < rpc * NB; e += LB_THREADS) {
    const int r = e / NB, c = e % NB;
    const bool ok = r < nloc;
    lb_cp16(&Vs[r * NB + lb_sw(r, c)], ok ? &V[static_cast<long long>(r0 + r) * ldv + c] : V, ok);
  }
  for (int e = tid; e < rpc * CW; e += LB_THREADS) {
    const int r = e / CW, c = e % CW;
    const bool ok = r < nloc && c < nc;
    lb_cp16(&As[r * CW + lb_sw(r, c)], ok ? &A[static_cast<long long>(r0 + r) * lda + c0 + c] : A, ok);
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  for (int e = tid; e < NB * NB; e += LB_THREADS) {
    const int i = e / NB, k = e % NB;
    Tp[e] = (i < nbp && k < nbp) ? (use_th ? cconj(T[k * NB + i]) : T[i * NB + k]) : make_double2(0.0, 0.0);
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  if (stamp) dbg[1] = clock64();
  cluster_sync_all();  // inputs staged, barriers armed everywhere before any push
  if (stamp) dbg[2] = clock64();

  // partial W = V_r^H A_r (32 x CW) on the FP64 tensor pipe: 8x8 output
  // blocks, BPW per warp (or KS warps splitting the rows of one block)
  const int lane = tid & 31, w = tid >> 5, g = lane >> 2, t = lane & 3;
  constexpr int CB = CW / 8;                 // column blocks
  constexpr int OB = 4 * CB;                 // output blocks of W
  constexpr int BPW = OB >= 8 ? OB / 8 : 1;  // blocks per warp
  constexpr int KS = OB >= 8 ? 1 : 8 / OB;   // warps per block (row split)
  {
    const int wb = w / KS, kh = w % KS;
    const int rb = (wb * BPW) / CB;  // BPW divides CB: one block row per warp
    double cre[BPW][2], cim[BPW][2];
#pragma unroll
    for (int b = 0; b < BPW; ++b) cre[b][0] = cre[b][1] = cim[b][0] = cim[b][1] = 0.0;
    const int rlo = kh * (rpc / KS), rhi = rlo + rpc / KS;
#pragma unroll 2
    for (int r = rlo; r < rhi; r += 4) {
      const int rr = r + t;
      const double2 av = cconj(Vs[rr * NB + lb_sw(rr, rb * 8 + g)]);
#pragma unroll
      for (int b = 0; b < BPW; ++b) {
        const int cb = (wb * BPW + b) % CB;
        const double2 bv = As[rr * CW + lb_sw(rr, cb * 8 + g)];
        cmma(cre[b], cim[b], av, bv);
      }
    }
    if (KS > 1) {  // combine the row halves in a fixed order through Wp
      if (kh == 1)
#pragma unroll
        for (int e2 = 0; e2 < 2; ++e2)
          Wp[(rb * 8 + g) * CW + (wb % CB) * 8 + 2 * t + e2] = make_double2(cre[0][e2], cim[0][e2]);
      __syncthreads();
      if (kh == 0)
#pragma unroll
        for (int e2 = 0; e2 < 2; ++e2) {
          const double2 o = Wp[(rb * 8 + g) * CW + (wb % CB) * 8 + 2 * t + e2];
          cre[0][e2] += o.x;
          cim[0][e2] += o.y;
        }
    }
    if (stamp) dbg[3] = clock64() + static_cast<long long>(cre[0][0] * 0.0);
    // reduce-scatter: row i -> CTA i % CS, slot (source rank, i / CS)
    if (kh == 0) {
      const int i = rb * 8 + g;
      const unsigned owner = static_cast<unsigned>(i % CS);
#pragma unroll
      for (int b = 0; b < BPW; ++b)
#pragma unroll
        for (int e2 = 0; e2 < 2; ++e2) {
          const int jj = ((wb * BPW + b) % CB) * 8 + 2 * t + e2;
          double2* slot = &rs[(static_cast<int>(rank) * rows_owned + i / CS) * CW + jj];
          st_async_push(cl_map(slot, owner), make_double2(cre[b][e2], cim[b][e2]), cl_map(&bars[0], owner));
        }
    }
  }
  pmbar_wait(&bars[0], 0);
  if (stamp) dbg[4] = clock64();
  // owned rows: fixed-order sum over sources, then the all-gather; threads
  // split as (entry, group of destinations)
  {
    const int nent = my_rows * CW;
    const int groups = max(1, min(CS, LB_THREADS / max(1, nent)));
    for (int e = tid; e < nent * groups; e += LB_THREADS) {
      const int ent = e / groups, g = e % groups;
      const int li = ent / CW, jj = ent % CW;
      const int i = static_cast<int>(rank) + li * CS;
      double2 s = make_double2(0.0, 0.0);
      for (int src = 0; src < CS; ++src) s = cadd(s, rs[(src * rows_owned + li) * CW + jj]);
      for (int dst = g; dst < CS; dst += groups)
        st_async_push(cl_map(&Wf[i * CW + jj], dst), s, cl_map(&bars[1], dst));
    }
  }
  pmbar_wait(&bars[1], 0);
  if (stamp) dbg[5] = clock64();
  // W2 = T' W (32 x CW, K = 32) into Wp
  if (w < OB / BPW) {
    const int rb = (w * BPW) / CB;
    double cre[BPW][2], cim[BPW][2];
#pragma unroll
    for (int b = 0; b < BPW; ++b) cre[b][0] = cre[b][1] = cim[b][0] = cim[b][1] = 0.0;
#pragma unroll
    for (int k0 = 0; k0 < NB; k0 += 4) {
      const double2 av = Tp[(rb * 8 + g) * NB + k0 + t];
#pragma unroll
      for (int b = 0; b < BPW; ++b) {
        const int cb = (w * BPW + b) % CB;
        cmma(cre[b], cim[b], av, Wf[(k0 + t) * CW + cb * 8 + g]);
      }
    }
#pragma unroll
    for (int b = 0; b < BPW; ++b)
#pragma unroll
      for (int e2 = 0; e2 < 2; ++e2)
        Wp[(rb * 8 + g) * CW + ((w * BPW + b) % CB) * 8 + 2 * t + e2] = make_double2(cre[b][e2], cim[b][e2]);
  }
  __syncthreads();
  if (stamp) dbg[6] = clock64();
  // A_r <- A_r - V_r W2 on the tensor pipe: 8x8 blocks of the rpc x CW slice
  for (int blk = w; blk < (rpc / 8) * CB; blk += LB_THREADS / 32) {
    const int rb = blk / CB, cb = blk % CB, row = rb * 8 + g;
    double cre[2], cim[2];
#pragma unroll
    for (int e2 = 0; e2 < 2; ++e2) {
      const double2 c = As[row * CW + lb_sw(row, cb * 8 + 2 * t + e2)];
      cre[e2] = c.x;
      cim[e2] = c.y;
    }
#pragma unroll
    for (int k0 = 0; k0 < NB; k0 += 4) {
      const double2 av = Vs[row * NB + lb_sw(row, k0 + t)];
      cmma(cre, cim, make_double2(-av.x, -av.y), Wp[(k0 + t) * CW + cb * 8 + g]);
    }
    if (row < nloc)
#pragma unroll
      for (int e2 = 0; e2 < 2; ++e2) {
        const int col = cb * 8 + 2 * t + e2;
        if (col < nc) A[static_cast<long long>(r0 + row) * lda + c0 + col] = make_double2(cre[e2], cim[e2]);
      }
  }
  if (stamp) dbg[7] = clock64();
  cluster_sync_all();  // no CTA retires while a peer may still push into it
  if (stamp) dbg[8] = clock64();
}

constexpr size_t larfb_cluster_smem(int rpc, int cs, int cw) {
  return (size_t(rpc) * (NB + cw) + 2 * NB * cw + NB * NB + size_t(cs) * ((NB + cs - 1) / cs) * cw) * sizeof(double2);
}

template <int CW>
void larfb_launch(cudaLaunchConfig_t& cfg, const double2* V, long long ldv, const double2* T, double2* A,
                  long long lda, long long mp, long long ncols, int nbp, long long rpc, bool use_th, long long* dbg) {
  static std::once_flag attr_once;
  std::call_once(attr_once, [] {
    QT_CUDA(cudaFuncSetAttribute(larfb_cluster_kernel<CW>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    QT_CUDA(cudaFuncSetAttribute(larfb_cluster_kernel<CW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(larfb_cluster_smem(LB_MAX_RPC, 16, 32))));
  });
  QT_CUDA(cudaLaunchKernelEx(&cfg, larfb_cluster_kernel<CW>, V, ldv, T, A, lda, static_cast<int>(mp),
                             static_cast<int>(ncols), nbp, static_cast<int>(rpc), use_th ? 1 : 0, dbg));
}

// A (mp x ncols, ld lda) <- (I - V T' V^H) A for a panel of nbp <= 32
// reflectors; returns false when the panel is too tall for one cluster.
// largest cluster the block-reflector kernel can run with (16, 8 or 0)
int larfb_max_cs() {
  static const int max_cs = [] {  // probed once, thread-safe (magic static)
    QT_CUDA(cudaFuncSetAttribute(larfb_cluster_kernel<32>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    QT_CUDA(cudaFuncSetAttribute(larfb_cluster_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(larfb_cluster_smem(LB_MAX_RPC, 16, 32))));
    int found = 0;
    for (int cs : {16, 8}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cs, 1);
      cfg.blockDim = dim3(LB_THREADS);
      cfg.dynamicSmemBytes = larfb_cluster_smem(LB_MAX_RPC, cs, 32);
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, larfb_cluster_kernel<32>, &cfg) == cudaSuccess && n >= 1) {
        found = cs;
        break;
      }
      cudaGetLastError();
    }
    return found;
  }();
  return max_cs;
}

// the cluster path covers a panel of mp rows
bool larfb_cluster_fits(long long mp) {
  static const bool disabled = std::getenv("QT_NO_LARFB_CLUSTER") != nullptr;
  const int cs = larfb_max_cs();
  if (disabled || cs == 0) return false;
  const long long rpc = ceil_div(std::max<long long>(8, ceil_div(mp, cs)), 8) * 8;
  return rpc <= LB_MAX_RPC;
}

bool larfb_cluster(Engine& e, const double2* V, long long ldv, const double2* T, double2* A, long long lda,
                   long long mp, long long ncols, int nbp, bool use_th, cudaStream_t st = nullptr) {
  if (!st) st = e.stream;
  const int max_cs = larfb_max_cs();
  static const bool disabled = std::getenv("QT_NO_LARFB_CLUSTER") != nullptr;
  if (disabled || max_cs == 0 || ncols <= 0) return ncols <= 0 && !disabled && max_cs > 0;
  long long rpc = std::max<long long>(8, ceil_div(mp, max_cs));
  rpc = ceil_div(rpc, 8) * 8;
  if (rpc > LB_MAX_RPC) return false;
  const long long cs = ceil_div(mp, rpc);
  // narrowest column block that keeps <= 8 clusters (one per GPC) in flight
  int cw = 32;
  if (ceil_div(ncols, 8) <= 8)
    cw = 8;
  else if (ceil_div(ncols, 16) <= 8)
    cw = 16;
  static const int cw_narrow = std::getenv("QT_NARROW_CW") ? std::atoi(std::getenv("QT_NARROW_CW")) : 0;
  if (ncols <= NB && (cw_narrow == 8 || cw_narrow == 16 || cw_narrow == 32)) cw = cw_narrow;
  static const bool dbg_on = std::getenv("QT_LARFB_DEBUG") != nullptr;
  static long long* dbg = nullptr;
  if (dbg_on && !dbg) QT_CUDA(cudaMalloc(&dbg, 16 * sizeof(long long)));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(cs), static_cast<unsigned>(ceil_div(ncols, cw)));
  cfg.blockDim = dim3(LB_THREADS);
  cfg.dynamicSmemBytes = larfb_cluster_smem(static_cast<int>(rpc), static_cast<int>(cs), cw);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = static_cast<unsigned>(cs);
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (cw == 8)
    larfb_launch<8>(cfg, V, ldv, T, A, lda, mp, ncols, nbp, rpc, use_th, dbg);
  else if (cw == 16)
    larfb_launch<16>(cfg, V, ldv, T, A, lda, mp, ncols, nbp, rpc, use_th, dbg);
  else
    larfb_launch<32>(cfg, V, ldv, T, A, lda, mp, ncols, nbp, rpc, use_th, dbg);
  QT_LAUNCHED();
  if (dbg) {  // QT_LARFB_DEBUG=1: phase timings of CTA (0,0) on stderr
    long long h[9];
    QT_CUDA(cudaMemcpyAsync(h, dbg, sizeof(h), cudaMemcpyDeviceToHost, st));
    QT_CUDA(cudaStreamSynchronize(st));
    std::fprintf(stderr,
                 "larfb mp=%lld ncols=%lld cs=%lld rpc=%lld cw=%d cycles: stage %lld csync %lld W %lld rs %lld ag %lld "
                 "W2 %lld upd %lld exit %lld\n",
                 mp, ncols, cs, rpc, cw, h[1] - h[0], h[2] - h[1], h[3] - h[2], h[4] - h[3], h[5] - h[4],
                 h[6] - h[5], h[7] - h[6], h[8] - h[7]);
  }
  return true;
}

// Left-looking block update for the pipelined QR pair (and, in reverse with
// T instead of T^H, one column block of the explicit Q): the reflectors of
// panels 0..nq-1 (V columns q*32.., rows q*32.. of the shared V matrix, T
// factors T + q*32*32) applied in order to one column block A (m rows,
// ncols <= 32 columns), A <- H_{nq-1}^H ... H_0^H A, in ONE launch.  The
// block stays in shared memory across the nq rounds; each round stages V_q,
// forms the partial W = V_q^H A on the FP64 tensor pipe, reduce-scatters and
// all-gathers W through DSMEM (double-buffered inboxes and mbarriers, so no
// cluster barrier between rounds) and applies A -= V_q (T_q^H W).
template <int CW>
__global__ void __launch_bounds__(LB_THREADS, 1)
    larfb_multi_kernel(const double2* __restrict__ V, long long ldv, const double2* __restrict__ T, double2* A,
                       long long lda, int m, int ncols, int nq, int k, int rpc, int reverse, int use_th,
                       const double2* __restrict__ ph, long long ph_ld, long long ph_col0) {
  extern __shared__ __align__(16) double2 lsm[];
  const int CS = static_cast<int>(gridDim.x);
  const int rows_owned = (NB + CS - 1) / CS;
  double2* Vs = lsm;                          // [rpc][32]
  double2* As = Vs + rpc * NB;                // [rpc][CW]
  double2* Wp = As + rpc * CW;                // [32][CW]
  double2* Tp = Wp + NB * CW;                 // [32][32]
  double2* Wf = Tp + NB * NB;                 // [2][32][CW]
  double2* rs = Wf + 2 * NB * CW;             // [2][CS][rows_owned][CW]
  __shared__ uint64_t bars[2][2];             // [round parity][reduce-scatter, all-gather]

  const int tid = threadIdx.x;
  const unsigned rank = cluster_rank();
  const int my_rows = (NB - static_cast<int>(rank) + CS - 1) / CS;
  const long long c0 = static_cast<long long>(blockIdx.y) * CW;
  const int nc = static_cast<int>(min(static_cast<long long>(CW), ncols - c0));
  const int r0 = static_cast<int>(rank) * rpc;
  const int nloc = max(0, min(rpc, m - r0));
  const unsigned rs_bytes = static_cast<unsigned>(CS * my_rows * CW * sizeof(double2));
  const unsigned ag_bytes = static_cast<unsigned>(NB * CW * sizeof(double2));
  const size_t rs_half = static_cast<size_t>(CS) * rows_owned * CW;

  if (tid == 0) {
    for (int p = 0; p < 2; ++p) {
      pmbar_init(&bars[p][0], 1);
      pmbar_init(&bars[p][1], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int p = 0; p < 2 && p < nq; ++p) {
      pmbar_arm(&bars[p][0], rs_bytes);
      pmbar_arm(&bars[p][1], ag_bytes);
    }
  }
  for (int e = tid; e < rpc * CW; e += LB_THREADS) {
    const int r = e / CW, c = e % CW;
    const bool ok = r < nloc && c < nc;
    lb_cp16(&As[r * CW + lb_sw(r, c)], ok ? &A[static_cast<long long>(r0 + r) * lda + c0 + c] : A, ok);
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  cluster_sync_all();  // barriers initialised and armed everywhere before any push

  const int lane = tid & 31, w = tid >> 5, g = lane >> 2, t = lane & 3;
  constexpr int CB = CW / 8;
  constexpr int OB = 4 * CB;
  constexpr int BPW = OB >= 8 ? OB / 8 : 1;
  constexpr int KS = OB >= 8 ? 1 : 8 / OB;
  for (int it = 0; it < nq; ++it) {
    const int par = it & 1;
    const unsigned phase = static_cast<unsigned>((it >> 1) & 1);
    const int q = reverse ? nq - 1 - it : it;  // reverse: H_{nq-1} first (explicit Q, zungqr order)
    const int jq = q * NB;
    const int nbq = min(NB, k - jq);
    if (it >= 1 && it + 1 < nq && tid == 0) {  // round it+1 reuses parity par^1: its round it-1 waits are done
      pmbar_arm(&bars[par ^ 1][0], rs_bytes);
      pmbar_arm(&bars[par ^ 1][1], ag_bytes);
    }
    // stage V_q on the local rows (zero above row jq: H_q leaves those rows alone)
    for (int e = tid; e < rpc * NB; e += LB_THREADS) {
      const int r = e / NB, c = e % NB;
      const int gr = r0 + r;
      const bool ok = r < nloc && gr >= jq;
      lb_cp16(&Vs[r * NB + lb_sw(r, c)], ok ? &V[static_cast<long long>(gr) * ldv + jq + c] : V, ok);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    for (int e = tid; e < NB * NB; e += LB_THREADS) {
      const int i = e / NB, kk = e % NB;
      const double2* Tq = T + static_cast<long long>(q) * NB * NB;
      Tp[e] = (i < nbq && kk < nbq) ? (use_th ? cconj(Tq[kk * NB + i]) : Tq[i * NB + kk]) : make_double2(0.0, 0.0);
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    double2* rsq = rs + par * rs_half;
    double2* Wfq = Wf + par * NB * CW;
    {
      const int wb = w / KS, kh = w % KS;
      const int rb = (wb * BPW) / CB;
      double cre[BPW][2], cim[BPW][2];
#pragma unroll
      for (int b = 0; b < BPW; ++b) cre[b][0] = cre[b][1] = cim[b][0] = cim[b][1] = 0.0;
      const int rlo = kh * (rpc / KS), rhi = rlo + rpc / KS;
#pragma unroll 2
      for (int r = rlo; r < rhi; r += 4) {
        const int rr = r + t;
        const double2 av = cconj(Vs[rr * NB + lb_sw(rr, rb * 8 + g)]);
#pragma unroll
        for (int b = 0; b < BPW; ++b) {
          const int cb = (wb * BPW + b) % CB;
          cmma(cre[b], cim[b], av, As[rr * CW + lb_sw(rr, cb * 8 + g)]);
        }
      }
      if (KS > 1) {
        if (kh == 1)
#pragma unroll
          for (int e2 = 0; e2 < 2; ++e2)
            Wp[(rb * 8 + g) * CW + (wb % CB) * 8 + 2 * t + e2] = make_double2(cre[0][e2], cim[0][e2]);
        __syncthreads();
        if (kh == 0)
#pragma unroll
          for (int e2 = 0; e2 < 2; ++e2) {
            const double2 o = Wp[(rb * 8 + g) * CW + (wb % CB) * 8 + 2 * t + e2];
            cre[0][e2] += o.x;
            cim[0][e2] += o.y;
          }
      }
      if (kh == 0) {
        const int i = rb * 8 + g;
        const unsigned owner = static_cast<unsigned>(i % CS);
#pragma unroll
        for (int b = 0; b < BPW; ++b)
#pragma unroll
          for (int e2 = 0; e2 < 2; ++e2) {
            const int jj = ((wb * BPW + b) % CB) * 8 + 2 * t + e2;
            double2* slot = &rsq[(static_cast<int>(rank) * rows_owned + i / CS) * CW + jj];
            st_async_push(cl_map(slot, owner), make_double2(cre[b][e2], cim[b][e2]), cl_map(&bars[par][0], owner));
          }
      }
    }
    pmbar_wait(&bars[par][0], phase);
    {
      const int nent = my_rows * CW;
      const int groups = max(1, min(CS, LB_THREADS / max(1, nent)));
      for (int e = tid; e < nent * groups; e += LB_THREADS) {
        const int ent = e / groups, gg = e % groups;
        const int li = ent / CW, jj = ent % CW;
        const int i = static_cast<int>(rank) + li * CS;
        double2 s = make_double2(0.0, 0.0);
        for (int src = 0; src < CS; ++src) s = cadd(s, rsq[(src * rows_owned + li) * CW + jj]);
        for (int dst = gg; dst < CS; dst += groups)
          st_async_push(cl_map(&Wfq[i * CW + jj], dst), s, cl_map(&bars[par][1], dst));
      }
    }
    pmbar_wait(&bars[par][1], phase);
    if (w < OB / BPW) {  // W2 = T_q^H W
      const int rb = (w * BPW) / CB;
      double cre[BPW][2], cim[BPW][2];
#pragma unroll
      for (int b = 0; b < BPW; ++b) cre[b][0] = cre[b][1] = cim[b][0] = cim[b][1] = 0.0;
#pragma unroll
      for (int k0 = 0; k0 < NB; k0 += 4) {
        const double2 av = Tp[(rb * 8 + g) * NB + k0 + t];
#pragma unroll
        for (int b = 0; b < BPW; ++b) {
          const int cb = (w * BPW + b) % CB;
          cmma(cre[b], cim[b], av, Wfq[(k0 + t) * CW + cb * 8 + g]);
        }
      }
#pragma unroll
      for (int b = 0; b < BPW; ++b)
#pragma unroll
        for (int e2 = 0; e2 < 2; ++e2)
          Wp[(rb * 8 + g) * CW + ((w * BPW + b) % CB) * 8 + 2 * t + e2] = make_double2(cre[b][e2], cim[b][e2]);
    }
    __syncthreads();
    // A_r -= V_q W2 in shared memory
    for (int blk = w; blk < (rpc / 8) * CB; blk += LB_THREADS / 32) {
      const int rb = blk / CB, cb = blk % CB, row = rb * 8 + g;
      double cre[2], cim[2];
#pragma unroll
      for (int e2 = 0; e2 < 2; ++e2) {
        const double2 c = As[row * CW + lb_sw(row, cb * 8 + 2 * t + e2)];
        cre[e2] = c.x;
        cim[e2] = c.y;
      }
#pragma unroll
      for (int k0 = 0; k0 < NB; k0 += 4) {
        const double2 av = Vs[row * NB + lb_sw(row, k0 + t)];
        cmma(cre, cim, make_double2(-av.x, -av.y), Wp[(k0 + t) * CW + cb * 8 + g]);
      }
#pragma unroll
      for (int e2 = 0; e2 < 2; ++e2) As[row * CW + lb_sw(row, cb * 8 + 2 * t + e2)] = make_double2(cre[e2], cim[e2]);
    }
    __syncthreads();  // A updated before the next round's partials; Vs/Tp/Wp free for restaging
  }
  for (int e = tid; e < nloc * CW; e += LB_THREADS) {
    const int r = e / CW, c = e % CW;
    if (c >= nc) continue;
    double2 v = As[r * CW + lb_sw(r, c)];
    if (ph) {  // gauge phase R_cc / |R_cc| of global column gc (explicit Q, linalg.cpp:25-36)
      const long long gc = ph_col0 + c0 + c;
      const double2 d = ph[gc * ph_ld + gc];
      const double ad = hypot(d.x, d.y);
      if (ad != 0.0) v = cmul(v, make_double2(d.x / ad, d.y / ad));
    }
    A[static_cast<long long>(r0 + r) * lda + c0 + c] = v;
  }
  cluster_sync_all();  // no CTA retires while a peer may still push into it
}

constexpr size_t larfb_multi_smem(int rpc, int cs, int cw) {
  return (size_t(rpc) * (NB + cw) + NB * cw + NB * NB + 2 * NB * cw + 2 * size_t(cs) * ((NB + cs - 1) / cs) * cw) *
         sizeof(double2);
}

template <int CW>
void larfb_multi_launch(cudaLaunchConfig_t& cfg, const double2* V, long long ldv, const double2* T, double2* A,
                        long long lda, long long m, long long ncols, int nq, long long k, long long rpc, bool reverse,
                        bool use_th, const double2* ph, long long ph_ld, long long ph_col0) {
  static bool attr = false;
  if (!attr) {
    QT_CUDA(cudaFuncSetAttribute(larfb_multi_kernel<CW>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    QT_CUDA(cudaFuncSetAttribute(larfb_multi_kernel<CW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(larfb_multi_smem(LB_MAX_RPC, 16, 32))));
    attr = true;
  }
  QT_CUDA(cudaLaunchKernelEx(&cfg, larfb_multi_kernel<CW>, V, ldv, T, A, lda, static_cast<int>(m),
                             static_cast<int>(ncols), nq, static_cast<int>(k), static_cast<int>(rpc), reverse ? 1 : 0,
                             use_th ? 1 : 0, ph, ph_ld, ph_col0));
}

// A (m x ncols <= 32, ld lda) <- H_{nq-1}^H ... H_0^H A with the reflectors of
// panels 0..nq-1 stored in V (ld ldv; panel q in columns q*32.., from row q*32)
// and T (32 x 32 per panel) of a k-column QR; false when m is too tall
// (reverse = true, use_th = false: A <- H_0 ... H_{nq-1} A, the explicit-Q order)
// (ph != nullptr: the written columns get the gauge phases of the diagonal of
// ph (ld ph_ld) at global columns ph_col0 + c)
bool larfb_multi(const double2* V, long long ldv, const double2* T, double2* A, long long lda, long long m,
                 long long ncols, int nq, long long k, cudaStream_t st, bool reverse = false, bool use_th = true,
                 const double2* ph = nullptr, long long ph_ld = 0, long long ph_col0 = 0) {
  const int max_cs = larfb_max_cs();
  if (max_cs == 0 || ncols <= 0 || ncols > NB) return false;
  if (nq <= 0) return true;
  long long rpc = std::max<long long>(8, ceil_div(m, max_cs));
  rpc = ceil_div(rpc, 8) * 8;
  if (rpc > LB_MAX_RPC) return false;
  const long long cs = ceil_div(m, rpc);
  const int cw = 8;  // four clusters of 8 columns: more SMs on the chain
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(cs), static_cast<unsigned>(ceil_div(ncols, cw)));
  cfg.blockDim = dim3(LB_THREADS);
  cfg.dynamicSmemBytes = larfb_multi_smem(static_cast<int>(rpc), static_cast<int>(cs), cw);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = static_cast<unsigned>(cs);
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  larfb_multi_launch<8>(cfg, V, ldv, T, A, lda, m, ncols, nq, k, rpc, reverse, use_th, ph, ph_ld, ph_col0);
  QT_LAUNCHED();
  return true;
}
