// mpk.cu -- K_mpk: fp64 matrix-powers kernels fused with the basis recurrence.
//
// Kernel families (plan.cu picks one per operator; all bit-identical):
//   k_level0_zm / k_level_zm      plane march over a pattern-compressed stencil
//                                 (the default for c1 c3 c5: 1-byte row ids)
//   k_level0_ss / k_level_ss      superset-mask pattern rows (small strides)
//   k_level0_pat / k_level_pat    table-walk pattern rows (any pattern operator)
//   k_level0_vs / k_level_vs      value stream: stencil structure, row-varying
//                                 values (c4), no column indices
//   k_level0_staged / k_level_staged, k_level0 / k_level   general CSR
//   opt-in experiments: k_mpk_wave (wavefront), *_win (TMA windows),
//   k_level_zp (row pairs), k_level_zt (shared-memory tile march),
//   k_resid_zm (split level 0) -- measured, see DESIGN.md 4a / 4b
//
// Reference: basis.py:210-225 `_recurrence_columns` over lacore.py:25-34 `spmv`
// (scipy csr_matvec).  One launch per level l builds BOTH P_{l+1} and R_{l+1}
// from a single pass over A (the reference runs the P and R recurrences one after
// the other, reading A 2s-1 times per block; here A is read s times):
//
//   w = (A y_l - theta_l y_l) [- mu_{l-1} y_{l-1}] ;  y_{l+1} = w / gamma_l
//
// Rounding is the reference's, bit for bit: each row sum starts at 0.0 and adds
// val*x in stored order with separately rounded multiply and add (what
// csr_matvec compiles to), and the recurrence is evaluated op by op with
// __dmul_rn/__dsub_rn/__ddiv_rn (numpy's element-wise order, no contraction).
// Level 0 also forms the true residual t = b - A x (adaptive.py:138) and the
// partial sums of ||t||^2 and ||r||^2 (adaptive.py:139,158) on the same pass.
//
// Roofline (HBM-bound): per level 12 nnz + 4 (n+1) bytes of A for
// CSR (1-2 n for a pattern operator, 8 ne n for a value stream) plus 16 n per
// generated column (+8 n with the Chebyshev two-back term).
#include "internal.cuh"
#include "rowops.cuh"

namespace {

__global__ void __launch_bounds__(MT_ROWS) k_level0_staged(Ctx c) {
  __shared__ double sm[MT_ROWS / 32];
  const SolverState* st = c.st;
  if (st->done) return;
  const int sbar = st->s_bar;
  const int sigma = c.cfg->sigma;
  const double th = st->prm.th[0], ga = st->prm.ga[0];
  const bool do_r = sbar >= 2;
  const double* P0 = c.Y;
  double* P1 = c.Y + c.ld;
  const double* R0 = c.Y + (int64_t)(sigma + 1) * c.ld;
  double* R1 = c.Y + (int64_t)(sigma + 2) * c.ld;
  double tt = 0.0, rr = 0.0;
  int bad = 0;
  const int64_t n_own = c.n_own, rlim = lvl_r_rows(c, sigma, 0);
  staged_rows(c, lvl_p_rows(c, sigma, 0), [&](int64_t i, const TileStage& ts) {
    const int beg = c.rp[i], end = c.rp[i + 1];
    const double p = P0[i], r = R0[i];
    double acc[3];
    const double* xs[3] = {c.x, P0, R0};
    if (do_r)
      row_dot_s<3>(ts, beg, end, xs, acc);
    else
      row_dot_s<2>(ts, beg, end, xs, acc);
    if (i < n_own) {
      const double t = __dsub_rn(c.b[i], acc[0]);
      tt = fma(t, t, tt);
      rr = fma(r, r, rr);
    }
    const double wp = recur(acc[1], p, 0.0, th, ga, 0.0, false);
    P1[i] = wp;
    bad |= !finite(wp);
    if (do_r && i < rlim) {
      const double wr = recur(acc[2], r, 0.0, th, ga, 0.0, false);
      R1[i] = wr;
      bad |= !finite(wr);
    }
  });
  tt = block_sum<MT_ROWS>(tt, sm);
  rr = block_sum<MT_ROWS>(rr, sm);
  if (threadIdx.x == 0) {
    c.part_t[blockIdx.x] = tt;
    c.part_r[blockIdx.x] = rr;
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&c.st->breakdown, 1);
}

__global__ void __launch_bounds__(MT_ROWS) k_level_staged(Ctx c, int l) {
  const SolverState* st = c.st;
  if (st->done) return;
  const int sbar = st->s_bar;
  if (l >= sbar) return;
  const int sigma = c.cfg->sigma;
  const double th = st->prm.th[l], ga = st->prm.ga[l], mu = st->prm.mu[l - 1];
  const bool use_mu = !(mu == 0.0);  // basis.py:217 `if mu != 0.0` (NaN counts)
  const bool do_r = l < sbar - 1;
  const double* Pl = c.Y + (int64_t)l * c.ld;
  const double* Pm = Pl - c.ld;
  double* Pn = c.Y + (int64_t)(l + 1) * c.ld;
  const double* Rl = c.Y + (int64_t)(sigma + 1 + l) * c.ld;
  const double* Rm = Rl - c.ld;
  double* Rn = c.Y + (int64_t)(sigma + 2 + l) * c.ld;
  int bad = 0;
  const int64_t rlim = lvl_r_rows(c, sigma, l);
  staged_rows(c, lvl_p_rows(c, sigma, l), [&](int64_t i, const TileStage& ts) {
    const int beg = c.rp[i], end = c.rp[i + 1];
    double acc[2];
    const double* xs[2] = {Pl, Rl};
    const bool rr = do_r && i < rlim;
    if (rr)
      row_dot_s<2>(ts, beg, end, xs, acc);
    else
      row_dot_s<1>(ts, beg, end, xs, acc);
    const double wp = recur(acc[0], Pl[i], use_mu ? Pm[i] : 0.0, th, ga, mu, use_mu);
    Pn[i] = wp;
    bad |= !finite(wp);
    if (rr) {
      const double wr = recur(acc[1], Rl[i], use_mu ? Rm[i] : 0.0, th, ga, mu, use_mu);
      Rn[i] = wr;
      bad |= !finite(wr);
    }
  });
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&c.st->breakdown, 1);
}

// ---------------------------------------------------------------------------
// Wavefront matrix-powers pass: levels l0 .. l0+nl-1 of the block in ONE
// persistent launch, so each CSR tile (and each freshly generated basis row) is
// re-read from L2 instead of HBM by the later levels of the pass.
//
// Work item (l, t) = level l on row tile t.  It needs level l-1 on the tiles
// dep[t] = [lo, hi] its rows' columns touch (host-computed from the CSR, made
// monotone in t).  Items are ordered by F = t + (l - l0) * D, then l; with the
// lag D > max(hi - t) every dependency comes strictly earlier in that order.
// CTAs are co-resident (grid <= occupancy x SMs) and claim positions in order
// from one atomic counter per pass, so any item a CTA waits on was claimed by
// a running CTA that only waits on even earlier items: no deadlock.  Dynamic
// claiming (not a static round robin) keeps CTAs from drifting apart: an item
// claimed Delta positions earlier also STARTED about Delta / G item-times
// earlier.  D carries slack (~6 G / nl tiles, twice the items in flight) so a
// dependency is normally complete when it is checked.
//
// Completion: per level, one counter per WAVE_GROUP tiles (zeroed by a memset
// node every outer loop).  Row arithmetic is the level kernels', so the basis
// is bit-identical to the level-by-level path.
//
// Warp roles (WAVE_THREADS = 8 consumer warps + 1 producer warp):
//  * the producer enumerates this CTA's items, checks their dependencies
//    (acquire loads of the counters; it remembers per level how far it has
//    verified -- dep ranges are monotone and a CTA's items of one level come in
//    increasing t), stages the tile's CSR by TMA into a free buffer and arrives
//    on full[s]; it publishes an item's completion (release add) once the
//    consumers have arrived on empty[s].  It publishes finished items ALSO
//    while spinning on a dependency: an item some other CTA waits for must
//    never sit unpublished behind a wait of ours (that could close a cycle).
//  * consumers wait on full[s], compute one row each, arrive on empty[s]; no
//    CTA-wide barrier on the per-item path.
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;\n" : "=l"(t));
  return t;
}
__device__ __forceinline__ void mbar_arrive1(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(done)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return done != 0;
}
// named barrier over the consumer warps only
__device__ __forceinline__ void consumers_sync() {
  asm volatile("bar.sync 1, %0;\n" ::"r"(MT_ROWS) : "memory");
}

#ifdef WAVE_DBG
// side-build instrumentation (tools/wave_sweep.py --dbg): [0] consumer cycles
// waiting on full, [1] consumer loop cycles, [2] consumer items (warp 0),
// [3] producer dep-wait cycles, [4] producer stage-wait cycles, [5] producer
// row_ptr cycles, [6] producer loop cycles, [7] dep-wait spin rounds
__device__ unsigned long long g_wave_dbg[8];
#define WDBG(...) __VA_ARGS__
#else
#define WDBG(...)
#endif

__global__ void __launch_bounds__(WAVE_THREADS, 4) k_mpk_wave(Ctx c, WaveArgs a) {
  extern __shared__ __align__(16) unsigned char msm[];
  __shared__ __align__(8) uint64_t full[MT_STAGES], empty[MT_STAGES];
  __shared__ int tb[MT_STAGES][2];
  __shared__ int titem[MT_STAGES][2];  // (level, tile) staged in each buffer; level -1: stop
  __shared__ int vhi[SMAX];            // producer: per input level, groups [.., vhi] verified
  __shared__ double sm[MT_ROWS / 32];
  __shared__ long long ntl[SMAX];      // tiles of each level of the pass (CA-MPK prefix rows)
  const SolverState* st = c.st;
  if (st->done) return;
  const int sbar = st->s_bar;
  const int sigma = c.cfg->sigma;
  const int l0 = a.l0;
  const int lend = (l0 + a.nl < sbar) ? l0 + a.nl : sbar;  // levels >= s_bar: nothing to build
  if (l0 >= lend) return;
  const int tid = threadIdx.x;
  const int cap = c.stage_cap;
  const size_t sb = wave_stage_bytes(cap);
  if (tid < SMAX) {
    ntl[tid] = (tid < a.nl) ? (lvl_p_rows(c, sigma, l0 + tid) + MT_ROWS - 1) / MT_ROWS : 0;
    vhi[tid] = -1;
  }
  if (tid == 0) {
    for (int s = 0; s < MT_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], MT_ROWS / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (tid >= MT_ROWS) {  // ---------------- producer warp
    const int lane = tid & 31;
    const int64_t npos = a.nF * a.nl;
    int64_t issued = 0, pub = 0;  // items staged / items whose completion is published
    WDBG(unsigned long long d_dep = 0, d_stage = 0, d_rp = 0, d_spin = 0; const long long d_t0 = clock64();)
    // publish item m (stage m % S) once its consumers are done; block or poll
    auto publish = [&](bool block) {
      while (pub < issued) {
        const int s = (int)(pub % MT_STAGES);
        const uint32_t par = (uint32_t)((pub / MT_STAGES) & 1);
        if (block)
          mbar_wait(&empty[s], par);
        else if (!mbar_test(&empty[s], par))
          return;
        const int l = titem[s][0];
        if (lane == 0 && l + 1 < lend)
          red_release_add(a.cnt + (int64_t)l * a.ngroups + titem[s][1] / WAVE_GROUP, 1);
        ++pub;
      }
    };
    for (;;) {
      int il = -1;
      int64_t it = 0;
      for (;;) {  // claim the next position of the pass; skip the empty ones
        unsigned int w = 0;
        if (lane == 0) w = atomicAdd(a.claim, 1u);
        const int64_t wpos = (int64_t)__shfl_sync(0xffffffffu, w, 0);
        if (wpos >= npos) break;
        const int64_t F = wpos / a.nl;
        const int li = (int)(wpos - F * a.nl);
        const int64_t t = F - (int64_t)li * a.D;
        if (l0 + li < lend && t >= 0 && t < ntl[li]) {
          il = l0 + li;
          it = t;
          break;
        }
      }
      if (il > l0) {  // wait for level il-1 on the dep tiles, publishing meanwhile
        const int2 d = a.dep[it];
        const int64_t nprev = ntl[il - 1 - l0];
        const int64_t hi_t = d.y < nprev ? d.y : nprev - 1;
        const int ghi = (int)(hi_t / WAVE_GROUP);
        const int gs = max((int)(d.x / WAVE_GROUP), vhi[il - 1] + 1);
        if (gs <= ghi) {
          const int* cnt = a.cnt + (int64_t)(il - 1) * a.ngroups;
          const uint64_t t0 = global_ns();
          WDBG(const long long c0 = clock64();)
          for (;;) {
            WDBG(++d_spin;)
            int ok = 1;
            for (int g = gs + lane; g <= ghi; g += 32) {
              const int64_t left = nprev - (int64_t)g * WAVE_GROUP;
              const int need = left < WAVE_GROUP ? (int)left : WAVE_GROUP;
              ok &= ld_acquire(cnt + g) >= need;
            }
            if (__all_sync(0xffffffffu, ok)) break;
            publish(false);
            if (global_ns() - t0 > 4000000000ull) __trap();  // lost item: fail, never hang
            __nanosleep(32);
          }
          WDBG(d_dep += clock64() - c0;)
          __syncwarp();
          if (lane == 0) vhi[il - 1] = ghi;
          __syncwarp();
        }
      }
      WDBG(const long long c1 = clock64();)
      // the tile's CSR segment (row_ptr loads) before blocking on a free stage
      int bv = 0, bc = 0;
      uint32_t nbv = 0, nbc = 0;
      if (il >= 0 && lane == 0) {
        const int64_t nrows = lvl_p_rows(c, sigma, il);
        const int64_t r0 = it * MT_ROWS;
        const int64_t r1 = r0 + MT_ROWS < nrows ? r0 + MT_ROWS : nrows;
        const int beg = c.rp[r0], end = c.rp[r1];
        bv = beg & ~1;
        bc = beg & ~3;
        nbv = (uint32_t)(((end - bv) * 8 + 15) / 16 * 16);
        nbc = (uint32_t)(((end - bc) * 4 + 15) / 16 * 16);
      }
      const int s = (int)(issued % MT_STAGES);
      WDBG(const long long c2 = clock64(); d_rp += (unsigned long long)(nbv + c2 - c1 - nbv);)
      // stage s is free once item issued - S is consumed (and published)
      while (pub + MT_STAGES <= issued) publish(true);
      WDBG(d_stage += clock64() - c2;)
      if (lane == 0) {
        titem[s][0] = il;
        titem[s][1] = (int)it;
        if (il < 0) {
          mbar_arrive1(&full[s]);  // stop marker
        } else {
          tb[s][0] = bv;
          tb[s][1] = bc;
          unsigned char* base = msm + (size_t)s * sb;
          const int64_t r0 = it * MT_ROWS;
          const int64_t rn = lvl_p_rows(c, sigma, il) - r0;
          const uint32_t nbr = (uint32_t)((((rn < MT_ROWS ? rn : MT_ROWS) + 1) * 4 + 15) / 16 * 16);
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
          mbar_arrive_tx(&full[s], nbv + nbc + nbr);
          if (nbv) bulk_g2s(base, c.val + bv, nbv, &full[s]);
          if (nbc) bulk_g2s(base + (size_t)(cap + 2) * 8, c.col + bc, nbc, &full[s]);
          bulk_g2s(base + stage_bytes(cap), c.rp + r0, nbr, &full[s]);
        }
      }
      __syncwarp();
      if (il < 0) break;
      ++issued;
    }
    publish(true);
    WDBG(if (lane == 0) {
      atomicAdd(&g_wave_dbg[3], d_dep);
      atomicAdd(&g_wave_dbg[4], d_stage);
      atomicAdd(&g_wave_dbg[5], d_rp);
      atomicAdd(&g_wave_dbg[6], (unsigned long long)(clock64() - d_t0));
      atomicAdd(&g_wave_dbg[7], d_spin);
    })
    return;
  }

  // ---------------- consumer warps: one row per thread per item
  double tt = 0.0, rr = 0.0;
  int bad = 0;
  const int64_t n_own = c.n_own;
  WDBG(unsigned long long d_full = 0, d_items = 0; const long long d_t1 = clock64();)
  for (int64_t k = 0;; ++k) {
    const int s = (int)(k % MT_STAGES);
    WDBG(const long long c0 = clock64();)
    mbar_wait(&full[s], (uint32_t)((k / MT_STAGES) & 1));
    WDBG(d_full += clock64() - c0; ++d_items;)
    const int l = titem[s][0];
    if (l < 0) break;
    const int64_t t = titem[s][1];
    TileStage ts;
    unsigned char* base = msm + (size_t)s * sb;
    ts.val = reinterpret_cast<const double*>(base);
    ts.col = reinterpret_cast<const int*>(base + (size_t)(cap + 2) * 8);
    ts.beg_v = tb[s][0];
    ts.beg_c = tb[s][1];
    const int* rps = reinterpret_cast<const int*>(base + stage_bytes(cap));
    const int64_t i = t * MT_ROWS + tid;
    const double th = st->prm.th[l], ga = st->prm.ga[l];
    if (l == 0) {
      const double* P0 = c.Y;
      double* P1 = c.Y + c.ld;
      const double* R0 = c.Y + (int64_t)(sigma + 1) * c.ld;
      double* R1 = c.Y + (int64_t)(sigma + 2) * c.ld;
      const bool do_r = sbar >= 2;
      if (i < lvl_p_rows(c, sigma, 0)) {
        const int beg = rps[tid], end = rps[tid + 1];
        const double p = P0[i], r = R0[i];
        double acc[3];
        const double* xs[3] = {c.x, P0, R0};
        if (do_r)
          row_dot_s<3>(ts, beg, end, xs, acc);
        else
          row_dot_s<2>(ts, beg, end, xs, acc);
        if (i < n_own) {
          const double tv = __dsub_rn(c.b[i], acc[0]);
          tt = fma(tv, tv, tt);
          rr = fma(r, r, rr);
        }
        const double wp = recur(acc[1], p, 0.0, th, ga, 0.0, false);
        P1[i] = wp;
        bad |= !finite(wp);
        if (do_r && i < lvl_r_rows(c, sigma, 0)) {
          const double wr = recur(acc[2], r, 0.0, th, ga, 0.0, false);
          R1[i] = wr;
          bad |= !finite(wr);
        }
      }
    } else {
      const double mu = st->prm.mu[l - 1];
      const bool use_mu = !(mu == 0.0);  // basis.py:217 `if mu != 0.0` (NaN counts)
      const bool do_r = l < sbar - 1;
      const double* Pl = c.Y + (int64_t)l * c.ld;
      const double* Pm = Pl - c.ld;
      double* Pn = c.Y + (int64_t)(l + 1) * c.ld;
      const double* Rl = c.Y + (int64_t)(sigma + 1 + l) * c.ld;
      const double* Rm = Rl - c.ld;
      double* Rn = c.Y + (int64_t)(sigma + 2 + l) * c.ld;
      if (i < lvl_p_rows(c, sigma, l)) {
        const int beg = rps[tid], end = rps[tid + 1];
        double acc[2];
        const double* xs[2] = {Pl, Rl};
        const bool rrow = do_r && i < lvl_r_rows(c, sigma, l);
        // inputs produced earlier in this launch when l > l0: coherent loads
        if (rrow)
          row_dot_s<2, LdCa, WAVE_BATCH>(ts, beg, end, xs, acc);
        else
          row_dot_s<1, LdCa, WAVE_BATCH>(ts, beg, end, xs, acc);
        const double wp =
            recur(acc[0], __ldca(Pl + i), use_mu ? __ldca(Pm + i) : 0.0, th, ga, mu, use_mu);
        Pn[i] = wp;
        bad |= !finite(wp);
        if (rrow) {
          const double wr =
              recur(acc[1], __ldca(Rl + i), use_mu ? __ldca(Rm + i) : 0.0, th, ga, mu, use_mu);
          Rn[i] = wr;
          bad |= !finite(wr);
        }
      }
    }
    __syncwarp();
    if ((tid & 31) == 0) mbar_arrive1(&empty[s]);  // this warp's rows are written
  }
  if (__any_sync(0xffffffffu, bad) && (tid & 31) == 0) atomicOr(&c.st->breakdown, 1);
  WDBG(if (tid == 0) {
    atomicAdd(&g_wave_dbg[0], d_full);
    atomicAdd(&g_wave_dbg[1], (unsigned long long)(clock64() - d_t1));
    atomicAdd(&g_wave_dbg[2], d_items);
  })
  if (l0 == 0) {  // level-0 norm partials over the consumer warps; slots beyond the grid zero
    double v[2] = {tt, rr};
    for (int q = 0; q < 2; ++q) {
      double x = warp_sum(v[q]);
      if ((tid & 31) == 0) sm[tid >> 5] = x;
      consumers_sync();
      if (tid == 0) {
        double r = 0.0;
#pragma unroll
        for (int w = 0; w < MT_ROWS / 32; ++w) r += sm[w];
        v[q] = r;
      }
      consumers_sync();
    }
    if (tid == 0) {
      c.part_t[blockIdx.x] = v[0];
      c.part_r[blockIdx.x] = v[1];
      for (int j = blockIdx.x + gridDim.x; j < c.red_n; j += gridDim.x) c.part_t[j] = c.part_r[j] = 0.0;
    }
  }
}

template <typename ID>
__global__ void __launch_bounds__(ROWS_PER_CTA) k_level0_pat(Ctx c) {
  __shared__ double sm[ROWS_PER_CTA / 32];
  const SolverState* st = c.st;
  if (st->done) return;
  const PatSmem T = load_patterns(c);
  const int sbar = st->s_bar;
  const int sigma = c.cfg->sigma;
  const double th = st->prm.th[0], ga = st->prm.ga[0];
  const bool do_r = sbar >= 2;
  const double* P0 = c.Y;
  double* P1 = c.Y + c.ld;
  const double* R0 = c.Y + (int64_t)(sigma + 1) * c.ld;
  double* R1 = c.Y + (int64_t)(sigma + 2) * c.ld;
  double tt = 0.0, rr = 0.0;
  int bad = 0;
  const int64_t n_own = c.n_own, plim = lvl_p_rows(c, sigma, 0), rlim = lvl_r_rows(c, sigma, 0);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int pid_next = i < plim ? row_pattern<ID>(c, i) : 0;  // ids one row ahead
  for (; i < plim; i += stride) {
    const int pid = pid_next;
    {
      const double* pf[3] = {c.x, P0, R0};
      prefetch_next<3>(c, i, stride, pf);
    }
    if (i + stride < plim) pid_next = row_pattern<ID>(c, i + stride);
    const int b = T.ptr[pid], e = T.ptr[pid + 1];
    const double p = P0[i], r = R0[i];
    double acc[3];
    const double* xs[3] = {c.x, P0, R0};
    if (do_r)
      row_dot_p<3>(T, b, e, (int)i, xs, acc);
    else
      row_dot_p<2>(T, b, e, (int)i, xs, acc);
    if (i < n_own) {
      const double t = __dsub_rn(c.b[i], acc[0]);
      tt = fma(t, t, tt);
      rr = fma(r, r, rr);
    }
    const double wp = recur(acc[1], p, 0.0, th, ga, 0.0, false);
    P1[i] = wp;
    bad |= !finite(wp);
    if (do_r && i < rlim) {
      const double wr = recur(acc[2], r, 0.0, th, ga, 0.0, false);
      R1[i] = wr;
      bad |= !finite(wr);
    }
  }
  tt = block_sum<ROWS_PER_CTA>(tt, sm);
  rr = block_sum<ROWS_PER_CTA>(rr, sm);
  if (threadIdx.x == 0) {
    c.part_t[blockIdx.x] = tt;
    c.part_r[blockIdx.x] = rr;
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&c.st->breakdown, 1);
}

// (an explicit min-blocks of 1 lets ptxas take ~85 registers: 2 CTAs/SM;
// 0 = no min-blocks hint)
#ifndef PAT_MINB
#define PAT_MINB 0
#endif
#if PAT_MINB > 0
#define PAT_LB __launch_bounds__(ROWS_PER_CTA, PAT_MINB)
#else
#define PAT_LB __launch_bounds__(ROWS_PER_CTA)
#endif
template <typename ID>
__global__ void PAT_LB k_level_pat(Ctx c, int l) {
  const SolverState* st = c.st;
  if (st->done) return;
  const int sbar = st->s_bar;
  if (l >= sbar) return;
  const PatSmem T = load_patterns(c);
  const int sigma = c.cfg->sigma;
  const double th = st->prm.th[l], ga = st->prm.ga[l], mu = st->prm.mu[l - 1];
  const bool use_mu = !(mu == 0.0);  // basis.py:217 `if mu != 0.0` (NaN counts)
  const bool do_r = l < sbar - 1;
  const double* Pl = c.Y + (int64_t)l * c.ld;
  const double* Pm = Pl - c.ld;
  double* Pn = c.Y + (int64_t)(l + 1) * c.ld;
  const double* Rl = c.Y + (int64_t)(sigma + 1 + l) * c.ld;
  const double* Rm = Rl - c.ld;
  double* Rn = c.Y + (int64_t)(sigma + 2 + l) * c.ld;
  int bad = 0;
  const int64_t plim = lvl_p_rows(c, sigma, l), rlim = lvl_r_rows(c, sigma, l);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int pid_next = i < plim ? row_pattern<ID>(c, i) : 0;  // ids one row ahead
  for (; i < plim; i += stride) {
    const int pid = pid_next;
    {
      const double* pf[2] = {Pl, Rl};
      prefetch_next<2>(c, i, stride, pf);
    }
    if (i + stride < plim) pid_next = row_pattern<ID>(c, i + stride);
    const int b = T.ptr[pid], e = T.ptr[pid + 1];
    double acc[2];
    const double* xs[2] = {Pl, Rl};
    const bool rrow = do_r && i < rlim;
    if (rrow)
      row_dot_p<2>(T, b, e, (int)i, xs, acc);
    else
      row_dot_p<1>(T, b, e, (int)i, xs, acc);
    const double wp = recur(acc[0], Pl[i], use_mu ? Pm[i] : 0.0, th, ga, mu, use_mu);
    Pn[i] = wp;
    bad |= !finite(wp);
    if (rrow) {
      const double wr = recur(acc[1], Rl[i], use_mu ? Rm[i] : 0.0, th, ga, mu, use_mu);
      Rn[i] = wr;
      bad |= !finite(wr);
    }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&c.st->breakdown, 1);
}

// Superset-mask pattern kernels: k_level0_pat / k_level_pat with the row sum
// unrolled over the union of offsets (row_dot_m).  Same rows, same order of
// rounded operations: bit-identical to the table-walking kernels above.
#ifndef SS_MINB
#define SS_MINB 0
#endif
#if SS_MINB > 0
#define SS_LB __launch_bounds__(ROWS_PER_CTA, SS_MINB)
#else
#define SS_LB __launch_bounds__(ROWS_PER_CTA)
#endif
template <typename ID, int NE>
__global__ void SS_LB k_level0_ss(Ctx c) {
  __shared__ double sm[ROWS_PER_CTA / 32];
  const SolverState* st = c.st;
  if (st->done) return;
  const SsSmem S = load_ss(c);
  const int sbar = st->s_bar;
  const int sigma = c.cfg->sigma;
  const double th = st->prm.th[0], ga = st->prm.ga[0];
  const bool do_r = sbar >= 2;
  const double* P0 = c.Y;
  double* P1 = c.Y + c.ld;
  const double* R0 = c.Y + (int64_t)(sigma + 1) * c.ld;
  double* R1 = c.Y + (int64_t)(sigma + 2) * c.ld;
  double tt = 0.0, rr = 0.0;
  int bad = 0;
  const int64_t n_own = c.n_own, plim = lvl_p_rows(c, sigma, 0), rlim = lvl_r_rows(c, sigma, 0);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int pid_next = i < plim ? row_pattern<ID>(c, i) : 0;
  for (; i < plim; i += stride) {
    const int pid = pid_next;
    {
      const double* pf[3] = {c.x, P0, R0};
      prefetch_next<3>(c, i, stride, pf);
    }
    if (i + stride < plim) pid_next = row_pattern<ID>(c, i + stride);
    double acc[3];
    const double* xs[3] = {c.x, P0, R0};
    const bool rrow = do_r && i < rlim;
    if (rrow)
      row_dot_m<3, NE>(c, S, pid, i, xs, acc);
    else
      row_dot_m<2, NE>(c, S, pid, i, xs, acc);
    const double p = P0[i];
    if (i < n_own) {
      const double r = R0[i];
      const double t = __dsub_rn(c.b[i], acc[0]);
      tt = fma(t, t, tt);
      rr = fma(r, r, rr);
    }
    const double wp = recur(acc[1], p, 0.0, th, ga, 0.0, false);
    P1[i] = wp;
    bad |= !finite(wp);
    if (rrow) {
      const double wr = recur(acc[2], R0[i], 0.0, th, ga, 0.0, false);
      R1[i] = wr;
      bad |= !finite(wr);
    }
  }
  tt = block_sum<ROWS_PER_CTA>(tt, sm);
  rr = block_sum<ROWS_PER_CTA>(rr, sm);
  if (threadIdx.x == 0) {
    c.part_t[blockIdx.x] = tt;
    c.part_r[blockIdx.x] = rr;
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&c.st->breakdown, 1);
}

template <typename ID, int NE>
__global__ void SS_LB k_level_ss(Ctx c, int l) {
  const SolverState* st = c.st;
  if (st->done) return;
  const int sbar = st->s_bar;
  if (l >= sbar) return;
  const SsSmem S = load_ss(c);
  const int sigma = c.cfg->sigma;
  const double th = st->prm.th[l], ga = st->prm.ga[l], mu = st->prm.mu[l - 1];
  const bool use_mu = !(mu == 0.0);  // basis.py:217 `if mu != 0.0` (NaN counts)
  const bool do_r = l < sbar - 1;
  const double* Pl = c.Y + (int64_t)l * c.ld;
  const double* Pm = Pl - c.ld;
  double* Pn = c.Y + (int64_t)(l + 1) * c.ld;
  const double* Rl = c.Y + (int64_t)(sigma + 1 + l) * c.ld;
  const double* Rm = Rl - c.ld;
  double* Rn = c.Y + (int64_t)(sigma + 2 + l) * c.ld;
  int bad = 0;
  const int64_t plim = lvl_p_rows(c, sigma, l), rlim = lvl_r_rows(c, sigma, l);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int pid_next = i < plim ? row_pattern<ID>(c, i) : 0;
  for (; i < plim; i += stride) {
    const int pid = pid_next;
    {
      const double* pf[2] = {Pl, Rl};
      prefetch_next<2>(c, i, stride, pf);
    }
    if (i + stride < plim) pid_next = row_pattern<ID>(c, i + stride);
    double acc[2];
    const double* xs[2] = {Pl, Rl};
    const bool rrow = do_r && i < rlim;
    if (rrow)
      row_dot_m<2, NE>(c, S, pid, i, xs, acc);
    else
      row_dot_m<1, NE>(c, S, pid, i, xs, acc);
    const double wp = recur(acc[0], Pl[i], use_mu ? Pm[i] : 0.0, th, ga, mu, use_mu);
    Pn[i] = wp;
    bad |= !finite(wp);
    if (rrow) {
      const double wr = recur(acc[1], Rl[i], use_mu ? Rm[i] : 0.0, th, ga, mu, use_mu);
      Rn[i] = wr;
      bad |= !finite(wr);
    }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&c.st->breakdown, 1);
}

// ---------------------------------------------------------------------------
// Plane-march pattern kernels (Ctx::zm_*).  The union of offsets is
// [-S, ..., 0, ..., +S] (a stencil: S is the plane stride).  A work item is
// 256 consecutive columns c (c = row mod S) x zm_zc consecutive steps; each
// thread walks its column, keeping x[r - S], x[r], x[r + S] in registers, so
// per row and vector one coalesced load (the plane ahead) replaces three
// gathers; the other slots are gathered as in row_dot_m.  The adds run over
// the slots in union order = stored order, absent slots adding +0.0 (exact,
// see row_dot_m): bit-identical to the other level kernels.
// plane table of a row-partitioned march (Ctx::zm_base) in dynamic shared
// memory after the pattern table (load_ss); nullptr: plane z starts at z * S.
// Callers run load_ss first (its barrier also covers this copy: the copy is
// issued before it by the same threads -- see k_level0_zm / k_level_zm).
__device__ __forceinline__ int* zm_plane_smem(const Ctx& c) {
  extern __shared__ __align__(16) double psm[];
  return reinterpret_cast<int*>(reinterpret_cast<char*>(psm) + ss_smem_bytes_dev(c.pat_np));
}
__device__ __forceinline__ void zm_plane_copy(const Ctx& c) {
  if (!c.zm_base) return;
  int* sb = zm_plane_smem(c);
  for (int i = threadIdx.x; i < c.zm_np; i += blockDim.x) sb[i] = __ldg(c.zm_base + i);
}
__device__ __forceinline__ const int* zm_plane_table(const Ctx& c) {
  return c.zm_base ? zm_plane_smem(c) : nullptr;
}

#ifndef ZM_L2PF  // per-thread L2 prefetch of the plane ZM_L2PF steps ahead (c5w: 1 -> +1.5 %, 2 -> -1.3 %, 3 -> -0.6 %, 4-8: 0)
#define ZM_L2PF 2
#endif
#ifndef ZM_PIPE  // plane-ahead loads one step early (measured slower: registers)
#define ZM_PIPE 0
#endif
template <bool UNIT>
__device__ __forceinline__ double recur_t(double ay, double y, double y2, double th, double ga,
                                          double mu, bool use_mu) {
  double w = __dsub_rn(ay, __dmul_rn(th, y));
  if (use_mu) w = __dsub_rn(w, __dmul_rn(mu, y2));
  return UNIT ? w : __ddiv_rn(w, ga);
}

// one column of one work item.  NV input vectors xs[0..NV) (level 0: x, P0, R0
// with NV = 3; else P_l, R_l with NV = 2, or P_l alone with NV = 1).
// MODE: ZM_LEVEL level l >= 1 (NV = 1 or 2 inputs, each with an output);
// ZM_L0 fused level 0 (x, P0, R0 in; P1, R1 out; ||b - A x||^2 and ||r||^2
// partials); ZM_L0PR level 0 without the residual (P0, R0 in, P1, R1 out,
// ||r||^2); ZM_RESID the true residual alone (x in, ||b - A x||^2, no output)
// RK: recurrence kind, bit 0 = non-unit gamma (IEEE division), bit 1 = mu != 0
// (two-back term) -- compile-time, so the Newton levels carry neither
enum { ZM_LEVEL = 0, ZM_L0 = 1, ZM_L0PR = 2, ZM_RESID = 3 };
template <typename ID, int NE, int NV, int MODE, int RK, bool TAB>
__device__ __forceinline__ void zm_column(const Ctx& c, const SsSmem& T, const int* __restrict__ sbase,
                                          int col, int z0, int z1,
                                          const double* const* __restrict__ xs,
                                          const double* const* __restrict__ ym,
                                          double* const* __restrict__ yo, double th, double ga,
                                          double mu, bool use_mu, int plim, int rlim, int& bad,
                                          double& tt, double& rr) {
  constexpr int KC = NE / 2;
  constexpr bool UNIT = (RK & 1) == 0, MU = (RK & 2) != 0 && MODE == ZM_LEVEL;
  constexpr int NO = MODE == ZM_RESID ? 0 : MODE == ZM_L0 ? NV - 1 : NV;  // output vectors
  constexpr int Q0 = MODE == ZM_L0 ? 1 : 0;  // first input vector with an output
  constexpr bool TT = MODE == ZM_L0 || MODE == ZM_RESID;  // ||b - A x||^2 (acc[0])
  constexpr bool RR = MODE == ZM_L0 || MODE == ZM_L0PR;   // ||r||^2 (the last input)
  // 32-bit row indices (plan.cu enables the march only for ld + S < 2^31).
  // Plane z of the walk starts at local row sbase[z] (a row-partitioned plan:
  // owned planes, then ghost planes by depth) or z * S (sbase == nullptr).
  // Vectors hold ld >= local rows entries.
  const int S = (int)c.zm_S, n = (int)(c.ld < INT32_MAX ? c.ld : INT32_MAX), n_own = (int)c.n_own;
  const int np = c.zm_np;
  if (z1 > np) z1 = np;
  auto row_of = [&](int z) { return (TAB ? sbase[z] : z * S) + col; };
  int r = row_of(z0);
  double pv[NV], cu[NV];
  {
    const int rp = z0 > 0 ? row_of(z0 - 1) : -1;
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      pv[q] = rp >= 0 && rp < n ? __ldg(xs[q] + rp) : 0.0;
      cu[q] = r < n ? __ldg(xs[q] + r) : 0.0;
    }
  }
  // row ids two steps ahead and the row of the next plane one step ahead
  const ID* pidp = reinterpret_cast<const ID*>(c.pid);
  int r1 = z0 + 1 < np ? row_of(z0 + 1) : n;  // row of plane z + 1
  int pid_cur = r < plim ? (int)__ldg(pidp + r) : 0;
  int pid_n1 = (z0 + 1 < z1 && r1 < plim) ? (int)__ldg(pidp + r1) : 0;
  for (int z = z0; z < z1; ++z) {
    const int pid = pid_cur;
    const int r2 = z + 2 < np ? row_of(z + 2) : n;
    const int pid_n2 = (z + 2 < z1 && r2 < plim) ? (int)__ldg(pidp + r2) : 0;
    double nx[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) nx[q] = r1 < n ? __ldg(xs[q] + r1) : 0.0;
#if ZM_L2PF > 0
    if (z + ZM_L2PF < np) {
      const int rf = row_of(z + ZM_L2PF);
      if (rf < n) {
#pragma unroll
        for (int q = 0; q < NV; ++q) asm volatile("prefetch.global.L2 [%0];" ::"l"(xs[q] + rf));
        if (TT && rf < n_own) asm volatile("prefetch.global.L2 [%0];" ::"l"(c.b + rf));
      }
    }
#endif
    if (r < plim) {
      const bool rrow = r < rlim;  // the last vector (R) is produced on this row
      // Absent slots carry the value 0.0 in the pattern table; they read the
      // row's own entry (offset 0: always in range) or the register slot as
      // is.  Every input a live level reads is finite (a non-finite column
      // ends the solve: basis.py:220, adaptive.py:146), so an absent slot adds
      // 0.0 * x = +-0.0, which leaves any partial sum csr_matvec can hold
      // unchanged (a sum that starts at +0.0 is never -0.0 under
      // round-to-nearest): bit-identical to skipping the slot.
      double xb[NV][NE];
      const int4 eo = T.eoff[pid];  // middle-slot offsets of this row (0: absent)
#pragma unroll
      for (int k = 1; k < NE - 1; ++k) {
        if (k == KC) continue;
        const int o = NE == 7 ? (k == 1 ? eo.x : k == 2 ? eo.y : k == 4 ? eo.z : eo.w)
                              : (k == 1 ? eo.x : eo.y);
#pragma unroll
        for (int q = 0; q < NV; ++q) xb[q][k] = __ldg(xs[q] + (r + o));
      }
#pragma unroll
      for (int q = 0; q < NV; ++q) {
        xb[q][0] = pv[q];
        xb[q][KC] = cu[q];
        xb[q][NE - 1] = nx[q];
      }
      const double2* v2 = reinterpret_cast<const double2*>(T.val + pid * SS_MAX_NE);
      double acc[NV];
#pragma unroll
      for (int q = 0; q < NV; ++q) acc[q] = 0.0;
#pragma unroll
      for (int k2 = 0; k2 < (NE + 1) / 2; ++k2) {
        const double2 vv = v2[k2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int k = 2 * k2 + h;
          if (k < NE) {
            const double v = h ? vv.y : vv.x;
#pragma unroll
            for (int q = 0; q < NV; ++q) acc[q] = __dadd_rn(acc[q], __dmul_rn(v, xb[q][k]));
          }
        }
      }
      if (TT && r < n_own) {
        const double t = __dsub_rn(c.b[r], acc[0]);
        tt = fma(t, t, tt);
      }
      if (RR && r < n_own) rr = fma(cu[NV - 1], cu[NV - 1], rr);
#pragma unroll
      for (int q = 0; q < NO; ++q) {
        if (q == NO - 1 && NO > 1 && !rrow) break;
        const double y2 = MU ? ym[q][r] : 0.0;
        const double w = recur_t<UNIT>(acc[Q0 + q], cu[Q0 + q], y2, th, ga, mu, MU);
        yo[q][r] = w;
        bad |= !finite(w);
      }
    }
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      pv[q] = cu[q];
      cu[q] = nx[q];
    }
    pid_cur = pid_n1;
    pid_n1 = pid_n2;
    r = r1;
    r1 = r2;
  }
}

template <typename ID, int NE, int NV, int MODE, int RK>
__device__ __forceinline__ void zm_items(const Ctx& c, int lvl, const SsSmem& T,
                                         const double* const* xs,
                                         const double* const* ym, double* const* yo, double th,
                                         double ga, double mu, bool use_mu, int64_t plim,
                                         int64_t rlim, int& bad, double& tt, double& rr) {
  // level 0 and the residual use fixed stripes with their own item size
  // (zm_zc0: whole rounds of items over the grid), levels >= 1 zm_zc
  const bool l0 = MODE != ZM_LEVEL;
  const int items = (int)(l0 ? c.zm_items0 : c.zm_items), ncb = c.zm_ncb;
  const int zcs = l0 ? c.zm_zc0 : c.zm_zc, S = (int)c.zm_S;
  const int* sbase = zm_plane_table(c);
  // levels >= 1 with Ctx::zm_ctr: the CTA claims items from a per-level
  // counter instead of a fixed stripe, so a CTA that started late (its SM
  // slot held by a Leja-point kernel of the side branch) takes fewer items
  // instead of delaying the whole level.  The row arithmetic is unchanged.
  // (only while the Leja chain of this block runs: st->leja_on; a Chebyshev
  // or monomial basis has no side branch and keeps the fixed stripes)
  const bool dyn = MODE == ZM_LEVEL && c.zm_ctr != nullptr && c.st->leja_on;
  __shared__ int s_claim;
  unsigned* ctr = dyn ? c.zm_ctr + 2 * lvl : nullptr;
  int it = blockIdx.x;
  if (dyn) {
    if (threadIdx.x == 0) s_claim = (int)atomicAdd(ctr, 1u);
    __syncthreads();
    it = s_claim;
  }
  for (; it < items;) {
    const int cb = it % ncb, zc = it / ncb;
    int col;
    if (c.zm_o > 0) {
      // 2-D tile of the plane: 32 consecutive columns per warp (x), the 8
      // warps on consecutive lines of stride zm_o (y), so a row's +-zm_o
      // neighbours are mostly rows another warp of this CTA just loaded (L1)
      const int ntx = c.zm_o >> 5;
      const int ty = (cb / ntx) * (ROWS_PER_CTA / 32) + (threadIdx.x >> 5);
      col = ty * c.zm_o + (cb % ntx) * 32 + (threadIdx.x & 31);
      if (ty >= S / c.zm_o) goto next_item;
    } else {
      col = cb * ROWS_PER_CTA + threadIdx.x;
    }
    if (col >= S) goto next_item;
    {
      const int z0 = zc * zcs;
      if (sbase)  // plane table (partitioned) or arithmetic planes, a compile-time choice
        zm_column<ID, NE, NV, MODE, RK, true>(c, T, sbase, col, z0, z0 + zcs, xs, ym, yo, th, ga,
                                              mu, use_mu, (int)plim, (int)rlim, bad, tt, rr);
      else
        zm_column<ID, NE, NV, MODE, RK, false>(c, T, sbase, col, z0, z0 + zcs, xs, ym, yo, th, ga,
                                               mu, use_mu, (int)plim, (int)rlim, bad, tt, rr);
    }
  next_item:
    if (dyn) {
      __syncthreads();  // every thread has read s_claim
      if (threadIdx.x == 0) s_claim = (int)atomicAdd(ctr, 1u);
      __syncthreads();
      it = s_claim;
    } else {
      it += gridDim.x;
    }
  }
  if (dyn && threadIdx.x == 0 && atomicAdd(ctr + 1, 1u) == gridDim.x - 1) {
    atomicExch(ctr, 0u);  // the last CTA out resets the counters for the next launch
    atomicExch(ctr + 1, 0u);
  }
}

// the level's column pointers, formed on the host: kept opaque to the
// compiler's index arithmetic, so each gather is one wide add off a base
// register instead of a re-derived column * ld product
struct ZmPtrs {
  const double* xs[3];
  const double* ym[2];
  double* yo[2];
};

inline ZmPtrs zm_ptrs(const Ctx& c, int l, int sigma) {
  ZmPtrs z;
  const int64_t ld = c.ld;
  if (l == 0) {
    z.xs[0] = c.x;
    z.xs[1] = c.Y;
    z.xs[2] = c.Y + (int64_t)(sigma + 1) * ld;
    z.ym[0] = z.ym[1] = nullptr;
    z.yo[0] = c.Y + ld;
    z.yo[1] = c.Y + (int64_t)(sigma + 2) * ld;
  } else {
    z.xs[0] = c.Y + (int64_t)l * ld;
    z.xs[1] = c.Y + (int64_t)(sigma + 1 + l) * ld;
    z.xs[2] = nullptr;
    z.ym[0] = z.xs[0] - ld;
    z.ym[1] = z.xs[1] - ld;
    z.yo[0] = c.Y + (int64_t)(l + 1) * ld;
    z.yo[1] = c.Y + (int64_t)(sigma + 2 + l) * ld;
  }
  return z;
}

#ifndef ZM0_MINB  // 64 registers, no spills: 4 CTAs/SM (1.52 vs 1.58 ms/outer at 3)
#define ZM0_MINB 4
#endif
template <typename ID, int NE, bool SPLIT>
__global__ void __launch_bounds__(ROWS_PER_CTA, ZM0_MINB) k_level0_zm(Ctx c, ZmPtrs zp) {
  __shared__ double sm[ROWS_PER_CTA / 32];
  const SolverState* st = c.st;
  if (st->done) return;
  zm_plane_copy(c);
  const SsSmem T = load_ss(c);
  const int sbar = st->s_bar;
  const int sigma = c.cfg->sigma;
  const double th = st->prm.th[0], ga = st->prm.ga[0];
  const bool do_r = sbar >= 2;
  double* yo[2] = {zp.yo[0], zp.yo[1]};
  const double* xs[3] = {zp.xs[0], zp.xs[1], zp.xs[2]};
  double tt = 0.0, rr = 0.0;
  int bad = 0;
  const int64_t plim = lvl_p_rows(c, sigma, 0), rlim = do_r ? lvl_r_rows(c, sigma, 0) : 0;
  if (SPLIT) {  // the true residual runs beside the levels (k_resid_zm)
    const double* xs2[2] = {xs[1], xs[2]};
    if (ga == 1.0)
      zm_items<ID, NE, 2, ZM_L0PR, 0>(c, 0, T, xs2, nullptr, yo, th, ga, 0.0, false, plim, rlim, bad, tt, rr);
    else
      zm_items<ID, NE, 2, ZM_L0PR, 1>(c, 0, T, xs2, nullptr, yo, th, ga, 0.0, false, plim, rlim, bad, tt, rr);
  } else if (ga == 1.0) {
    zm_items<ID, NE, 3, ZM_L0, 0>(c, 0, T, xs, nullptr, yo, th, ga, 0.0, false, plim, rlim, bad, tt, rr);
  } else {
    zm_items<ID, NE, 3, ZM_L0, 1>(c, 0, T, xs, nullptr, yo, th, ga, 0.0, false, plim, rlim, bad, tt, rr);
  }
  rr = block_sum<ROWS_PER_CTA>(rr, sm);
  if (!SPLIT) tt = block_sum<ROWS_PER_CTA>(tt, sm);
  if (threadIdx.x == 0) {
    if (!SPLIT) c.part_t[blockIdx.x] = tt;  // split: k_resid_zm writes these slots
    c.part_r[blockIdx.x] = rr;
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&c.st->breakdown, 1);
}

// the true residual t = b - A x of the outer loop (adaptive.py:138) on its own:
// ||t||^2 partials over the owned rows into part_t (same grid as level 0).
// It needs only x and b, so the outer-loop graph runs it on a side branch
// beside the matrix-powers levels (joined before the Gram kernel packs the
// norms); the row sums are the same rounded operations as everywhere.
template <typename ID, int NE>
__global__ void __launch_bounds__(ROWS_PER_CTA, ZM0_MINB) k_resid_zm(Ctx c, ZmPtrs zp) {
  __shared__ double sm[ROWS_PER_CTA / 32];
  const SolverState* st = c.st;
  if (st->done) return;
  zm_plane_copy(c);
  const SsSmem T = load_ss(c);
  const double* xs[1] = {zp.xs[0]};
  double tt = 0.0, rr = 0.0;
  int bad = 0;
  zm_items<ID, NE, 1, ZM_RESID, 0>(c, 0, T, xs, nullptr, nullptr, 0.0, 1.0, 0.0, false, c.n_own, 0,
                                   bad, tt, rr);
  tt = block_sum<ROWS_PER_CTA>(tt, sm);
  if (threadIdx.x == 0) c.part_t[blockIdx.x] = tt;
}

#ifndef ZM_MINB
#define ZM_MINB 4
#endif
template <typename ID, int NE>
__global__ void __launch_bounds__(ROWS_PER_CTA, ZM_MINB) k_level_zm(Ctx c, int l, ZmPtrs zp) {
  const SolverState* st = c.st;
  if (st->done) return;
  const int sbar = st->s_bar;
  if (l >= sbar) return;
  zm_plane_copy(c);
  const SsSmem T = load_ss(c);
  const int sigma = c.cfg->sigma;
  const double th = st->prm.th[l], ga = st->prm.ga[l], mu = st->prm.mu[l - 1];
  const bool use_mu = !(mu == 0.0);  // basis.py:217 `if mu != 0.0` (NaN counts)
  const bool do_r = l < sbar - 1;
  const double* xs[2] = {zp.xs[0], zp.xs[1]};
  const double* ym[2] = {zp.ym[0], zp.ym[1]};
  double* yo[2] = {zp.yo[0], zp.yo[1]};
  int bad = 0;
  double tt = 0.0, rr = 0.0;
  const int64_t plim = lvl_p_rows(c, sigma, l), rlim = lvl_r_rows(c, sigma, l);
  const int rk = (ga == 1.0 ? 0 : 1) | (use_mu ? 2 : 0);
#define ZM_RK(NV, RL)                                                                          \
  switch (rk) {                                                                                \
    case 0: zm_items<ID, NE, NV, ZM_LEVEL, 0>(c, l, T, xs, ym, yo, th, ga, mu, use_mu, plim, RL, bad, tt, rr); break; \
    case 1: zm_items<ID, NE, NV, ZM_LEVEL, 1>(c, l, T, xs, ym, yo, th, ga, mu, use_mu, plim, RL, bad, tt, rr); break; \
    case 2: zm_items<ID, NE, NV, ZM_LEVEL, 2>(c, l, T, xs, ym, yo, th, ga, mu, use_mu, plim, RL, bad, tt, rr); break; \
    default: zm_items<ID, NE, NV, ZM_LEVEL, 3>(c, l, T, xs, ym, yo, th, ga, mu, use_mu, plim, RL, bad, tt, rr); break; \
  }
  if (do_r) {
    ZM_RK(2, rlim)
  } else {
    ZM_RK(1, plim)
  }
#undef ZM_RK
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&c.st->breakdown, 1);
}

// ---------------------------------------------------------------------------
// Tile march with the plane in shared memory (levels >= 1; Ctx::zt_on).  For
// the 3-D stencil union [-S, -o, -1, 0, 1, o, S] a work item is a 32 x 8 tile
// of one plane (32 consecutive columns per warp, the 8 warps on lines of
// stride o) marched over zm_zc planes.  Each plane's tile values sit in
// shared memory (double-buffered by plane parity): the centres come from the
// threads' own registers (the previous step's plane-ahead load), the one-cell
// halo (two lines of 32, two columns of 8) is fetched by 96 threads with
// cp.async one step ahead, and one barrier per plane publishes both.  The
// +-1 / +-o slots are then shared-memory reads; -S and +S stay in registers.
// Same products and adds in union order: bit-identical.
constexpr int ZT_W = 34, ZT_H = 10, ZT_CELLS = ZT_W * ZT_H;  // tile + halo

__device__ __forceinline__ void cp_async8(void* dst, const void* src, bool in_range) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
               "r"(in_range ? 8 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

template <typename ID, int NV, int RK>
__device__ __forceinline__ void zt_item(const Ctx& c, const SsSmem& T, double* __restrict__ sb,
                                        int tile, int z0, int z1,
                                        const double* const* __restrict__ xs,
                                        const double* const* __restrict__ ym,
                                        double* const* __restrict__ yo, double th, double ga,
                                        double mu, int plim, int rlim, int& bad) {
  constexpr bool UNIT = (RK & 1) == 0, MU = (RK & 2) != 0;
  const int S = (int)c.zm_S, o = c.zm_o, n = (int)(c.ld < INT32_MAX ? c.ld : INT32_MAX);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int ntx = o >> 5;
  const int tx0 = (tile % ntx) * 32, ty0 = (tile / ntx) * 8;
  const int col = (ty0 + w) * o + tx0 + lane;
  // halo cell of this thread (threads 0..95): lines -1 / 8 (64), columns -1 / 32 (32)
  int hcol = 0, hcell = -1;
  if (threadIdx.x < 64) {
    const int hy = threadIdx.x < 32 ? -1 : 8;
    hcol = (ty0 + hy) * o + tx0 + lane;
    hcell = (hy + 1) * ZT_W + lane + 1;
  } else if (threadIdx.x < 96) {
    const int t = threadIdx.x - 64, hy = t & 7, hx = t < 8 ? -1 : t < 16 ? 32 : -2;
    if (hx != -2) {
      hcol = (ty0 + hy) * o + tx0 + hx;
      hcell = (hy + 1) * ZT_W + hx + 1;
    }
  }
  const int ccell = (w + 1) * ZT_W + lane + 1;
  int r = z0 * S + col;
  const double* px[NV];
  double* po[NV];
  const double* pm[NV];
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    px[q] = xs[q] + r;
    po[q] = yo[q] + r;
    pm[q] = ym[q] + r;
  }
  double pv[NV], cu[NV];
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    pv[q] = r >= S && r - S < n ? __ldg(px[q] - S) : 0.0;
    cu[q] = r < n ? __ldg(px[q]) : 0.0;
  }
  // plane z0: centres and halo into buffer z0 & 1
  {
    double* b = sb + (z0 & 1) * NV * ZT_CELLS;
#pragma unroll
    for (int q = 0; q < NV; ++q) b[q * ZT_CELLS + ccell] = cu[q];
    if (hcell >= 0) {
      const int hr = z0 * S + hcol;
      const bool ok = hr >= 0 && hr < n;
#pragma unroll
      for (int q = 0; q < NV; ++q) cp_async8(b + q * ZT_CELLS + hcell, xs[q] + (ok ? hr : 0), ok);
    }
    cp_async_commit();
  }
  const ID* pidp = reinterpret_cast<const ID*>(c.pid);
  // absent slots: value 0.0 times a finite in-range (or zero-filled) entry
  int pid_cur = r < plim ? (int)__ldg(pidp + r) : 0;
  int pid_n1 = (z0 + 1 < z1 && r + S < plim) ? (int)__ldg(pidp + r + S) : 0;
  for (int z = z0; z < z1; ++z) {
    cp_async_wait_all();
    __syncthreads();  // plane z's centres and halo visible; plane z-1's buffer free
    const double* b = sb + (z & 1) * NV * ZT_CELLS;
    double* bn = sb + ((z + 1) & 1) * NV * ZT_CELLS;
    if (z + 1 < z1) {
      if (hcell >= 0) {
        const int hr = (z + 1) * S + hcol;
        const bool ok = hr >= 0 && hr < n;
#pragma unroll
        for (int q = 0; q < NV; ++q) cp_async8(bn + q * ZT_CELLS + hcell, xs[q] + (ok ? hr : 0), ok);
      }
      cp_async_commit();
    }
    const int pid = pid_cur;
    const int pid_n2 = (z + 2 < z1 && r + 2 * S < plim) ? (int)__ldg(pidp + r + 2 * S) : 0;
    double nx[NV];
    const bool hasn = r + S < n;
#pragma unroll
    for (int q = 0; q < NV; ++q) nx[q] = hasn ? __ldg(px[q] + S) : 0.0;
    if (r < plim) {
      const bool rrow = r < rlim;
      const double2* v2 = reinterpret_cast<const double2*>(T.val + pid * SS_MAX_NE);
      const double2 v01 = v2[0], v23 = v2[1], v45 = v2[2], v6 = v2[3];
      double acc[NV];
#pragma unroll
      for (int q = 0; q < NV; ++q) {
        const double* bq = b + q * ZT_CELLS + ccell;
        const double xo_m = bq[-ZT_W], x1_m = bq[-1], x1_p = bq[1], xo_p = bq[ZT_W];
        double a = __dadd_rn(0.0, __dmul_rn(v01.x, pv[q]));
        a = __dadd_rn(a, __dmul_rn(v01.y, xo_m));
        a = __dadd_rn(a, __dmul_rn(v23.x, x1_m));
        a = __dadd_rn(a, __dmul_rn(v23.y, cu[q]));
        a = __dadd_rn(a, __dmul_rn(v45.x, x1_p));
        a = __dadd_rn(a, __dmul_rn(v45.y, xo_p));
        acc[q] = __dadd_rn(a, __dmul_rn(v6.x, nx[q]));
      }
#pragma unroll
      for (int q = 0; q < NV; ++q) {
        if (q == NV - 1 && NV > 1 && !rrow) break;
        const double y2 = MU ? *pm[q] : 0.0;
        const double wv = recur_t<UNIT>(acc[q], cu[q], y2, th, ga, mu, MU);
        *po[q] = wv;
        bad |= !finite(wv);
      }
    }
    if (z + 1 < z1) {
#pragma unroll
      for (int q = 0; q < NV; ++q) bn[q * ZT_CELLS + ccell] = nx[q];
    }
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      pv[q] = cu[q];
      cu[q] = nx[q];
      px[q] += S;
      po[q] += S;
      if (MU) pm[q] += S;
    }
    pid_cur = pid_n1;
    pid_n1 = pid_n2;
    r += S;
  }
  __syncthreads();  // the next item reuses the buffers
}

template <typename ID>
__global__ void __launch_bounds__(ROWS_PER_CTA, ZM_MINB) k_level_zt(Ctx c, int l, ZmPtrs zp) {
  __shared__ __align__(16) double sb[2 * 2 * ZT_CELLS];
  const SolverState* st = c.st;
  if (st->done) return;
  const int sbar = st->s_bar;
  if (l >= sbar) return;
  const SsSmem T = load_ss(c);
  const int sigma = c.cfg->sigma;
  const double th = st->prm.th[l], ga = st->prm.ga[l], mu = st->prm.mu[l - 1];
  const bool use_mu = !(mu == 0.0);  // basis.py:217 `if mu != 0.0` (NaN counts)
  const bool do_r = l < sbar - 1;
  const double* xs[2] = {zp.xs[0], zp.xs[1]};
  const double* ym[2] = {zp.ym[0], zp.ym[1]};
  double* yo[2] = {zp.yo[0], zp.yo[1]};
  int bad = 0;
  const int plim = (int)lvl_p_rows(c, sigma, l), rlim = (int)lvl_r_rows(c, sigma, l);
  const int rk = (ga == 1.0 ? 0 : 1) | (use_mu ? 2 : 0);
  const int items = (int)c.zm_items, ncb = c.zm_ncb, zcs = c.zm_zc;
  const int steps = (int)((c.n + c.zm_S - 1) / c.zm_S);
  for (int it = blockIdx.x; it < items; it += gridDim.x) {
    const int tile = it % ncb, z0 = (it / ncb) * zcs;
    const int z1 = min(z0 + zcs, steps);
#define ZT_CALL(NV, RKV, RL) \
  zt_item<ID, NV, RKV>(c, T, sb, tile, z0, z1, xs, ym, yo, th, ga, mu, plim, RL, bad)
    if (do_r) {
      switch (rk) {
        case 0: ZT_CALL(2, 0, rlim); break;
        case 1: ZT_CALL(2, 1, rlim); break;
        case 2: ZT_CALL(2, 2, rlim); break;
        default: ZT_CALL(2, 3, rlim); break;
      }
    } else {
      switch (rk) {
        case 0: ZT_CALL(1, 0, plim); break;
        case 1: ZT_CALL(1, 1, plim); break;
        case 2: ZT_CALL(1, 2, plim); break;
        default: ZT_CALL(1, 3, plim); break;
      }
    }
#undef ZT_CALL
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&c.st->breakdown, 1);
}

// ---------------------------------------------------------------------------
// Row-pair plane march (levels >= 1; Ctx::zm_pair).  The union is the 2-D /
// 3-D stencil form [-S, (-o,) -1, 0, 1, (o,) S] with S and o even: a thread
// owns two adjacent columns (rows r, r + 1 with r even), so every even-offset
// slot is ONE aligned 16-byte load serving both rows, the +-1 slots of one
// row are the other row's centre, and only x[r - 1] and x[r + 2] are single
// loads: per vector and row pair 4 (5 in 3-D) load instructions instead of
// 10 (14).  Each row keeps its own pattern mask and values; products and adds
// in union order as everywhere else: bit-identical.
__device__ __forceinline__ double2 ld2(const double* p) {
  return __ldg(reinterpret_cast<const double2*>(p));
}

template <typename ID, int NE, int NV, int RK>
__device__ __forceinline__ void zp_column(const Ctx& c, const SsSmem& T, int col, int z0, int z1,
                                          const double* const* __restrict__ xs,
                                          const double* const* __restrict__ ym,
                                          double* const* __restrict__ yo, double th, double ga,
                                          double mu, bool use_mu, int plim, int rlim, int& bad) {
  static_assert(NE == 5 || NE == 7, "pair march: 2-D or 3-D stencil unions");
  constexpr bool UNIT = (RK & 1) == 0, MU = (RK & 2) != 0;
  constexpr bool D3 = NE == 7;
  constexpr int KM1 = D3 ? 2 : 1, KC = NE / 2, KP1 = KC + 1;  // slots of -1, 0, +1
  const int S = (int)c.zm_S, n = (int)(c.ld < INT32_MAX ? c.ld : INT32_MAX);
  const int o = D3 ? c.ss_off[NE - 2] : 0;
  int r = z0 * S + col;  // even
  if (r >= plim) return;
  const double* px[NV];
  double* po[NV];
  const double* pm[NV];
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    px[q] = xs[q] + r;
    po[q] = yo[q] + r;
    pm[q] = ym[q] + r;
  }
  double2 pv[NV], cu[NV];
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    pv[q] = r >= S ? ld2(px[q] - S) : make_double2(0.0, 0.0);
    cu[q] = ld2(px[q]);
  }
#if ZM_PIPE
  double2 nxa[NV];
#pragma unroll
  for (int q = 0; q < NV; ++q) nxa[q] = r + S < n ? ld2(px[q] + S) : make_double2(0.0, 0.0);
#endif
  const ID* pidp = reinterpret_cast<const ID*>(c.pid) + r;
  int p0 = (int)__ldg(pidp), p1 = (int)__ldg(pidp + 1);
  int q0 = 0, q1 = 0;
  if (z0 + 1 < z1 && r + S < plim) {
    q0 = (int)__ldg(pidp + S);
    q1 = (int)__ldg(pidp + S + 1);
  }
  unsigned mc0 = T.mask[p0], mc1 = T.mask[p1];
  for (int z = z0; z < z1 && r < plim; ++z) {
    const int pid0 = p0, pid1 = p1;
    const unsigned m0 = mc0, m1 = mc1;
    int t0 = 0, t1 = 0;
    if (z + 2 < z1 && r + 2 * S < plim) {
      t0 = (int)__ldg(pidp + 2 * S);
      t1 = (int)__ldg(pidp + 2 * S + 1);
    }
    const unsigned mu01 = m0 | m1;
    const bool row1 = r + 1 < plim;
    const bool rr0 = r < rlim, rr1 = r + 1 < rlim;
#if ZM_PIPE
    const bool hasn = z + 1 < z1 && r + 2 * S < n;
#else
    const bool hasn = r + S < n;
#endif
    double2 nx[NV], lo[NV], hi[NV];
    double lm1[NV], rp2[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      const bool want = q < NV - 1 || NV == 1 || rr0;  // the R vector only on R rows
#if ZM_PIPE
      nx[q] = nxa[q];
      nxa[q] = hasn ? ld2(px[q] + 2 * S) : make_double2(0.0, 0.0);
#else
      nx[q] = hasn ? ld2(px[q] + S) : make_double2(0.0, 0.0);
#endif
      lo[q] = hi[q] = make_double2(0.0, 0.0);
      if (D3) {
        if (want && (mu01 & 2u)) lo[q] = ld2(px[q] - o);
        if (want && (mu01 & (1u << (NE - 2)))) hi[q] = ld2(px[q] + o);
      }
      lm1[q] = (want && (m0 >> KM1) & 1u) ? __ldg(px[q] - 1) : 0.0;
      rp2[q] = (want && row1 && (m1 >> KP1) & 1u) ? __ldg(px[q] + 2) : 0.0;
    }
    // slot values of row r (.x) and row r + 1 (.y), absent slots 0.0
    double a[2][NV][NE];
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      a[0][q][0] = pv[q].x;
      a[1][q][0] = pv[q].y;
      if (D3) {
        a[0][q][1] = lo[q].x;
        a[1][q][1] = lo[q].y;
        a[0][q][NE - 2] = hi[q].x;
        a[1][q][NE - 2] = hi[q].y;
      }
      a[0][q][KM1] = lm1[q];
      a[1][q][KM1] = cu[q].x;
      a[0][q][KC] = cu[q].x;
      a[1][q][KC] = cu[q].y;
      a[0][q][KP1] = cu[q].y;
      a[1][q][KP1] = rp2[q];
      a[0][q][NE - 1] = nx[q].x;
      a[1][q][NE - 1] = nx[q].y;
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const unsigned m = h ? m1 : m0;
      const int pid = h ? pid1 : pid0;
      if (h == 1 && !row1) break;
      const double2* v2 = reinterpret_cast<const double2*>(T.val + pid * SS_MAX_NE);
      double acc[NV];
#pragma unroll
      for (int q = 0; q < NV; ++q) acc[q] = 0.0;
#pragma unroll
      for (int k2 = 0; k2 < (NE + 1) / 2; ++k2) {
        const double2 vv = v2[k2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int k = 2 * k2 + e;
          if (k < NE) {
            const double v = e ? vv.y : vv.x;
            const bool on = (m >> k) & 1u;
#pragma unroll
            for (int q = 0; q < NV; ++q)
              acc[q] = __dadd_rn(acc[q], __dmul_rn(v, on ? a[h][q][k] : 0.0));
          }
        }
      }
      const bool rrow = h ? rr1 : rr0;
#pragma unroll
      for (int q = 0; q < NV; ++q) {
        if (q == NV - 1 && NV > 1 && !rrow) break;
        const double y2 = MU ? pm[q][h] : 0.0;
        const double w = recur_t<UNIT>(acc[q], h ? cu[q].y : cu[q].x, y2, th, ga, mu, MU);
        po[q][h] = w;
        bad |= !finite(w);
      }
    }
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      pv[q] = cu[q];
      cu[q] = nx[q];
      px[q] += S;
      po[q] += S;
      if (MU) pm[q] += S;
    }
    p0 = q0;
    p1 = q1;
    mc0 = T.mask[q0];
    mc1 = T.mask[q1];
    q0 = t0;
    q1 = t1;
    pidp += S;
    r += S;
  }
}

template <typename ID, int NE, int NV, int RK>
__device__ __forceinline__ void zp_items(const Ctx& c, const SsSmem& T, const double* const* xs,
                                         const double* const* ym, double* const* yo, double th,
                                         double ga, double mu, bool use_mu, int64_t plim,
                                         int64_t rlim, int& bad) {
  const int S = (int)c.zm_S, zcs = c.zm_zc, items = (int)c.zp_items;
  const int ncb = (S + 2 * ROWS_PER_CTA - 1) / (2 * ROWS_PER_CTA);  // 512 columns per item
  for (int it = blockIdx.x; it < items; it += gridDim.x) {
    const int cb = it % ncb, zc = it / ncb;
    const int col = 2 * (cb * ROWS_PER_CTA + threadIdx.x);
    if (col >= S) continue;
    const int z0 = zc * zcs;
    zp_column<ID, NE, NV, RK>(c, T, col, z0, z0 + zcs, xs, ym, yo, th, ga, mu, use_mu, (int)plim,
                                (int)rlim, bad);
  }
}

#ifndef ZP_MINB
#define ZP_MINB 0
#endif
#if ZP_MINB > 0
#define ZP_LB __launch_bounds__(ROWS_PER_CTA, ZP_MINB)
#else
#define ZP_LB __launch_bounds__(ROWS_PER_CTA)
#endif
template <typename ID, int NE>
__global__ void ZP_LB k_level_zp(Ctx c, int l, ZmPtrs zp) {
  const SolverState* st = c.st;
  if (st->done) return;
  const int sbar = st->s_bar;
  if (l >= sbar) return;
  const SsSmem T = load_ss(c);
  const int sigma = c.cfg->sigma;
  const double th = st->prm.th[l], ga = st->prm.ga[l], mu = st->prm.mu[l - 1];
  const bool use_mu = !(mu == 0.0);  // basis.py:217 `if mu != 0.0` (NaN counts)
  const bool do_r = l < sbar - 1;
  const double* xs[2] = {zp.xs[0], zp.xs[1]};
  const double* ym[2] = {zp.ym[0], zp.ym[1]};
  double* yo[2] = {zp.yo[0], zp.yo[1]};
  int bad = 0;
  const int64_t plim = lvl_p_rows(c, sigma, l), rlim = lvl_r_rows(c, sigma, l);
  const int rk = (ga == 1.0 ? 0 : 1) | (use_mu ? 2 : 0);
#define ZP_RK(NV, RL)                                                                       \
  switch (rk) {                                                                             \
    case 0: zp_items<ID, NE, NV, 0>(c, T, xs, ym, yo, th, ga, mu, use_mu, plim, RL, bad); break; \
    case 1: zp_items<ID, NE, NV, 1>(c, T, xs, ym, yo, th, ga, mu, use_mu, plim, RL, bad); break; \
    case 2: zp_items<ID, NE, NV, 2>(c, T, xs, ym, yo, th, ga, mu, use_mu, plim, RL, bad); break; \
    default: zp_items<ID, NE, NV, 3>(c, T, xs, ym, yo, th, ga, mu, use_mu, plim, RL, bad); break; \
  }
  if (do_r) {
    ZP_RK(2, rlim)
  } else {
    ZP_RK(1, plim)
  }
#undef ZP_RK
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&c.st->breakdown, 1);
}

// ---------------------------------------------------------------------------
// Value-stream stencil kernels (Ctx::vs_*): operators with a stencil's column
// structure but row-varying values (c4: 27-point variable coefficients) do not
// compress to patterns; here the column structure is the union of offsets
// (kernel parameters) and the values stream slot-major, coalesced, 8 bytes per
// slot and row -- no column indices, no row pointers (12 nnz + 4 n bytes of
// CSR become 8 ne n).  One row per thread, slots in union order = stored order,
// in chunks of VS_CHUNK (gathers of a chunk in flight together).  An absent
// slot has value 0.0 and gathers from the clamped index (in range, finite:
// see zm_column): adding 0.0 * x = +-0.0 is exact -- bit-identical to CSR.
#ifndef VS_CHUNK
#define VS_CHUNK 5  // slots per batch of gathers (c4j: 3.80 ms/outer; 9: 4.1, 14: 4.6, 27: 4.3)
#endif
template <int NV, int NE>
__device__ __forceinline__ void vs_row(const Ctx& c, int i, int nm1,
                                       const double* const* __restrict__ xs, double* acc) {
#pragma unroll
  for (int q = 0; q < NV; ++q) acc[q] = 0.0;
  const double* vp = c.vs_val + i;
  const int64_t ldv = c.ld;
#pragma unroll
  for (int k0 = 0; k0 < NE; k0 += VS_CHUNK) {
    double v[VS_CHUNK], xb[NV][VS_CHUNK];
#pragma unroll
    for (int kk = 0; kk < VS_CHUNK; ++kk) {
      const int k = k0 + kk;
      if (k < NE) {
        v[kk] = __ldg(vp + (int64_t)k * ldv);
        const int j = min(max(i + c.vs_off[k], 0), nm1);
#pragma unroll
        for (int q = 0; q < NV; ++q) xb[q][kk] = __ldg(xs[q] + j);
      }
    }
#pragma unroll
    for (int kk = 0; kk < VS_CHUNK; ++kk) {
      if (k0 + kk < NE) {
#pragma unroll
        for (int q = 0; q < NV; ++q) acc[q] = __dadd_rn(acc[q], __dmul_rn(v[kk], xb[q][kk]));
      }
    }
  }
}

template <int NE>
__global__ void __launch_bounds__(ROWS_PER_CTA) k_level0_vs(Ctx c, ZmPtrs zp) {
  __shared__ double sm[ROWS_PER_CTA / 32];
  const SolverState* st = c.st;
  if (st->done) return;
  const int sbar = st->s_bar;
  const int sigma = c.cfg->sigma;
  const double th = st->prm.th[0], ga = st->prm.ga[0];
  const bool do_r = sbar >= 2;
  const double* xs[3] = {zp.xs[0], zp.xs[1], zp.xs[2]};
  double tt = 0.0, rr = 0.0;
  int bad = 0;
  const int n_own = (int)c.n_own, plim = (int)lvl_p_rows(c, sigma, 0);
  const int rlim = do_r ? (int)lvl_r_rows(c, sigma, 0) : 0, nm1 = (int)c.n - 1;
  const int stride = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < plim; i += stride) {
    double acc[3];
    vs_row<3, NE>(c, i, nm1, xs, acc);
    const double p = xs[1][i], r = xs[2][i];
    if (i < n_own) {
      const double t = __dsub_rn(c.b[i], acc[0]);
      tt = fma(t, t, tt);
      rr = fma(r, r, rr);
    }
    const double wp = recur(acc[1], p, 0.0, th, ga, 0.0, false);
    zp.yo[0][i] = wp;
    bad |= !finite(wp);
    if (i < rlim) {
      const double wr = recur(acc[2], r, 0.0, th, ga, 0.0, false);
      zp.yo[1][i] = wr;
      bad |= !finite(wr);
    }
  }
  tt = block_sum<ROWS_PER_CTA>(tt, sm);
  rr = block_sum<ROWS_PER_CTA>(rr, sm);
  if (threadIdx.x == 0) {
    c.part_t[blockIdx.x] = tt;
    c.part_r[blockIdx.x] = rr;
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&c.st->breakdown, 1);
}

template <int NE>
__global__ void __launch_bounds__(ROWS_PER_CTA) k_level_vs(Ctx c, int l, ZmPtrs zp) {
  const SolverState* st = c.st;
  if (st->done) return;
  const int sbar = st->s_bar;
  if (l >= sbar) return;
  const int sigma = c.cfg->sigma;
  const double th = st->prm.th[l], ga = st->prm.ga[l], mu = st->prm.mu[l - 1];
  const bool use_mu = !(mu == 0.0);  // basis.py:217 `if mu != 0.0` (NaN counts)
  const bool do_r = l < sbar - 1;
  const int plim = (int)lvl_p_rows(c, sigma, l), rlim = (int)lvl_r_rows(c, sigma, l);
  const int nm1 = (int)c.n - 1;
  const int stride = gridDim.x * blockDim.x;
  int bad = 0;
  const double* xs[2] = {zp.xs[0], zp.xs[1]};
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < plim; i += stride) {
    double acc[2];
    const bool rrow = do_r && i < rlim;
    if (rrow)
      vs_row<2, NE>(c, i, nm1, xs, acc);
    else
      vs_row<1, NE>(c, i, nm1, xs, acc);
    const double wp = recur(acc[0], xs[0][i], use_mu ? zp.ym[0][i] : 0.0, th, ga, mu, use_mu);
    zp.yo[0][i] = wp;
    bad |= !finite(wp);
    if (rrow) {
      const double wr = recur(acc[1], xs[1][i], use_mu ? zp.ym[1][i] : 0.0, th, ga, mu, use_mu);
      zp.yo[1][i] = wr;
      bad |= !finite(wr);
    }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&c.st->breakdown, 1);
}

// ---------------------------------------------------------------------------
// Windowed pattern kernels.  A CTA walks 256-row tiles; for each tile one TMA
// bulk copy per input vector brings the contiguous window [base - R,
// base + 256 + R) into shared memory (with the tile's row ids), double
// buffered under an mbarrier, so every column within R of its row (the
// diagonal, +-1, +-nx of a stencil) is a shared-memory read; only farther
// columns are gathered from L2.  Same row arithmetic and order as the other
// kernels: bit-identical.
constexpr int WT = MT_ROWS;  // 256 rows per tile

__host__ __device__ __forceinline__ int win_len(int r) { return WT + 2 * r; }
__host__ __device__ __forceinline__ size_t win_stage_bytes(int r, int nvw, int pid_bytes) {
  return ((size_t)nvw * win_len(r) * 8 + (size_t)WT * pid_bytes + 15) / 16 * 16;
}
__host__ __device__ __forceinline__ size_t win_table_bytes(int np, int ne) {
  return (pattern_smem_bytes_dev(np, ne) + 15) / 16 * 16;
}

template <int NVW, typename ID>
struct WinPipe {
  unsigned char* base;  // stage 0
  size_t sb;
  uint64_t* bars;
  int r, wl;
  __device__ __forceinline__ double* win(int s, int q) const {
    return reinterpret_cast<double*>(base + s * sb) + (size_t)q * wl;
  }
  __device__ __forceinline__ const ID* ids(int s) const {
    return reinterpret_cast<const ID*>(base + s * sb + (size_t)NVW * wl * 8);
  }
  // thread 0: stage tile `tile` of the vectors into buffer s
  __device__ __forceinline__ void issue(const Ctx& c, const double* const* vecs, int64_t tile, int s) const {
    const int64_t t0 = tile * WT;
    const int64_t lo = t0 - r > 0 ? t0 - r : 0;
    const int64_t hi = t0 + WT + r < c.ld ? t0 + WT + r : c.ld;
    const uint32_t vb = (uint32_t)((hi - lo) * 8);
    const uint32_t ib = (uint32_t)(WT * sizeof(ID));
    mbar_arrive_tx(&bars[s], NVW * vb + ib);
#pragma unroll
    for (int q = 0; q < NVW; ++q) bulk_g2s(win(s, q) + (lo - (t0 - r)), vecs[q] + lo, vb, &bars[s]);
    bulk_g2s((void*)ids(s), reinterpret_cast<const ID*>(c.pid) + t0, ib, &bars[s]);
  }
};

// row sum of NV staged vectors: near columns from the window, far ones gathered
template <int NV, int NVW, typename ID>
__device__ __forceinline__ void row_dot_win(const PatSmem& T, const WinPipe<NVW, ID>& W, int s,
                                            int b, int e, int i, int tid,
                                            const double* const* __restrict__ xs, double* acc) {
  constexpr int B = NV >= 3 ? 4 : 8;
#pragma unroll
  for (int q = 0; q < NV; ++q) acc[q] = 0.0;
  const int r = W.r;
  for (int jj = b; jj < e; jj += B) {
    const int m = e - jj;
    double xb[NV][B];
#pragma unroll
    for (int k = 0; k < B; ++k) {
      const int off = T.off[jj + (k < m ? k : 0)];
      const bool near = off >= -r && off <= r;
      if (near) {
#pragma unroll
        for (int q = 0; q < NV; ++q) xb[q][k] = W.win(s, q)[tid + r + off];
      } else {
#pragma unroll
        for (int q = 0; q < NV; ++q) xb[q][k] = __ldg(xs[q] + i + off);
      }
    }
#pragma unroll
    for (int k = 0; k < B; ++k) {
      if (k < m) {
        const double v = T.val[jj + k];
#pragma unroll
        for (int q = 0; q < NV; ++q) acc[q] = __dadd_rn(acc[q], __dmul_rn(v, xb[q][k]));
      }
    }
  }
}

template <int NVW, typename ID, class Body>
__device__ __forceinline__ void win_tiles(const Ctx& c, int64_t nrows, const double* const* vecs,
                                          Body&& body) {
  extern __shared__ __align__(16) double psm[];
  __shared__ __align__(8) uint64_t bars[2];
  const PatSmem T = load_patterns(c);
  WinPipe<NVW, ID> W;
  W.base = reinterpret_cast<unsigned char*>(psm) + win_table_bytes(c.pat_np, c.pat_ne);
  W.r = c.win_r;
  W.wl = win_len(c.win_r);
  W.sb = win_stage_bytes(c.win_r, NVW, sizeof(ID));
  W.bars = bars;
  const int tid = threadIdx.x;
  const int64_t ntiles = (nrows + WT - 1) / WT;
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (tid == 0)
    for (int s = 0; s < 2; ++s) {
      const int64_t t = blockIdx.x + (int64_t)s * gridDim.x;
      if (t < ntiles) W.issue(c, vecs, t, s);
    }
  int64_t k = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++k) {
    const int s = (int)(k & 1);
    mbar_wait(&bars[s], (uint32_t)((k >> 1) & 1));
    const int64_t i = tile * WT + tid;
    if (i < nrows) body(T, W, s, i, tid, (int)W.ids(s)[tid]);
    __syncthreads();  // stage s free
    if (tid == 0) {
      const int64_t t = tile + 2 * (int64_t)gridDim.x;
      if (t < ntiles) {
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        W.issue(c, vecs, t, s);
      }
    }
  }
}

template <typename ID>
__global__ void __launch_bounds__(WT) k_level0_win(Ctx c) {
  __shared__ double sm[WT / 32];
  const SolverState* st = c.st;
  if (st->done) return;
  const int sbar = st->s_bar;
  const int sigma = c.cfg->sigma;
  const double th = st->prm.th[0], ga = st->prm.ga[0];
  const bool do_r = sbar >= 2;
  const double* P0 = c.Y;
  double* P1 = c.Y + c.ld;
  const double* R0 = c.Y + (int64_t)(sigma + 1) * c.ld;
  double* R1 = c.Y + (int64_t)(sigma + 2) * c.ld;
  double tt = 0.0, rr = 0.0;
  int bad = 0;
  const int64_t n_own = c.n_own, plim = lvl_p_rows(c, sigma, 0), rlim = lvl_r_rows(c, sigma, 0);
  const double* vecs[3] = {c.x, P0, R0};
  win_tiles<3, ID>(c, plim, vecs, [&](const PatSmem& T, const WinPipe<3, ID>& W, int s, int64_t i,
                                      int tid, int pid) {
    const int b = T.ptr[pid], e = T.ptr[pid + 1];
    const double p = W.win(s, 1)[tid + W.r], r = W.win(s, 2)[tid + W.r];
    double acc[3];
    if (do_r)
      row_dot_win<3>(T, W, s, b, e, (int)i, tid, vecs, acc);
    else
      row_dot_win<2>(T, W, s, b, e, (int)i, tid, vecs, acc);
    if (i < n_own) {
      const double t = __dsub_rn(c.b[i], acc[0]);
      tt = fma(t, t, tt);
      rr = fma(r, r, rr);
    }
    const double wp = recur(acc[1], p, 0.0, th, ga, 0.0, false);
    P1[i] = wp;
    bad |= !finite(wp);
    if (do_r && i < rlim) {
      const double wr = recur(acc[2], r, 0.0, th, ga, 0.0, false);
      R1[i] = wr;
      bad |= !finite(wr);
    }
  });
  tt = block_sum<WT>(tt, sm);
  rr = block_sum<WT>(rr, sm);
  if (threadIdx.x == 0) {
    c.part_t[blockIdx.x] = tt;
    c.part_r[blockIdx.x] = rr;
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&c.st->breakdown, 1);
}

template <typename ID>
__global__ void __launch_bounds__(WT) k_level_win(Ctx c, int l) {
  const SolverState* st = c.st;
  if (st->done) return;
  const int sbar = st->s_bar;
  if (l >= sbar) return;
  const int sigma = c.cfg->sigma;
  const double th = st->prm.th[l], ga = st->prm.ga[l], mu = st->prm.mu[l - 1];
  const bool use_mu = !(mu == 0.0);  // basis.py:217 `if mu != 0.0` (NaN counts)
  const bool do_r = l < sbar - 1;
  const double* Pl = c.Y + (int64_t)l * c.ld;
  const double* Pm = Pl - c.ld;
  double* Pn = c.Y + (int64_t)(l + 1) * c.ld;
  const double* Rl = c.Y + (int64_t)(sigma + 1 + l) * c.ld;
  const double* Rm = Rl - c.ld;
  double* Rn = c.Y + (int64_t)(sigma + 2 + l) * c.ld;
  int bad = 0;
  const int64_t plim = lvl_p_rows(c, sigma, l), rlim = lvl_r_rows(c, sigma, l);
  const double* vecs[2] = {Pl, Rl};
  win_tiles<2, ID>(c, plim, vecs, [&](const PatSmem& T, const WinPipe<2, ID>& W, int s, int64_t i,
                                      int tid, int pid) {
    const int b = T.ptr[pid], e = T.ptr[pid + 1];
    const bool rrow = do_r && i < rlim;
    double acc[2];
    if (rrow)
      row_dot_win<2>(T, W, s, b, e, (int)i, tid, vecs, acc);
    else
      row_dot_win<1>(T, W, s, b, e, (int)i, tid, vecs, acc);
    const double wp = recur(acc[0], W.win(s, 0)[tid + W.r], use_mu ? Pm[i] : 0.0, th, ga, mu, use_mu);
    Pn[i] = wp;
    bad |= !finite(wp);
    if (rrow) {
      const double wr = recur(acc[1], W.win(s, 1)[tid + W.r], use_mu ? Rm[i] : 0.0, th, ga, mu, use_mu);
      Rn[i] = wr;
      bad |= !finite(wr);
    }
  });
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&c.st->breakdown, 1);
}

// ---------------------------------------------------------------------------
// Level 0 of an outer loop: t = b - A x (norm partial), ||r0||^2 partial,
// P_1 and (if s_bar >= 2) R_1.
__global__ void __launch_bounds__(ROWS_PER_CTA) k_level0(Ctx c) {
  __shared__ double sm[ROWS_PER_CTA / 32];
  const SolverState* st = c.st;
  if (st->done) return;
  const int sbar = st->s_bar;
  const int sigma = c.cfg->sigma;
  const double th = st->prm.th[0], ga = st->prm.ga[0];
  const bool do_r = sbar >= 2;
  const double* P0 = c.Y;
  double* P1 = c.Y + c.ld;
  const double* R0 = c.Y + (int64_t)(sigma + 1) * c.ld;
  double* R1 = c.Y + (int64_t)(sigma + 2) * c.ld;
  double tt = 0.0, rr = 0.0;
  int bad = 0;
  const int64_t n_own = c.n_own, plim = lvl_p_rows(c, sigma, 0), rlim = lvl_r_rows(c, sigma, 0);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < plim; i += stride) {
    const int beg = c.rp[i], end = c.rp[i + 1];
    const double p = P0[i], r = R0[i];
    double acc[3];
    if (do_r) {
      const double* xs[3] = {c.x, P0, R0};
      row_dot<3>(c.col, c.val, beg, end, xs, acc);
    } else {
      const double* xs[2] = {c.x, P0};
      row_dot<2>(c.col, c.val, beg, end, xs, acc);
    }
    if (i < n_own) {
      const double t = __dsub_rn(c.b[i], acc[0]);
      tt = fma(t, t, tt);
      rr = fma(r, r, rr);
    }
    const double wp = recur(acc[1], p, 0.0, th, ga, 0.0, false);
    P1[i] = wp;
    bad |= !finite(wp);
    if (do_r && i < rlim) {
      const double wr = recur(acc[2], r, 0.0, th, ga, 0.0, false);
      R1[i] = wr;
      bad |= !finite(wr);
    }
  }
  tt = block_sum<ROWS_PER_CTA>(tt, sm);
  rr = block_sum<ROWS_PER_CTA>(rr, sm);
  if (threadIdx.x == 0) {
    c.part_t[blockIdx.x] = tt;
    c.part_r[blockIdx.x] = rr;
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&c.st->breakdown, 1);
}

// Level l >= 1: P_{l+1} (l < s_bar) and R_{l+1} (l < s_bar - 1).
template <bool DO_R>
__device__ __forceinline__ int level_rows(const Ctx& c, int l, int sigma, double th, double ga,
                                          double mu, bool use_mu) {
  const int64_t plim = lvl_p_rows(c, sigma, l), rlim = lvl_r_rows(c, sigma, l);
  const double* Pl = c.Y + (int64_t)l * c.ld;
  const double* Pm = Pl - c.ld;
  double* Pn = c.Y + (int64_t)(l + 1) * c.ld;
  const double* Rl = c.Y + (int64_t)(sigma + 1 + l) * c.ld;
  const double* Rm = Rl - c.ld;
  double* Rn = c.Y + (int64_t)(sigma + 2 + l) * c.ld;
  int bad = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < plim; i += stride) {
    const int beg = c.rp[i], end = c.rp[i + 1];
    const bool rr = DO_R && i < rlim;
    double acc[2];
    if (rr) {
      const double* xs[2] = {Pl, Rl};
      row_dot<2>(c.col, c.val, beg, end, xs, acc);
    } else {
      const double* xs[1] = {Pl};
      row_dot<1>(c.col, c.val, beg, end, xs, acc);
    }
    const double wp = recur(acc[0], Pl[i], use_mu ? Pm[i] : 0.0, th, ga, mu, use_mu);
    Pn[i] = wp;
    bad |= !finite(wp);
    if (rr) {
      const double wr = recur(acc[1], Rl[i], use_mu ? Rm[i] : 0.0, th, ga, mu, use_mu);
      Rn[i] = wr;
      bad |= !finite(wr);
    }
  }
  return bad;
}

__global__ void __launch_bounds__(ROWS_PER_CTA) k_level(Ctx c, int l) {
  const SolverState* st = c.st;
  if (st->done) return;
  const int sbar = st->s_bar;
  if (l >= sbar) return;
  const int sigma = c.cfg->sigma;
  const double th = st->prm.th[l], ga = st->prm.ga[l], mu = st->prm.mu[l - 1];
  const bool use_mu = !(mu == 0.0);  // basis.py:217 `if mu != 0.0` (NaN counts)
  int bad = (l < sbar - 1) ? level_rows<true>(c, l, sigma, th, ga, mu, use_mu)
                           : level_rows<false>(c, l, sigma, th, ga, mu, use_mu);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&c.st->breakdown, 1);
}

// Initial residual (adaptive.py:121-123): r = b - A x0 into Y[:, sigma+1], p = r into
// Y[:, 0], x = x0; partial ||b||^2 into part_t (for nb, adaptive.py:118).
__global__ void __launch_bounds__(ROWS_PER_CTA) k_init_residual(Ctx c, const double* x0) {
  __shared__ double sm[ROWS_PER_CTA / 32];
  const int sigma = c.cfg->sigma;
  double* P0 = c.Y;
  double* R0 = c.Y + (int64_t)(sigma + 1) * c.ld;
  double bb = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < c.lvl_rows[SMAX]; i += stride) {
    if (i >= c.n_own) {  // ghost rows: x from x0; p, r arrive with the first halo exchange
      c.x[i] = x0[i];
      continue;
    }
    double acc[1];
    const double* xs[1] = {x0};
    row_dot<1>(c.col, c.val, c.rp[i], c.rp[i + 1], xs, acc);
    const double bi = c.b[i];
    const double r = __dsub_rn(bi, acc[0]);
    R0[i] = r;
    P0[i] = r;
    c.x[i] = x0[i];
    bb = fma(bi, bi, bb);
  }
  bb = block_sum<ROWS_PER_CTA>(bb, sm);
  if (threadIdx.x == 0) c.part_t[blockIdx.x] = bb;
}

// Full-trace diagnostics (adaptive.py:205-215): tv = b - A x_j; partials of
// ||tv||^2, ||r_j||^2, ||tv - r_j||^2.  x_j / r_j were formed by k_diag_form.
__global__ void __launch_bounds__(ROWS_PER_CTA) k_diag_resid(Ctx c, int j) {
  __shared__ double sm[ROWS_PER_CTA / 32];
  if (j >= c.st->diag_n) return;
  double s_t = 0.0, s_r = 0.0, s_g = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < c.n_own; i += stride) {
    double acc[1];
    const double* xs[1] = {c.xj};
    row_dot<1>(c.col, c.val, c.rp[i], c.rp[i + 1], xs, acc);
    const double tv = __dsub_rn(c.b[i], acc[0]);
    const double r = c.rj[i];
    const double g = __dsub_rn(tv, r);
    s_t = fma(tv, tv, s_t);
    s_r = fma(r, r, s_r);
    s_g = fma(g, g, s_g);
  }
  s_t = block_sum<ROWS_PER_CTA>(s_t, sm);
  s_r = block_sum<ROWS_PER_CTA>(s_r, sm);
  s_g = block_sum<ROWS_PER_CTA>(s_g, sm);
  if (threadIdx.x == 0) {
    c.part_d[blockIdx.x] = s_t;
    c.part_d[RED_BLOCKS + blockIdx.x] = s_r;
    c.part_d[2 * RED_BLOCKS + blockIdx.x] = s_g;
  }
}

// ---- unit-entry kernels (explicit parameters, no solver state) ------------
__global__ void __launch_bounds__(ROWS_PER_CTA)
    k_spmv(const int* __restrict__ rp, const int* __restrict__ col,
           const double* __restrict__ val, int64_t n, const double* __restrict__ x, double* y) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    double acc[1];
    const double* xs[1] = {x};
    row_dot<1>(col, val, rp[i], rp[i + 1], xs, acc);
    y[i] = acc[0];
  }
}

// one level of a standalone block build (columns: P at 0..s, R at s+1..2s)
__global__ void __launch_bounds__(ROWS_PER_CTA)
    k_block_level(const int* __restrict__ rp, const int* __restrict__ col,
                  const double* __restrict__ val, int64_t n, int64_t ld, double* Y, int s, int l,
                  double th, double ga, double mu, int* breakdown) {
  const bool use_mu = (l >= 1) && !(mu == 0.0);
  const bool do_p = l < s, do_r = l < s - 1;
  const double* Pl = Y + (int64_t)l * ld;
  double* Pn = Y + (int64_t)(l + 1) * ld;
  const double* Rl = Y + (int64_t)(s + 1 + l) * ld;
  double* Rn = Y + (int64_t)(s + 2 + l) * ld;
  int bad = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int beg = rp[i], end = rp[i + 1];
    double acc[2];
    const double* xs[2] = {Pl, Rl};
    row_dot<2>(col, val, beg, end, xs, acc);
    if (do_p) {
      double w = recur(acc[0], Pl[i], use_mu ? Pl[i - ld] : 0.0, th, ga, mu, use_mu);
      Pn[i] = w;
      bad |= !finite(w);
    }
    if (do_r) {
      double w = recur(acc[1], Rl[i], use_mu ? Rl[i - ld] : 0.0, th, ga, mu, use_mu);
      Rn[i] = w;
      bad |= !finite(w);
    }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(breakdown, 1);
}

inline int grid_rows(int64_t n) {
  int64_t g = (n + ROWS_PER_CTA - 1) / ROWS_PER_CTA;
  if (g > RED_BLOCKS) g = RED_BLOCKS;
  if (g < 1) g = 1;
  return (int)g;
}

}  // namespace

// The row-streaming kernels always launch RED_BLOCKS CTAs (grid-stride) so the
// partial-sum arrays have a fixed length and the reductions a fixed order.
size_t staged_smem_bytes(int cap) { return MT_STAGES * stage_bytes(cap); }

// The attribute is per kernel and process-wide, and several plans (ranks of a
// virtual group, different matrices) may coexist: raise it once to the staging
// ceiling instead of to one plan's tile size.
void staged_prepare(int cap) {
  (void)cap;
  const int bytes = 200 * 1024;
  cudaFuncSetAttribute(k_level0_staged, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  cudaFuncSetAttribute(k_level_staged, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  cudaFuncSetAttribute(k_mpk_wave, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

int wave_ctas_per_sm(int cap) {
  int a = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, k_mpk_wave, WAVE_THREADS, MT_STAGES * wave_stage_bytes(cap));
  return a;
}

// co-residency of the whole grid is what makes the spin-waits safe: launch
// cooperatively (the runtime refuses a grid that cannot be co-resident)
#ifdef WAVE_DBG
extern "C" int sscg_debug_wave_counters(unsigned long long* out8) {
  cudaMemcpyFromSymbol(out8, g_wave_dbg, sizeof(unsigned long long) * 8);
  static const unsigned long long zero[8] = {};
  cudaMemcpyToSymbol(g_wave_dbg, zero, sizeof(zero));
  return (int)cudaGetLastError();
}
#endif

cudaError_t launch_wave(const Ctx& c, const WaveArgs& a, int grid, cudaStream_t s) {
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(grid);
  lc.blockDim = dim3(WAVE_THREADS);
  lc.dynamicSmemBytes = MT_STAGES * wave_stage_bytes(c.stage_cap);
  lc.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  return cudaLaunchKernelEx(&lc, k_mpk_wave, c, a);
}

int staged_ctas_per_sm(int cap) {
  int a = 0, b = 0;
  const size_t bytes = staged_smem_bytes(cap);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, k_level0_staged, MT_ROWS, bytes);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_level_staged, MT_ROWS, bytes);
  return a < b ? a : b;
}

// the side-branch residual of a split level 0 (capture_outer)
void launch_resid(const Ctx& c, int sigma, cudaStream_t s) {
  const size_t bytes = ss_smem_bytes_dev(c.pat_np) + (c.zm_base ? 4 * (size_t)c.zm_np : 0);
  const ZmPtrs zp = zm_ptrs(c, 0, sigma);
  if (c.pid_bytes == 1) {
    switch (c.ss_ne) {
      case 3: k_resid_zm<uint8_t, 3><<<c.red_n, ROWS_PER_CTA, bytes, s>>>(c, zp); break;
      case 5: k_resid_zm<uint8_t, 5><<<c.red_n, ROWS_PER_CTA, bytes, s>>>(c, zp); break;
      default: k_resid_zm<uint8_t, 7><<<c.red_n, ROWS_PER_CTA, bytes, s>>>(c, zp); break;
    }
  } else {
    switch (c.ss_ne) {
      case 3: k_resid_zm<uint16_t, 3><<<c.red_n, ROWS_PER_CTA, bytes, s>>>(c, zp); break;
      case 5: k_resid_zm<uint16_t, 5><<<c.red_n, ROWS_PER_CTA, bytes, s>>>(c, zp); break;
      default: k_resid_zm<uint16_t, 7><<<c.red_n, ROWS_PER_CTA, bytes, s>>>(c, zp); break;
    }
  }
}

void launch_init_residual(const Ctx& c, const double* x0, cudaStream_t s) {
  k_init_residual<<<c.red_n, ROWS_PER_CTA, 0, s>>>(c, x0);
}
size_t pattern_smem_bytes(int np, int ne) {
  return (size_t)ne * 12 + (size_t)(np + 1) * 4;
}

void pattern_prepare() {
  const int bytes = 48 * 1024;
  cudaFuncSetAttribute(k_level0_pat<uint8_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  cudaFuncSetAttribute(k_level0_pat<uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  cudaFuncSetAttribute(k_level_pat<uint8_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  cudaFuncSetAttribute(k_level_pat<uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

size_t ss_smem_bytes(int np) { return ss_smem_bytes_dev(np); }

int ss_ne_bucket(int ne) { return ne <= 3 ? 3 : ne <= 5 ? 5 : ne <= 7 ? 7 : 8; }

template <typename ID, int NE>
void ss_occ(size_t bytes, int* a, int* b) {
  const int lim = 48 * 1024;
  cudaFuncSetAttribute(k_level0_ss<ID, NE>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
  cudaFuncSetAttribute(k_level_ss<ID, NE>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(a, k_level0_ss<ID, NE>, ROWS_PER_CTA, bytes);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(b, k_level_ss<ID, NE>, ROWS_PER_CTA, bytes);
}

template <typename ID, int NE>
void zm_occ(size_t bytes, int* a, int* b) {
  const int lim = 48 * 1024;
  cudaFuncSetAttribute(k_level0_zm<ID, NE, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
  cudaFuncSetAttribute(k_level0_zm<ID, NE, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
  cudaFuncSetAttribute(k_resid_zm<ID, NE>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
  cudaFuncSetAttribute(k_level_zm<ID, NE>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(a, k_level0_zm<ID, NE, false>, ROWS_PER_CTA, bytes);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(b, k_level_zm<ID, NE>, ROWS_PER_CTA, bytes);
}

// plane-march kernels for a symmetric union of 3, 5 or 7 offsets
int zm_ctas_per_sm(int np, int ne, int pid_bytes, int* out2) {
  int a = 0, b = 0;
  const size_t bytes = ss_smem_bytes_dev(np);
  if (ne != 3 && ne != 5 && ne != 7) return 0;
  if (pid_bytes == 1) {
    if (ne == 3) zm_occ<uint8_t, 3>(bytes, &a, &b);
    else if (ne == 5) zm_occ<uint8_t, 5>(bytes, &a, &b);
    else zm_occ<uint8_t, 7>(bytes, &a, &b);
  } else {
    if (ne == 3) zm_occ<uint16_t, 3>(bytes, &a, &b);
    else if (ne == 5) zm_occ<uint16_t, 5>(bytes, &a, &b);
    else zm_occ<uint16_t, 7>(bytes, &a, &b);
  }
  out2[0] = a;
  out2[1] = b;
  return a < b ? a : b;
}

// row-pair march (levels >= 1) for 5- and 7-slot unions
int zp_ctas_per_sm(int np, int ne, int pid_bytes) {
  int b = 0;
  const size_t bytes = ss_smem_bytes_dev(np);
  const int lim = 48 * 1024;
#define ZP_OCC(ID, NE)                                                                       \
  cudaFuncSetAttribute(k_level_zp<ID, NE>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim); \
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_level_zp<ID, NE>, ROWS_PER_CTA, bytes);
  if (pid_bytes == 1) {
    if (ne == 5) { ZP_OCC(uint8_t, 5) } else if (ne == 7) { ZP_OCC(uint8_t, 7) }
  } else {
    if (ne == 5) { ZP_OCC(uint16_t, 5) } else if (ne == 7) { ZP_OCC(uint16_t, 7) }
  }
#undef ZP_OCC
  return b;
}

// value-stream kernels: CTAs per SM of level 0 and levels >= 1
int vs_ctas_per_sm(int ne, int* out2) {
  const int nb = ne <= 9 ? 9 : ne <= 18 ? 18 : ne <= 27 ? 27 : 32;
  int a = 0, b = 0;
#define VS_OCC(NE)                                                                   \
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, k_level0_vs<NE>, ROWS_PER_CTA, 0); \
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_level_vs<NE>, ROWS_PER_CTA, 0);
  if (nb == 9) { VS_OCC(9) } else if (nb == 18) { VS_OCC(18) } else if (nb == 27) { VS_OCC(27) } else { VS_OCC(32) }
#undef VS_OCC
  out2[0] = a;
  out2[1] = b;
  return a < b ? a : b;
}

int ss_ctas_per_sm(int np, int ne, int pid_bytes, int* out2) {
  int a = 0, b = 0;
  const size_t bytes = ss_smem_bytes_dev(np);
  const int nb = ss_ne_bucket(ne);
  if (pid_bytes == 1) {
    if (nb == 3) ss_occ<uint8_t, 3>(bytes, &a, &b);
    else if (nb == 5) ss_occ<uint8_t, 5>(bytes, &a, &b);
    else if (nb == 7) ss_occ<uint8_t, 7>(bytes, &a, &b);
    else ss_occ<uint8_t, 8>(bytes, &a, &b);
  } else {
    if (nb == 3) ss_occ<uint16_t, 3>(bytes, &a, &b);
    else if (nb == 5) ss_occ<uint16_t, 5>(bytes, &a, &b);
    else if (nb == 7) ss_occ<uint16_t, 7>(bytes, &a, &b);
    else ss_occ<uint16_t, 8>(bytes, &a, &b);
  }
  out2[0] = a;
  out2[1] = b;
  return a < b ? a : b;
}

// level 0 (the partial-sum kernel) and levels >= 1: out[0], out[1]
int pattern_ctas_per_sm(int np, int ne, int pid_bytes, int* out2) {
  int a = 0, b = 0;
  const size_t bytes = pattern_smem_bytes(np, ne);
  if (pid_bytes == 1) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, k_level0_pat<uint8_t>, ROWS_PER_CTA, bytes);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_level_pat<uint8_t>, ROWS_PER_CTA, bytes);
  } else {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, k_level0_pat<uint16_t>, ROWS_PER_CTA, bytes);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_level_pat<uint16_t>, ROWS_PER_CTA, bytes);
  }
  out2[0] = a;
  out2[1] = b;
  return a < b ? a : b;
}

size_t window_smem_bytes(int np, int ne, int r, int nvw, int pid_bytes) {
  return win_table_bytes(np, ne) + 2 * win_stage_bytes(r, nvw, pid_bytes);
}

int window_ctas_per_sm(int np, int ne, int r, int pid_bytes, int* out2) {
  const size_t b0 = window_smem_bytes(np, ne, r, 3, pid_bytes), b1 = window_smem_bytes(np, ne, r, 2, pid_bytes);
  const int lim = 200 * 1024;
  if (pid_bytes == 1) {
    cudaFuncSetAttribute(k_level0_win<uint8_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
    cudaFuncSetAttribute(k_level_win<uint8_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&out2[0], k_level0_win<uint8_t>, WT, b0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&out2[1], k_level_win<uint8_t>, WT, b1);
  } else {
    cudaFuncSetAttribute(k_level0_win<uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
    cudaFuncSetAttribute(k_level_win<uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&out2[0], k_level0_win<uint16_t>, WT, b0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&out2[1], k_level_win<uint16_t>, WT, b1);
  }
  return out2[0] < out2[1] ? out2[0] : out2[1];
}

void launch_level(const Ctx& c, int level, int sigma, cudaStream_t s, bool with_resid) {
  if (c.pid && c.win_r >= 0) {
    const int nvw = level == 0 ? 3 : 2;
    const size_t bytes = window_smem_bytes(c.pat_np, c.pat_ne, c.win_r, nvw, c.pid_bytes);
    if (c.pid_bytes == 1) {
      if (level == 0)
        k_level0_win<uint8_t><<<c.red_n, WT, bytes, s>>>(c);
      else
        k_level_win<uint8_t><<<c.win_grid, WT, bytes, s>>>(c, level);
    } else {
      if (level == 0)
        k_level0_win<uint16_t><<<c.red_n, WT, bytes, s>>>(c);
      else
        k_level_win<uint16_t><<<c.win_grid, WT, bytes, s>>>(c, level);
    }
    return;
  }
  if (c.vs_ne > 0) {
    const ZmPtrs zp = zm_ptrs(c, level, sigma);
    const int ne = c.vs_ne <= 9 ? 9 : c.vs_ne <= 18 ? 18 : c.vs_ne <= 27 ? 27 : 32;
#define VS_LAUNCH(NE)                                                        \
  if (level == 0)                                                            \
    k_level0_vs<NE><<<c.red_n, ROWS_PER_CTA, 0, s>>>(c, zp);                 \
  else                                                                       \
    k_level_vs<NE><<<c.pat_grid, ROWS_PER_CTA, 0, s>>>(c, level, zp);
    switch (ne) {
      case 9: VS_LAUNCH(9) break;
      case 18: VS_LAUNCH(18) break;
      case 27: VS_LAUNCH(27) break;
      default: VS_LAUNCH(32) break;
    }
#undef VS_LAUNCH
    return;
  }
  if (c.pid && c.ss_ne > 0 && c.zm_S > 0) {
    const size_t bytes = ss_smem_bytes_dev(c.pat_np) + (c.zm_base ? 4 * (size_t)c.zm_np : 0);
    const ZmPtrs zp = zm_ptrs(c, level, sigma);
#define ZM_LAUNCH(ID, NE)                                                      \
  if (level == 0 && c.zm_split) {                                             \
    if (with_resid) k_resid_zm<ID, NE><<<c.red_n, ROWS_PER_CTA, bytes, s>>>(c, zp); \
    k_level0_zm<ID, NE, true><<<c.red_n, ROWS_PER_CTA, bytes, s>>>(c, zp);     \
  } else if (level == 0)                                                       \
    k_level0_zm<ID, NE, false><<<c.red_n, ROWS_PER_CTA, bytes, s>>>(c, zp);    \
  else if (c.zt_on && NE == 7)                                                 \
    k_level_zt<ID><<<c.pat_grid, ROWS_PER_CTA, bytes, s>>>(c, level, zp);      \
  else if (c.zm_pair && NE >= 5)                                               \
    k_level_zp<ID, (NE >= 5 ? NE : 5)><<<c.zp_grid, ROWS_PER_CTA, bytes, s>>>(c, level, zp); \
  else                                                                         \
    k_level_zm<ID, NE><<<c.pat_grid, ROWS_PER_CTA, bytes, s>>>(c, level, zp);
#define ZM_NE_SWITCH(ID)                   \
  switch (c.ss_ne) {                       \
    case 3: ZM_LAUNCH(ID, 3) break;        \
    case 5: ZM_LAUNCH(ID, 5) break;        \
    default: ZM_LAUNCH(ID, 7) break;       \
  }
    if (c.pid_bytes == 1) {
      ZM_NE_SWITCH(uint8_t)
    } else {
      ZM_NE_SWITCH(uint16_t)
    }
    return;
  }
  if (c.pid && c.ss_ne > 0) {
    const size_t bytes = ss_smem_bytes_dev(c.pat_np);
    const int ne = ss_ne_bucket(c.ss_ne);
#define SS_LAUNCH(ID, NE)                                                      \
  if (level == 0)                                                              \
    k_level0_ss<ID, NE><<<c.red_n, ROWS_PER_CTA, bytes, s>>>(c);               \
  else                                                                         \
    k_level_ss<ID, NE><<<c.pat_grid, ROWS_PER_CTA, bytes, s>>>(c, level);
#define SS_NE_SWITCH(ID)                   \
  switch (ne) {                            \
    case 3: SS_LAUNCH(ID, 3) break;        \
    case 5: SS_LAUNCH(ID, 5) break;        \
    case 7: SS_LAUNCH(ID, 7) break;        \
    default: SS_LAUNCH(ID, 8) break;       \
  }
    if (c.pid_bytes == 1) {
      SS_NE_SWITCH(uint8_t)
    } else {
      SS_NE_SWITCH(uint16_t)
    }
    return;
  }
  if (c.pid) {
    const size_t bytes = pattern_smem_bytes(c.pat_np, c.pat_ne);
    if (c.pid_bytes == 1) {
      if (level == 0)
        k_level0_pat<uint8_t><<<c.red_n, ROWS_PER_CTA, bytes, s>>>(c);
      else
        k_level_pat<uint8_t><<<c.pat_grid, ROWS_PER_CTA, bytes, s>>>(c, level);
    } else {
      if (level == 0)
        k_level0_pat<uint16_t><<<c.red_n, ROWS_PER_CTA, bytes, s>>>(c);
      else
        k_level_pat<uint16_t><<<c.pat_grid, ROWS_PER_CTA, bytes, s>>>(c, level);
    }
    return;
  }
  if (c.stage_cap > 0) {
    const size_t bytes = staged_smem_bytes(c.stage_cap);
    if (level == 0)
      k_level0_staged<<<c.red_n, MT_ROWS, bytes, s>>>(c);
    else
      k_level_staged<<<c.red_n, MT_ROWS, bytes, s>>>(c, level);
    return;
  }
  if (level == 0)
    k_level0<<<c.red_n, ROWS_PER_CTA, 0, s>>>(c);
  else
    k_level<<<c.red_n, ROWS_PER_CTA, 0, s>>>(c, level);
}
void launch_spmv(const int* rp, const int* col, const double* val, int64_t n, const double* x,
                 double* y, cudaStream_t s) {
  k_spmv<<<grid_rows(n), ROWS_PER_CTA, 0, s>>>(rp, col, val, n, x, y);
}
void launch_block_levels(const int* rp, const int* col, const double* val, int64_t n, int64_t ld,
                         double* Y, int s, const double* th, const double* ga, const double* mu,
                         int* breakdown, cudaStream_t st) {
  for (int l = 0; l < s; ++l)
    k_block_level<<<grid_rows(n), ROWS_PER_CTA, 0, st>>>(rp, col, val, n, ld, Y, s, l, th[l], ga[l],
                                                          l >= 1 ? mu[l - 1] : 0.0, breakdown);
}
void launch_diag_resid(const Ctx& c, int j, cudaStream_t s) {
  k_diag_resid<<<c.red_n, ROWS_PER_CTA, 0, s>>>(c, j);
}
