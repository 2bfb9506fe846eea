// stage_pl.cuh — the P-part line kernel (fast mode, inviscid), included inside
// kernels_fast.cu's anonymous namespace (it uses Ops<>, vel, face_normal,
// es_flux_fast and the async-copy helpers defined there).
//
// One fused, persistent kernel per SSPRK3 stage: split-form volume flux
// differencing (dg_rhs.hpp:23-71) over symmetric node pairs, the precomputed
// split bathymetry source (dg_rhs.hpp:154-183), the entropy-stable interface
// flux (fluxes.hpp:136-166, re-evaluated bitwise on both sides of a face),
// -1/J (dg_rhs.hpp:289-292), the SSPRK3 combination (timeloop.hpp:114-127),
// the element mean, Zhang-Shu limiter and dry-node cut (limiter.hpp:24-84) and
// the reject signal (timeloop.hpp:205-209).
//
// Work decomposition.  A CTA owns a group of E consecutive elements.  Every
// xi-line and eta-line of the group is cut into P chunks of ~(N+1)/P nodes;
// the thread owning chunk K of a line ("part" K) keeps the chunk's nodal data
// and accumulators in registers.  The pair triangle of the line splits into P
// diagonal triangles (evaluated in registers by their owner) and P(P-1)/2
// off-diagonal blocks; a compile-time balancer splits each block (k,l) between
// its two owners, who stream the other chunk's nodes from shared memory, so
// every pair is evaluated exactly once and the work per part is even.  The
// streamed nodes' contributions go back through slot-major exchange slots,
// summed by the owner in a fixed order (reproducible).
//
// Against the half-line kernel this (a) sizes the register footprint with P
// (occupancy at high N), (b) streams partner nodes with runtime loops (compact
// code: the instruction cache was 18% of the stall samples at N=15), (c) stores
// u/2, v/2 once per node instead of re-dividing in every streamer, (d) uses an
// odd row stride for both line directions (conflict-free for odd N+1 too) and
// (e) folds Dtilde/8 into Dtilde/4 (one coefficient per pair side).
//
// Warps are part-uniform: the P parts run different compile-time code paths
// (no divergence), while the line direction is a per-lane runtime choice of
// stride and metric fields — the eta-line contribution is the negation of the
// formula evaluated with the raw (y_xi, x_xi) metrics, so it shares the code.
#pragma once

template <int V>
struct PLI {
  static constexpr int value = V;
};
// compile-time loop: f(PLI<I>{}) for I in [B, E)
template <int B, int E, class Fn>
__device__ __forceinline__ void pl_for(Fn&& f) {
  if constexpr (B < E) {
    f(PLI<B>{});
    pl_for<B + 1, E>(f);
  }
}

template <int N1_, int P_, int E_>
struct PLP {
  static constexpr int N1 = N1_, P = P_, E = E_, NP = N1 * N1;
  static constexpr int lo(int k) { return k * N1 / P; }
  static constexpr int rs(int k) { return lo(k + 1) - lo(k); }
  static constexpr int R = (N1 + P - 1) / P;        // register slots per thread
  static constexpr int LPD = E * N1, LPP = 2 * LPD;  // lines per direction / per part
  static constexpr int WR = (LPP + 31) / 32, LS = 32 * WR;  // warps per part, line slots
  static constexpr int THREADS = LS * P;
  static constexpr int PAD = (N1 & 1) ? N1 : N1 + 1;  // odd row stride
  static constexpr int EPAD = N1 * PAD;
  static constexpr int GPAD = E * EPAD;
  static constexpr int GNP = E * NP;
  enum { F_H, F_HU, F_HV, F_YE, F_XE, F_YX, F_XX, F_U2, F_V2, kLine };
  enum { N_JAC, N_SX, N_SY, N_WH, N_WHU, N_WHV, kNode };
  static constexpr int kSurf = 14;  // one face flux ~ 7 pairs (half-pair units)

  // Block split.  Block (k,l), k < l: part k streams nodes lo(l)..lo(l)+c-1 of
  // chunk l (pairing each with all its own nodes); part l streams all of chunk
  // k, pairing with its own nodes c..rs(l)-1.  Exchange slots: sa[k][l] + t for
  // part k's streamed node t, sb[k][l] + s for part l's streamed node s.
  struct Split {
    int c[P][P], sa[P][P], sb[P][P], ns, w[P];
  };
  static constexpr Split split() {
    Split s{};
    int W[P] = {};
    for (int k = 0; k < P; ++k) {
      W[k] = rs(k) * (rs(k) - 1);
      if (k == 0) W[k] += 2 + kSurf;
      if (k == P - 1) W[k] += 2 + kSurf;
    }
    // greedy by block distance, then coordinate-descent passes
    for (int pass = 0; pass < 6; ++pass)
      for (int d = 1; d < P; ++d)
        for (int k = 0; k + d < P; ++k) {
          const int l = k + d, a = rs(k), b = rs(l);
          if (pass > 0) {  // take the block's current share back out
            const int c0 = s.c[k][l];
            W[k] -= 2 * a * c0 + c0;
            W[l] -= 2 * a * (b - c0) + (c0 < b ? a : 0);
          }
          int best = 0, bw = 1 << 30;
          for (int c = 0; c <= b; ++c) {
            const int wk = W[k] + 2 * a * c + c;
            const int wl = W[l] + 2 * a * (b - c) + (c < b ? a : 0);
            const int m = wk > wl ? wk : wl;
            if (m < bw) {
              bw = m;
              best = c;
            }
          }
          s.c[k][l] = best;
          W[k] += 2 * a * best + best;
          W[l] += 2 * a * (b - best) + (best < b ? a : 0);
        }
    int ns = 0;
    for (int d = 1; d < P; ++d)
      for (int k = 0; k + d < P; ++k) {
        const int l = k + d;
        s.sa[k][l] = ns;
        ns += s.c[k][l];
        s.sb[k][l] = ns;
        if (s.c[k][l] < rs(l)) ns += rs(k);
      }
    s.ns = ns;
    for (int k = 0; k < P; ++k) s.w[k] = W[k];
    return s;
  }
  static constexpr Split SP = split();
  static constexpr int XS = SP.ns > 0 ? SP.ns : 1;  // exchange slots per line
  // ---- shared-memory plan (doubles) ----
  static constexpr int LINE = 0;                            // [kLine][E][N1][PAD]
  static constexpr int ACC = LINE + kLine * GPAD;           // eta lines: [3][E][N1][PAD]
  static constexpr int XCH = ACC + 3 * GPAD;                // [3*XS][LS]
  static constexpr int GNPA = (GNP + 3) & ~1;               // node field stride (+1 shift slack)
  static constexpr int NODE = (XCH + 3 * XS * LS + 1) & ~1;  // [kNode][GNPA], bulk copies
  static constexpr int TR = NODE + kNode * GNPA;            // [7][E][4][N1] traces
  static constexpr int EFO = (TR + 7 * E * 4 * N1 + 1) & ~1;  // int4 [E][4]
  static constexpr int RED = EFO + E * 4 * 2;               // [P][LPD][5] xi-thread partials
  static constexpr int ELM = RED + P * LPD * 5;             // [E][4]: avg0..2, theta
  static constexpr int BAR = (ELM + E * 4 + 1) & ~1;
  static constexpr int TOTAL = BAR + 2;
  static constexpr size_t bytes = TOTAL * sizeof(double);
};

// Symmetric two-point contravariant flux of a node pair, scaled (4F0, 4F1, 4F2)
// so Dtilde/4 weighs all three: a is the register-owned side (gha = g h_a),
// u2/v2 are half velocities.  19 DP instructions per pair with both scatters.
__device__ __forceinline__ void pl_pair(double gha, double hua, double hva, double ua2,
                                        double va2, double Aa, double Ba, double hb, double hub,
                                        double hvb, double ub2, double vb2, double Ab, double Bb,
                                        double& F0, double& T1, double& T2) {
  const double Shu = hua + hub, Shv = hva + hvb, Su = ua2 + ub2, Sv = va2 + vb2;
  const double SA = Aa + Ab, SB = Ba + Bb;
  F0 = SA * Shu - SB * Shv;
  const double Q = gha * hb;  // g h_a h_b = 2 * pressure (fluxes.hpp:33)
  T1 = Su * F0 + Q * SA;
  T2 = Sv * F0 - Q * SB;
}

template <int N1>
__device__ __forceinline__ double pl_d4(int a, int b) {  // Dtilde(a,b) / 4
  return c_ops[Ops<N1>::base + N1 * N1 + a * N1 + b];
}

// The register-resident chunk of one line.
template <int R>
struct PLRegs {
  double h[R], hu[R], hv[R], u2[R], v2[R], A[R], B[R], gh[R], r0[R], r1[R], r2[R];
};

// volume work of part K: own chunk -> registers, diagonal triangle, streamed blocks
template <class PL, int K>
__device__ __forceinline__ void pl_volume(PLRegs<PL::R>& X, const double* __restrict__ Lb,
                                          int off0, int st, int fa, int fb, double g,
                                          double* xch) {
  constexpr int N1 = PL::N1, P = PL::P, R = PL::R, GP = PL::GPAD, LS = PL::LS;
  constexpr int L0 = PL::lo(K), RK = PL::rs(K);
#pragma unroll
  for (int s = 0; s < R; ++s) {
    X.r0[s] = X.r1[s] = X.r2[s] = 0.0;
    if (s < RK) {
      const int q = off0 + (L0 + s) * st;
      X.h[s] = Lb[PL::F_H * GP + q];
      X.hu[s] = Lb[PL::F_HU * GP + q];
      X.hv[s] = Lb[PL::F_HV * GP + q];
      X.u2[s] = Lb[PL::F_U2 * GP + q];
      X.v2[s] = Lb[PL::F_V2 * GP + q];
      X.A[s] = Lb[fa + q];
      X.B[s] = Lb[fb + q];
      X.gh[s] = g * X.h[s];
    } else {
      X.h[s] = X.hu[s] = X.hv[s] = X.u2[s] = X.v2[s] = X.A[s] = X.B[s] = X.gh[s] = 0.0;
    }
  }
  // diagonal triangle (+ the corner self pair: Dtilde(i,i) != 0 only at i = 0, N)
#pragma unroll
  for (int s = 0; s < RK; ++s)
#pragma unroll
    for (int s2 = s; s2 < RK; ++s2) {
      const int a = L0 + s, b = L0 + s2;
      if (s == s2 && a != 0 && a != N1 - 1) continue;
      double F0, T1, T2;
      pl_pair(X.gh[s], X.hu[s], X.hv[s], X.u2[s], X.v2[s], X.A[s], X.B[s], X.h[s2], X.hu[s2],
              X.hv[s2], X.u2[s2], X.v2[s2], X.A[s2], X.B[s2], F0, T1, T2);
      const double dab = Ops<N1>::D4(a, b);
      X.r0[s] += dab * F0;
      X.r1[s] += dab * T1;
      X.r2[s] += dab * T2;
      if (s != s2) {
        const double dba = Ops<N1>::D4(b, a);
        X.r0[s2] += dba * F0;
        X.r1[s2] += dba * T1;
        X.r2[s2] += dba * T2;
      }
    }
  // blocks (K, l), l > K: stream the first c nodes of chunk l
  pl_for<K + 1, P>([&](auto LI) {
    constexpr int l = decltype(LI)::value;
    constexpr int c = PL::SP.c[K][l], L1 = PL::lo(l), slot = PL::SP.sa[K][l];
#pragma unroll 1
    for (int t = 0; t < c; ++t) {
      const int b = L1 + t, q = off0 + b * st;
      const double hb = Lb[PL::F_H * GP + q], hub = Lb[PL::F_HU * GP + q],
                   hvb = Lb[PL::F_HV * GP + q], ub2 = Lb[PL::F_U2 * GP + q],
                   vb2 = Lb[PL::F_V2 * GP + q], Ab = Lb[fa + q], Bb = Lb[fb + q];
      double c0 = 0.0, c1 = 0.0, c2 = 0.0;
#pragma unroll
      for (int s = 0; s < RK; ++s) {
        double F0, T1, T2;
        pl_pair(X.gh[s], X.hu[s], X.hv[s], X.u2[s], X.v2[s], X.A[s], X.B[s], hb, hub, hvb, ub2,
                vb2, Ab, Bb, F0, T1, T2);
        const double dab = pl_d4<N1>(L0 + s, b), dba = pl_d4<N1>(b, L0 + s);
        X.r0[s] += dab * F0;
        X.r1[s] += dab * T1;
        X.r2[s] += dab * T2;
        c0 += dba * F0;
        c1 += dba * T1;
        c2 += dba * T2;
      }
      double* x = xch + 3 * (slot + t) * LS;
      x[0] = c0;
      x[LS] = c1;
      x[2 * LS] = c2;
    }
  });
  // blocks (l, K), l < K: stream all of chunk l against own nodes c..RK-1
  pl_for<0, K>([&](auto LI) {
    constexpr int l = decltype(LI)::value;
    constexpr int c = PL::SP.c[l][K], L1 = PL::lo(l), n = PL::rs(l), slot = PL::SP.sb[l][K];
    if constexpr (c < RK) {
#pragma unroll 1
      for (int t = 0; t < n; ++t) {
        const int a = L1 + t, q = off0 + a * st;
        const double ha = Lb[PL::F_H * GP + q], hua = Lb[PL::F_HU * GP + q],
                     hva = Lb[PL::F_HV * GP + q], ua2 = Lb[PL::F_U2 * GP + q],
                     va2 = Lb[PL::F_V2 * GP + q], Aa = Lb[fa + q], Ba = Lb[fb + q];
        double c0 = 0.0, c1 = 0.0, c2 = 0.0;
#pragma unroll
        for (int s = c; s < RK; ++s) {
          double F0, T1, T2;
          pl_pair(X.gh[s], X.hu[s], X.hv[s], X.u2[s], X.v2[s], X.A[s], X.B[s], ha, hua, hva,
                  ua2, va2, Aa, Ba, F0, T1, T2);
          const double dba = pl_d4<N1>(L0 + s, a), dab = pl_d4<N1>(a, L0 + s);
          X.r0[s] += dba * F0;
          X.r1[s] += dba * T1;
          X.r2[s] += dba * T2;
          c0 += dab * F0;
          c1 += dab * T1;
          c2 += dab * T2;
        }
        double* x = xch + 3 * (slot + t) * LS;
        x[0] = c0;
        x[LS] = c1;
        x[2 * LS] = c2;
      }
    }
  });
}

// after the exchange barrier: add the contributions other parts computed for
// this part's nodes, in a fixed order
template <class PL, int K>
__device__ __forceinline__ void pl_receive(PLRegs<PL::R>& X, const double* xch) {
  constexpr int P = PL::P, LS = PL::LS, RK = PL::rs(K);
#pragma unroll
  for (int s = 0; s < RK; ++s) {
    pl_for<K + 1, P>([&](auto LI) {
      constexpr int l = decltype(LI)::value;
      constexpr int sbl = PL::SP.sb[K][l];
      if constexpr (PL::SP.c[K][l] < PL::rs(l)) {
        const double* x = xch + 3 * (sbl + s) * LS;
        X.r0[s] += x[0];
        X.r1[s] += x[LS];
        X.r2[s] += x[2 * LS];
      }
    });
    pl_for<0, K>([&](auto KI) {
      constexpr int k = decltype(KI)::value;
      constexpr int ck = PL::SP.c[k][K], sak = PL::SP.sa[k][K];
      if (s < ck) {
        const double* x = xch + 3 * (sak + s) * LS;
        X.r0[s] += x[0];
        X.r1[s] += x[LS];
        X.r2[s] += x[2 * LS];
      }
    });
  }
}

// line data of one group -> padded shared layout (8-byte cp.async per value),
// plus the group's element-face connectivity
template <class PL>
__device__ __forceinline__ void pl_prefetch_line(double* sm, const Mesh& M, const CState& in,
                                                 int g, int tid) {
  constexpr int N1 = PL::N1, NP = PL::NP, GP = PL::GPAD;
  const int e0 = M.e_lo + g * PL::E, ne = min(PL::E, M.n_owned - e0);
  const long long base = (long long)e0 * NP;
  const int cnt = ne * NP;
  for (int r = tid; r < cnt; r += PL::THREADS) {
    const int el = r / NP, q = r - el * NP;
    const int i = q / N1, j = q - i * N1;
    double* d = sm + PL::LINE + el * PL::EPAD + i * PL::PAD + j;
    const long long s = base + r;
    cp_async8(d + PL::F_H * GP, in.h + s);
    cp_async8(d + PL::F_HU * GP, in.hu + s);
    cp_async8(d + PL::F_HV * GP, in.hv + s);
    cp_async8(d + PL::F_YE * GP, M.ye + s);
    cp_async8(d + PL::F_XE * GP, M.xe + s);
    cp_async8(d + PL::F_YX * GP, M.yx + s);
    cp_async8(d + PL::F_XX * GP, M.xx + s);
  }
  const int4* ef = M.ef + (long long)e0 * 4;
  int4* dst = reinterpret_cast<int4*>(sm + PL::EFO);
  for (int k = tid; k < ne * 4; k += PL::THREADS)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst + k)),
                 "l"(ef + k)
                 : "memory");
}

// one thread: bulk-prefetch a group's node-range of `n` arrays into L2 (TMA,
// no shared memory): the later per-thread loads hit L2
__device__ __forceinline__ void l2_prefetch(const double* p, long long first, long long count) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p + first) & ~uintptr_t(15);
  const uintptr_t b = (reinterpret_cast<uintptr_t>(p + first + count) + 15) & ~uintptr_t(15);
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"((uint32_t)(b - a))
               : "memory");
}

// thread 0: node-phase fields of one group -> shared memory (TMA bulk copies).
// Bulk copies need 16-byte aligned sources: an odd first node is copied from
// one double earlier and the group's data starts at offset `shift`.
template <class PL>
__device__ __forceinline__ int pl_issue_node(double* sm, const Mesh& M, const StageArgs& A, int g,
                                             uint64_t* bar) {
  const int e0 = M.e_lo + g * PL::E, ne = min(PL::E, M.n_owned - e0);
  const long long off = (long long)e0 * PL::NP;
  const int shift = (int)(off & 1);
  const uint32_t fb = round16((size_t)(ne * PL::NP + shift) * sizeof(double));
  const bool wn = A.update && A.stage > 0;
  mbar_expect_tx(bar, (wn ? 6 : 3) * fb);
  double* nd = sm + PL::NODE;
  const long long o = off - shift;
  bulk_g2s(nd + PL::N_JAC * PL::GNPA, M.jac + o, fb, bar);
  bulk_g2s(nd + PL::N_SX * PL::GNPA, M.sx + o, fb, bar);
  bulk_g2s(nd + PL::N_SY * PL::GNPA, M.sy + o, fb, bar);
  if (wn) {
    bulk_g2s(nd + PL::N_WH * PL::GNPA, A.wn.h + o, fb, bar);
    bulk_g2s(nd + PL::N_WHU * PL::GNPA, A.wn.hu + o, fb, bar);
    bulk_g2s(nd + PL::N_WHV * PL::GNPA, A.wn.hv + o, fb, bar);
  }
  return shift;
}

template <class PL>
__device__ __forceinline__ void pl_prefetch_l2(const Mesh& M, const StageArgs& A, int g,
                                               bool line_fields) {
  const int e0 = M.e_lo + g * PL::E, ne = min(PL::E, M.n_owned - e0);
  const long long off = (long long)e0 * PL::NP, cnt = (long long)ne * PL::NP;
  if (line_fields) {
    const double* f[7] = {A.in.h, A.in.hu, A.in.hv, M.ye, M.xe, M.yx, M.xx};
#pragma unroll
    for (int k = 0; k < 7; ++k) l2_prefetch(f[k], off, cnt);
  } else {
    l2_prefetch(M.jac, off, cnt);
    l2_prefetch(M.sx, off, cnt);
    l2_prefetch(M.sy, off, cnt);
    if (A.update && A.stage > 0) {
      l2_prefetch(A.wn.h, off, cnt);
      l2_prefetch(A.wn.hu, off, cnt);
      l2_prefetch(A.wn.hv, off, cnt);
    }
  }
}

// interface flux at one own endpoint (dg_rhs.hpp:202-252): both sides evaluate
// the minus side's flux bitwise
__device__ __forceinline__ void pl_surface(int efy, int face, const double* tr, int TRS,
                                           double hs, double hus, double hvs, double om0,
                                           double om1, double g, double inv2g, double h_des,
                                           double iw0, double& r0, double& r1, double& r2) {
  const double bo = tr[6 * TRS];
  double wm0, wm1, wm2, wp0, wp1, wp2, bm, bp, nx, ny, js, sgn = 1.0;
  if (efy & EF_MINUS) {
    face_normal(face, om0, om1, nx, ny, js);
    wm0 = hs;
    wm1 = hus;
    wm2 = hvs;
    bm = bo;
    if (efy & EF_WALL) {  // exterior_state (mesh.hpp:382-386)
      const double mn = wm1 * nx + wm2 * ny;
      wp0 = wm0;
      wp1 = wm1 - 2.0 * mn * nx;
      wp2 = wm2 - 2.0 * mn * ny;
      bp = bm;
    } else {
      wp0 = tr[0];
      wp1 = tr[TRS];
      wp2 = tr[2 * TRS];
      bp = tr[3 * TRS];
    }
  } else {
    face_normal(efy & EF_NBR_FACE_MASK, tr[4 * TRS], tr[5 * TRS], nx, ny, js);
    wm0 = tr[0];
    wm1 = tr[TRS];
    wm2 = tr[2 * TRS];
    bm = tr[3 * TRS];
    wp0 = hs;
    wp1 = hus;
    wp2 = hvs;
    bp = bo;
    sgn = -1.0;
  }
  double f0, f1, f2;
  es_flux_fast(wm0, wm1, wm2, wp0, wp1, wp2, bm, bp, nx, ny, g, inv2g, h_des, f0, f1, f2);
  const double c = sgn * js * iw0;
  r0 += c * f0;
  r1 += c * f1;
  r2 += c * f2;
}

// part K after the exchange barrier: the contributions other parts computed
// for this part's nodes
template <class PL, int K>
__device__ __forceinline__ void pl_post_a(PLRegs<PL::R>& X, const double* sm, bool xi,
                                          int line) {
  pl_receive<PL, K>(X, sm + PL::XCH + line);
  if (!xi) {  // eta lines: the raw-metric formula is the negated contribution
#pragma unroll
    for (int s = 0; s < PL::R; ++s) {
      X.r0[s] = -X.r0[s];
      X.r1[s] = -X.r1[s];
      X.r2[s] = -X.r2[s];
    }
  }
}

// the interface flux at the own endpoints (parts 0 and P-1), then the eta
// lines hand their accumulators to the xi-line owners of the nodes
template <class PL, int K>
__device__ __forceinline__ void pl_post_b(PLRegs<PL::R>& X, double* sm, bool xi, int el, int li,
                                          const int (&efy)[2], double g, double inv2g,
                                          double h_des, double iw0) {
  constexpr int N1 = PL::N1, P = PL::P, GP = PL::GPAD, EP = PL::EPAD;
  constexpr int TRS = PL::E * 4 * N1;
  const int off0 = xi ? li : li * PL::PAD, st = xi ? PL::PAD : 1;
  // own face metrics: raw (y_eta, x_eta) on xi-lines, (y_xi, x_xi) on eta-lines
  if constexpr (K == 0) {
    if (efy[0] & EF_PRESENT) {
      const int face = xi ? 3 : 0;
      pl_surface(efy[0], face, sm + PL::TR + (el * 4 + face) * N1 + li, TRS, X.h[0], X.hu[0],
                 X.hv[0], X.A[0], X.B[0], g, inv2g, h_des, iw0, X.r0[0], X.r1[0], X.r2[0]);
    }
  }
  if constexpr (K == P - 1) {
    constexpr int SE = PL::rs(P - 1) - 1;
    if (efy[1] & EF_PRESENT) {
      const int face = xi ? 1 : 2;
      pl_surface(efy[1], face, sm + PL::TR + (el * 4 + face) * N1 + li, TRS, X.h[SE], X.hu[SE],
                 X.hv[SE], X.A[SE], X.B[SE], g, inv2g, h_des, iw0, X.r0[SE], X.r1[SE],
                 X.r2[SE]);
    }
  }
  if (!xi) {
    double* acc = sm + PL::ACC + el * EP;
#pragma unroll
    for (int s = 0; s < PL::rs(K); ++s) {
      const int q = off0 + (PL::lo(K) + s) * st;
      acc[0 * GP + q] = X.r0[s];
      acc[1 * GP + q] = X.r1[s];
      acc[2 * GP + q] = X.r2[s];
    }
  }
}

template <int N1, int P, int E, int MINB, bool FORCE>
__global__ void __launch_bounds__(PLP<N1, P, E>::THREADS, MINB)
    k_stage_pl(Mesh M, Phys Ph, StageArgs A, Flags* F) {
  using PL = PLP<N1, P, E>;
  using O = Ops<N1>;
  constexpr int NP = PL::NP, R = PL::R, GP = PL::GPAD, EP = PL::EPAD, LPD = PL::LPD;
  constexpr int TRS = E * 4 * N1;
  extern __shared__ __align__(16) double sm[];
  uint64_t* bar_node = reinterpret_cast<uint64_t*>(sm + PL::BAR);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int part = warp / PL::WR;                  // warp-uniform
  const int line = (warp % PL::WR) * 32 + lane;    // line slot within the part
  const bool line_ok = line < PL::LPP;
  const bool xi = line < LPD;
  const int ld = xi ? line : line - LPD;
  const int el = line_ok ? ld / N1 : 0, li = line_ok ? ld - (ld / N1) * N1 : 0;
  const int ngroups = (M.n_owned - M.e_lo + E - 1) / E;
  const double g = Ph.g, h_des = Ph.h_des, inv2g = 1.0 / (2.0 * g), iw0 = 1.0 / M.w0;

  if (tid == 0) {
    mbar_init(bar_node, 1);
    fence_mbar_init();
  }
  if ((int)blockIdx.x >= ngroups) return;
  pl_prefetch_line<PL>(sm, M, A.in, blockIdx.x, tid);
  cp_async_commit();
  uint32_t ph_node = 0;

  for (int grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
    const int e0 = M.e_lo + grp * E, ne = min(E, M.n_owned - e0);
    const bool active = line_ok && el < ne;
    const int e = e0 + el;
    cp_async_wait_all();
    __syncthreads();  // line(g) + connectivity(g) resident
    if (tid == 0) {  // node-phase data of g -> smem; line data of g+1 -> L2
      fence_proxy_async();
      pl_issue_node<PL>(sm, M, A, grp, bar_node);
#ifdef PL_L2_PREFETCH
      if (grp + (int)gridDim.x < ngroups) pl_prefetch_l2<PL>(M, A, grp + gridDim.x, true);
#endif
    }
    const int nshift = (int)(((long long)e0 * NP) & 1);
    // half velocities once per node (physics.hpp:23-36)
    for (int r = tid; r < ne * NP; r += PL::THREADS) {
      const int e2 = r / NP, q = r - e2 * NP, i = q / N1, j = q - i * N1;
      double* d = sm + PL::LINE + e2 * EP + i * PL::PAD + j;
      double u, v;
      vel(d[PL::F_H * GP], d[PL::F_HU * GP], d[PL::F_HV * GP], h_des, u, v);
      d[PL::F_U2 * GP] = 0.5 * u;
      d[PL::F_V2 * GP] = 0.5 * v;
    }
    // neighbour traces + own b for this line's endpoints (parts 0 and P-1)
    int efy[2] = {0, 0};
    if (active && (part == 0 || part == P - 1)) {
#pragma unroll
      for (int end = 0; end < 2; ++end) {
        if ((end == 0 && part != 0) || (end == 1 && part != P - 1)) continue;
        const int face = xi ? (end ? 1 : 3) : (end ? 2 : 0);
        const int4 ef = reinterpret_cast<const int4*>(sm + PL::EFO)[el * 4 + face];
        efy[end] = ef.y;
        double* tr = sm + PL::TR + (el * 4 + face) * N1 + li;
        cp_async8(tr + 6 * TRS, M.b + (long long)e * NP + face_node(N1, face, li));
        if ((ef.y & EF_PRESENT) && !(ef.y & EF_WALL)) {
          const int nf = ef.y & EF_NBR_FACE_MASK;
          const int tp = (ef.y & EF_REVERSED) ? N1 - 1 - li : li;
          const long long nb = (long long)ef.x * NP + face_node(N1, nf, tp);
          cp_async8(tr + 0 * TRS, A.in.h + nb);
          cp_async8(tr + 1 * TRS, A.in.hu + nb);
          cp_async8(tr + 2 * TRS, A.in.hv + nb);
          cp_async8(tr + 3 * TRS, M.b + nb);
          if (!(ef.y & EF_MINUS)) {
            const bool ew = nf == 1 || nf == 3;
            cp_async8(tr + 4 * TRS, (ew ? M.ye : M.yx) + nb);
            cp_async8(tr + 5 * TRS, (ew ? M.xe : M.xx) + nb);
          }
        }
      }
    }
    cp_async_commit();
    __syncthreads();  // half velocities visible

    PLRegs<R> X;
    if (active) {
      const int off0 = xi ? li : li * PL::PAD, st = xi ? PL::PAD : 1;
      const int fa = (xi ? PL::F_YE : PL::F_YX) * GP, fb = (xi ? PL::F_XE : PL::F_XX) * GP;
      const double* Lb = sm + PL::LINE + el * EP;
      double* xch = sm + PL::XCH + line;
      pl_for<0, P>([&](auto KI) {
        constexpr int k = decltype(KI)::value;
        if (part == k) pl_volume<PL, k>(X, Lb, off0, st, fa, fb, g, xch);
      });
    }
    __syncthreads();  // exchange slots published; the line buffer is free
    {
      const int gn = grp + gridDim.x;
      if (gn < ngroups) pl_prefetch_line<PL>(sm, M, A.in, gn, tid);
      cp_async_commit();
    }
    if (active) {
      pl_for<0, P>([&](auto KI) {
        constexpr int k = decltype(KI)::value;
        if (part == k) pl_post_a<PL, k>(X, sm, xi, line);
      });
    }
    asm volatile("cp.async.wait_group 1;" ::: "memory");  // traces(g); line(g+1) may fly
    if (active) {
      pl_for<0, P>([&](auto KI) {
        constexpr int k = decltype(KI)::value;
        if (part == k) pl_post_b<PL, k>(X, sm, xi, el, li, efy, g, inv2g, h_des, iw0);
      });
    }
    __syncthreads();  // eta accumulators in shared memory
    mbar_wait(bar_node, ph_node);
    ph_node ^= 1;

    // ---- node phase on the xi-line threads: nodes (k, li), k in the own chunk
    const int k0 = P == 1 ? 0 : (part * N1) / P;
    const int nk = ((part + 1) * N1) / P - k0;
    double* red = sm + PL::RED + (part * LPD + ld) * 5;
    if (xi && active) {
      const double* acc = sm + PL::ACC + el * EP;
      const double* Nd = sm + PL::NODE + nshift + el * NP;
      double s_area = 0.0, s0 = 0.0, s1 = 0.0, s2 = 0.0, mmin = 1.0e300;
      const double wj = O::w(li);
#pragma unroll
      for (int s = 0; s < R; ++s) {
        if (s >= nk) continue;
        const int k = k0 + s, q = k * N1 + li, qp = k * PL::PAD + li;
        const long long n = (long long)e * NP + q;
        const double jac = Nd[PL::N_JAC * PL::GNPA + q];
        const double ij = -1.0 / jac, hg2 = 0.5 * g * X.h[s];
        double rh = (acc[0 * GP + qp] + X.r0[s]) * ij;
        double rhu = (acc[1 * GP + qp] + X.r1[s] + hg2 * Nd[PL::N_SX * PL::GNPA + q]) * ij;
        double rhv = (acc[2 * GP + qp] + X.r2[s] + hg2 * Nd[PL::N_SY * PL::GNPA + q]) * ij;
        if (FORCE) {
          rh += A.fh[n];
          rhu += A.fhu[n];
          rhv += A.fhv[n];
        }
        if (A.rhs.h) {
          A.rhs.h[n] = rh;
          A.rhs.hu[n] = rhu;
          A.rhs.hv[n] = rhv;
        }
        double sh = X.h[s] + A.dt * rh;
        double shu = X.hu[s] + A.dt * rhu;
        double shv = X.hv[s] + A.dt * rhv;
        if (A.stage > 0 && A.update) {
          sh = A.ca * Nd[PL::N_WH * PL::GNPA + q] + A.cb * sh;
          shu = A.ca * Nd[PL::N_WHU * PL::GNPA + q] + A.cb * shu;
          shv = A.ca * Nd[PL::N_WHV * PL::GNPA + q] + A.cb * shv;
        }
        X.h[s] = sh;
        X.hu[s] = shu;
        X.hv[s] = shv;
        const double wq = O::w(k) * wj * jac;
        s_area += wq;
        s0 += wq * sh;
        s1 += wq * shu;
        s2 += wq * shv;
        mmin = smin(mmin, sh);
      }
      red[0] = s_area;
      red[1] = s0;
      red[2] = s1;
      red[3] = s2;
      red[4] = mmin;
    }
    __syncthreads();

    // ---- element means: one warp per element, fixed-shape reduction
    if (A.update) {
      constexpr int NW = PL::THREADS / 32, CNT = P * N1;
      for (int el2 = warp; el2 < ne; el2 += NW) {
        double a[5] = {0.0, 0.0, 0.0, 0.0, 1.0e300};
        for (int c = lane; c < CNT; c += 32) {
          const int pp = c / N1, l2 = c - pp * N1;
          const double* rr = sm + PL::RED + (pp * LPD + el2 * N1 + l2) * 5;
          a[0] += rr[0];
          a[1] += rr[1];
          a[2] += rr[2];
          a[3] += rr[3];
          a[4] = smin(a[4], rr[4]);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
          for (int c = 0; c < 4; ++c) a[c] += __shfl_xor_sync(0xffffffffu, a[c], o);
          a[4] = smin(a[4], __shfl_xor_sync(0xffffffffu, a[4], o));
        }
        if (lane == 0) {
          const double inv = 1.0 / a[0];
          const double avg0 = inv * a[1], avg1 = inv * a[2], avg2 = inv * a[3];
          const double mmin = a[4];
          double theta = 1.0;
          bool ok = true;
          if (avg0 < 0.0) {  // reject (timeloop.hpp:205-209)
            atomicExch(&F->reject, 1);
            if (!Ph.limiter) atomicExch(&F->abort, 1);
            ok = false;
          }
          if (ok && Ph.limiter && mmin < 0.0) {
            const double denom = avg0 - mmin;
            theta = denom < 1e-14 ? 1.0 : smin(1.0, avg0 / denom);
          }
          if (ok && !Ph.limiter && mmin < 0.0) atomicExch(&F->abort, 1);
          if (ok) {
            // the limited heights are a monotone map of the unlimited ones: the
            // element's minimum after limiting is the map of its minimum
            const double mlim = theta < 1.0 ? smax(theta * (mmin - avg0) + avg0, 0.0) : mmin;
            atomicMin(&F->min_h_key, order_key(mlim));
            if (theta < 1.0) atomicAdd(&F->n_limited, 1);
          }
          double* em = sm + PL::ELM + el2 * 4;
          em[0] = avg0;
          em[1] = avg1;
          em[2] = avg2;
          em[3] = ok ? theta : -1.0;  // -1: rejected element, nothing written
        }
      }
    }
    __syncthreads();

    // ---- limiter (limit_element, limiter.hpp:43-84) and write-out
    if (xi && active && A.update) {
      const double* em = sm + PL::ELM + el * 4;
      const double avg0 = em[0], avg1 = em[1], avg2 = em[2], theta = em[3];
      if (theta >= 0.0) {
#pragma unroll
        for (int s = 0; s < R; ++s) {
          if (s >= nk) continue;
          const long long n = (long long)e * NP + (k0 + s) * N1 + li;
          double sh = X.h[s], shu = X.hu[s], shv = X.hv[s];
          if (theta < 1.0) {
            sh = smax(theta * (sh - avg0) + avg0, 0.0);
            shu = theta * (shu - avg1) + avg1;
            shv = theta * (shv - avg2) + avg2;
          }
          if (Ph.limiter && sh < Ph.h_tol) {
            shu = 0.0;
            shv = 0.0;
          }
          A.out.h[n] = sh;
          A.out.hu[n] = shu;
          A.out.hv[n] = shv;
        }
      }
    }
  }
  cp_async_wait_all();
}
