// kernels_fast.cu — the throughput path (SWDG_MODE_FAST): one fused, persistent
// kernel per SSPRK3 stage on sm_100a, FP64 with FMA.
//
// Work decomposition.  Elements are processed in groups of E consecutive
// elements; a CTA owns 2*(N+1) "line threads" per element of its group:
// thread l < N+1 owns the xi-line j=l, thread l >= N+1 the eta-line
// i=l-(N+1).  A line thread keeps its line's nodal data and accumulators in
// registers and runs the split-form flux differencing (dg_rhs.hpp:23-71) over
// the UNORDERED node pairs of its line: the two-point flux F#(a,b) and the
// averaged metrics are symmetric, so each pair is evaluated
// once and scattered to both nodes with Dtilde(a,b), Dtilde(b,a) — 19 DP
// instructions per pair instead of 2x16.  The same thread adds its half of the
// split bathymetry source (dg_rhs.hpp:154-183) and the entropy-stable
// interface flux (fluxes.hpp:136-166) at its two endpoints, which are exactly
// the element's face nodes.  The eta-line threads then finish their nodes:
// -1/J, forcing, the SSPRK3 update (timeloop.hpp:114-127), the element mean,
// Zhang-Shu limiter and dry-node cut (limiter.hpp:24-84) and the reject
// signal (timeloop.hpp:205-209); the stage output is written once.
//
// Memory pipeline.  CTAs are persistent (grid = resident CTAs) and loop over
// groups.  While group g is computed, the TMA engine streams group g+1's
// line data (state + metrics + b + face connectivity) into shared memory with
// cp.async.bulk (one instruction per field per group, completion on an
// mbarrier), and group g's node-phase data (J, W^n) arrives the same way
// behind the line phase.  Neighbour face traces are scattered 8-byte reads;
// they are issued as cp.async (LDGSTS) right after the line data lands and
// consumed after the volume loop, so their L2 latency hides behind it.
//
// Conservation: both sides of a face evaluate the same flux bitwise — the
// minus side's normal/J_surf are computed from the minus element's face
// metrics with explicit round-to-nearest intrinsics on both sides, and the
// flux is evaluated at a single call site with the (minus, plus) ordering.
//
// HBM traffic per node and stage: state in 24 B, W^n 24 B (stages 2-3),
// metrics + J + b 48 B, state out 24 B; neighbour traces are L2 hits.
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "fast_common.cuh"

// The file is compiled once per degree range (build.py: SWDG_PART = 0, 1, 2 ->
// N+1 in [2,7], [8,11], [12,16]) so the three objects build in parallel; each
// object has its own constant operator table and exports its launchers with a
// _p<part> suffix (the dispatch is in kernels_common.cu).
#ifndef SWDG_PART
#define SWDG_PART 0
#define SWDG_N1_LO 2
#define SWDG_N1_HI 16
#endif
#if SWDG_PART == 0
#define SWDG_EXPORT(name) name##_p0
#elif SWDG_PART == 1
#define SWDG_EXPORT(name) name##_p1
#else
#define SWDG_EXPORT(name) name##_p2
#endif

// resident half-line CTAs per SM the register allocation is compiled for
// (__launch_bounds__ min blocks), per N+1; the -D overrides are for A/B builds
// viscous stages up to this N+1 take the node-per-thread kernel
#ifndef SWDG_VISC_NODE_MAX
#define SWDG_VISC_NODE_MAX 3  // measured: N=2 1.224 -> 1.013 ms/stage; N+1 = 4 slower (1.585 -> 1.798)
#endif
// half-line: min-height key reduced per CTA (1) or one atomic per element (0);
// -1 = per degree (hl_blockmin)
#ifndef SWDG_HL_BLOCKMIN
#define SWDG_HL_BLOCKMIN -1
#endif
#ifndef SWDG_HL_MB5
#define SWDG_HL_MB5 4
#endif
#ifndef SWDG_HL_MB6
#define SWDG_HL_MB6 4
#endif
#ifndef SWDG_HL_MB7
#define SWDG_HL_MB7 4
#endif

// viscous stages from this N+1 on: the eta lines apply the source and -1/J to
// their half before the hand-over (HL::PRE)
#ifndef SWDG_HL_PRE_VMIN
#define SWDG_HL_PRE_VMIN 16  // measured: viscous N=15 44.4 -> 40.1 ms/stage; N+1 = 13..15 1-4% slower
#endif

#ifndef SWDG_HL_CLAIM_AHEAD
#define SWDG_HL_CLAIM_AHEAD 0
#endif
#ifndef SWDG_HL_XROLL
#define SWDG_HL_XROLL 0  // > 0: roll the streamed-node loops from this N+1 on (A/B)
#endif

namespace swdg_dev {

namespace {

// dynamic group scheduling: groups [0, gridDim.x) are taken statically by the
// first wave, the rest in claim order (persistent CTAs stay in one wavefront)
__device__ __forceinline__ int next_group(int* ctr, int grp) {
  return ctr ? (int)gridDim.x + atomicAdd(ctr, 1) : grp + (int)gridDim.x;
}

// ===========================================================================
// Half-line variant (N+1 >= 5).  Every line is split into A = nodes [0,H) and
// B = [H,N+1); the A halves of 32 consecutive lines form one warp ("X"), their
// B halves the next warp ("Y"), so the two code paths never diverge inside a
// warp and each thread holds half a line: ~half the registers of the
// full-line kernel, twice the resident warps.  X evaluates the A-A pairs and
// the A x B0 cross pairs (streaming B0 nodes from shared memory), Y the B-B
// pairs and the A x B1 cross pairs (streaming A); the cross contributions for
// the streamed nodes go back through shared memory.  The line data lands in a
// row-padded layout (stride N+2) via 8-byte cp.async, so both the xi-line
// (column) and eta-line (row) reads are bank-conflict free.  The node phase
// runs on the xi-line threads, whose nodes (k, j) make coalesced rows.
template <int N1, bool V = false>
struct HL {
  static constexpr bool kVisc = V;
  static constexpr int NP = N1 * N1, LE = 2 * N1;
  static constexpr int H = (N1 + 1) / 2, NB = N1 - H;
  static constexpr int work_x(int b0) { return H * (H - 1) / 2 + H * b0; }
  static constexpr int work_y(int b0) { return NB * (NB - 1) / 2 + H * (NB - b0); }
  static constexpr int best_b0() {
    int best = 0, bd = 1 << 30;
    for (int b0 = 0; b0 <= NB; ++b0) {
      const int d = work_x(b0) > work_y(b0) ? work_x(b0) - work_y(b0) : work_y(b0) - work_x(b0);
      if (d < bd) {
        bd = d;
        best = b0;
      }
    }
    return best;
  }
  static constexpr int NB0 = best_b0();
  // Warp roles: (xi, X), (xi, Y), (eta, X), (eta, Y) — every branch on the line
  // direction or the half is warp-uniform.  A role covers the E*(N+1) lines of
  // its kind in WR warps; E maximises lane use with WR <= 2 (even E for odd N+1
  // keeps the bulk copies 16-byte aligned).
  static constexpr int lanes_used(int e) { return e * N1; }
  static constexpr int warps_for(int e) { return (e * N1 + 31) / 32; }
  static constexpr int pick_e() {
    // one warp per role while that fills >= 80% of the lanes (N+1 <= 10), else up
    // to two; odd E works for odd N+1 (the node-field bulk copies shift by one):
    // N+1 = 11 takes E = 5 (86% of 64 lanes), measured 8.6 -> 7.0 ms/stage
    int best = 2, bu = 0;
    const int wmax = 32 / N1 * N1 * 10 >= 32 * 8 ? 1 : 2;
    for (int e = 2; e <= 32; ++e) {
      if (warps_for(e) > wmax) break;
      const int u = 1000 * lanes_used(e) / (32 * warps_for(e));
      if (u > bu) {
        bu = u;
        best = e;
      }
    }
    return best;
  }
  static constexpr int E = pick_e();
  static constexpr int L = E * LE;          // lines per CTA
  static constexpr int WR = warps_for(E);   // warps per role
  static constexpr int WP = 2 * WR;         // warps per half (both directions)
  static constexpr int THREADS = 128 * WR;
  static constexpr int PAD = N1 | 1;       // odd padded row stride: conflict-free rows and columns
  static constexpr int EPAD = N1 * PAD;    // one padded element field
  static constexpr int GPAD = E * EPAD;
  static constexpr int GNP = (E * NP + 3) & ~1;  // node field stride (+ shift slack)
  // line fields; the viscous variant adds the physical viscous flux pairs
  enum { F_H, F_HU, F_HV, F_YE, F_XE, F_YX, F_XX, F_FVU, F_GVU, F_FVV, F_GVV };
  static constexpr int kLineFields = V ? 11 : 7;
  static constexpr int kTr = V ? 11 : 7;  // trace slots per face node
  // node fields staged per group; the viscous N+1 = 16 variant reads S_x, S_y
  // straight from global memory (its shared memory then fits two CTAs per SM)
  static constexpr bool kSxGlobal = V && N1 >= 16;
  enum { N_JAC, N_WH, N_WHU, N_WHV, N_SX, N_SY };
  static constexpr int kNodeFields = kSxGlobal ? 4 : 6;
  static constexpr int XS = 3 * (NB0 + H);  // exchange slots per line
  static constexpr int LP = 32 * WP;        // lane slots per part (>= L; tail lanes idle)
  // shared-memory plan, in doubles.  The line data is double-buffered (group
  // g+1 streams in while g is computed) when the second buffer still lets the
  // register-limited number of CTAs share an SM.
  static constexpr int LBUF = kLineFields * GPAD;
  static constexpr int rest() {
    return 3 * GPAD + LP * XS + kNodeFields * GNP + E * 4 * N1 * kTr + 2 * E * 4 * 2 +
           2 * E * 2 * 5 + 2;
  }
  static constexpr int kCtas = THREADS > 128 ? 1 : (N1 <= 8 ? 3 : 2);  // register-bound residency
  static constexpr bool DB = false && (size_t)(2 * LBUF + rest()) * 8 * kCtas + kCtas * 1024 <= 227 * 1024;
  static constexpr int NBUF = DB ? 2 : 1;
  static constexpr int LINE = 0;
  static constexpr int ACC = LINE + NBUF * LBUF;
  // eta-line hand-over: 3 accumulators, plus -1/J (PRE: the eta lines apply the
  // source and -1/J to their half before handing over)
  static constexpr bool PRE = V && N1 >= SWDG_HL_PRE_VMIN;
  static constexpr int XCH = ACC + (PRE ? 4 : 3) * GPAD;
  static constexpr int NODE = XCH + LP * XS;
  static constexpr int TR = NODE + kNodeFields * GNP;  // [kTr][E][4][N1]
  static constexpr int EFO = TR + E * 4 * N1 * kTr;     // int4 [NBUF][E][4]
  static constexpr int RED = EFO + 2 * E * 4 * 2;      // [2 parts][E][2 pieces][5]
  static constexpr int BAR = RED + 2 * E * 2 * 5;
  // one instantiation of the group loop per line direction (XI_SPLIT): measured
  // (B200, 1M elements) inviscid N=5 1.615 -> 1.463 ms/stage; slower at every
  // other degree (twice the code: N=8 4.34 -> 5.16, N=15 13.2 -> 27.0)
  static constexpr bool XI_SPLIT = !V && N1 == 6;
  static constexpr int TOTAL = BAR + 2;
  static constexpr size_t bytes = TOTAL * sizeof(double);
};

// symmetric two-point contravariant flux of one pair, scaled (4F0, 8F1, 8F2)
__device__ __forceinline__ void pair_flux(double ha, double ua, double va, double hua,
                                          double hva, double Aa, double Ba, double hb,
                                          double ub, double vb, double hub, double hvb,
                                          double Ab, double Bb, double g2, double& F0,
                                          double& T1, double& T2) {
  const double Shu = hua + hub, Shv = hva + hvb, Su = ua + ub, Sv = va + vb;
  const double SA = Aa + Ab, SB = Ba + Bb;
  F0 = SA * Shu - SB * Shv;
  const double Q = g2 * ha * hb;
  T1 = Su * F0 + Q * SA;
  T2 = Sv * F0 - Q * SB;
}

template <int N1>
using HArr = double[HL<N1>::H];

template <int N1, int PART>
__device__ __forceinline__ void hl_intra(const HArr<N1>& h, const HArr<N1>& u,
                                         const HArr<N1>& v, const HArr<N1>& hu,
                                         const HArr<N1>& hv, const HArr<N1>& Am,
                                         const HArr<N1>& Bm, HArr<N1>& r0, HArr<N1>& r1,
                                         HArr<N1>& r2, double g2) {
  using O = Ops<N1>;
  constexpr int H = HL<N1>::H, NK = PART ? N1 - H : H, OFF = PART ? H : 0;
  constexpr int CORNER = PART ? NK - 1 : 0;  // node 0 (X) / node N (Y): Dtilde(i,i) != 0
#pragma unroll
  for (int a = 0; a < NK; ++a) {
#pragma unroll
    for (int b = a; b < NK; ++b) {
      if (a == b && a != CORNER) continue;
      double F0, T1, T2;
      pair_flux(h[a], u[a], v[a], hu[a], hv[a], Am[a], Bm[a], h[b], u[b], v[b], hu[b], hv[b],
                Am[b], Bm[b], g2, F0, T1, T2);
      r0[a] += O::D4(OFF + a, OFF + b) * F0;
      r1[a] += O::D8(OFF + a, OFF + b) * T1;
      r2[a] += O::D8(OFF + a, OFF + b) * T2;
      if (a != b) {
        r0[b] += O::D4(OFF + b, OFF + a) * F0;
        r1[b] += O::D8(OFF + b, OFF + a) * T1;
        r2[b] += O::D8(OFF + b, OFF + a) * T2;
      }
    }
  }
}

template <int N1, bool V>
__device__ __forceinline__ void hl_prefetch_line(double* sm, const Mesh& M, const CState& in,
                                                 const StageArgs& A, int g, int tid, int buf) {
  using P = HL<N1, V>;
  const int e0 = M.e_lo + g * P::E, ne = min(P::E, M.n_owned - e0);
  const long long base = (long long)e0 * P::NP;
  const int cnt = ne * P::NP;
  // one node per pass, all fields; the padded shared offset of a thread's node
  // is the same for every group (divisions by constants, folded per pass)
  constexpr int PF = (P::E * P::NP + P::THREADS - 1) / P::THREADS;
#pragma unroll(PF <= 2 ? PF : 1)
  for (int m = 0; m < PF; ++m) {
    const int r = tid + m * P::THREADS;
    if (r >= cnt) break;
    const int el = r / P::NP, q = r - el * P::NP;
    const int i = q / N1, j = q - i * N1;
    double* d = sm + P::LINE + buf * P::LBUF + el * P::EPAD + i * P::PAD + j;
    const long long s = base + r;
    cp_async8(d + P::F_H * P::GPAD, in.h + s);
    cp_async8(d + P::F_HU * P::GPAD, in.hu + s);
    cp_async8(d + P::F_HV * P::GPAD, in.hv + s);
    cp_async8(d + P::F_YE * P::GPAD, M.ye + s);
    cp_async8(d + P::F_XE * P::GPAD, M.xe + s);
    cp_async8(d + P::F_YX * P::GPAD, M.yx + s);
    cp_async8(d + P::F_XX * P::GPAD, M.xx + s);
    if constexpr (V) {
      cp_async8(d + P::F_FVU * P::GPAD, A.fvu + s);
      cp_async8(d + P::F_GVU * P::GPAD, A.gvu + s);
      cp_async8(d + P::F_FVV * P::GPAD, A.fvv + s);
      cp_async8(d + P::F_GVV * P::GPAD, A.gvv + s);
    }
  }
  const int4* ef = M.ef + (long long)e0 * 4;
  int4* dst = reinterpret_cast<int4*>(sm + P::EFO) + buf * P::E * 4;
  for (int idx = tid; idx < ne * 4; idx += P::THREADS)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst + idx)),
                 "l"(ef + idx)
                 : "memory");
}

template <int N1, bool V>
__device__ __forceinline__ void hl_issue_node(double* sm, const Mesh& M, const StageArgs& A,
                                              int g, uint64_t* bar) {
  using P = HL<N1, V>;
  const int e0 = M.e_lo + g * P::E, ne = min(P::E, M.n_owned - e0);
  // bulk copies need 16-byte aligned sources: an odd first node is copied from
  // one double earlier and the group's data starts at offset (e0 * NP) & 1
  const int shift = (int)(((long long)e0 * P::NP) & 1);
  const uint32_t fb = round16((size_t)(ne * P::NP + shift) * sizeof(double));
  const bool wn = A.update && A.stage > 0;
  mbar_expect_tx(bar, ((wn ? 4 : 1) + (P::kSxGlobal ? 0 : 2)) * fb);
  const long long off = (long long)e0 * P::NP - shift;
  bulk_g2s(sm + P::NODE + P::N_JAC * P::GNP, M.jac + off, fb, bar);
  if constexpr (!P::kSxGlobal) {
    bulk_g2s(sm + P::NODE + P::N_SX * P::GNP, M.sx + off, fb, bar);
    bulk_g2s(sm + P::NODE + P::N_SY * P::GNP, M.sy + off, fb, bar);
  }
  if (wn) {
    bulk_g2s(sm + P::NODE + P::N_WH * P::GNP, A.wn.h + off, fb, bar);
    bulk_g2s(sm + P::NODE + P::N_WHU * P::GNP, A.wn.hu + off, fb, bar);
    bulk_g2s(sm + P::NODE + P::N_WHV * P::GNP, A.wn.hv + off, fb, bar);
  }
}

// strong-form divergence of the contravariant viscous fluxes along this line
// (viscosity.hpp:200-222): ft(m) = A(m) fv(m) - B(m) gv(m) for both directions
// (A,B = (y_eta,x_eta) on xi-lines, -(y_xi,x_xi) on eta-lines); subtract D ft
// from this half's momentum accumulators (the reference's res -= viscous_lhs)
template <int N1, int PART, bool V>
__device__ __forceinline__ void hl_visc_div(const double* Lb, int li, bool xi,
                                            const HArr<N1>& Am, const HArr<N1>& Bm,
                                            HArr<N1>& r1, HArr<N1>& r2) {
  using O = Ops<N1>;
  using P = HL<N1, V>;
  constexpr int H = P::H, NK = PART ? N1 - H : H, OFF = PART ? H : 0;
#pragma unroll
  for (int m = 0; m < N1; ++m) {
    const int q = xi ? m * P::PAD + li : li * P::PAD + m;
    double A_m, B_m;
    if (m >= OFF && m < OFF + NK) {  // own half: metrics already in registers
      A_m = Am[m - OFF];
      B_m = Bm[m - OFF];
    } else {
      A_m = xi ? Lb[P::F_YE * P::GPAD + q] : -Lb[P::F_YX * P::GPAD + q];
      B_m = xi ? Lb[P::F_XE * P::GPAD + q] : -Lb[P::F_XX * P::GPAD + q];
    }
    const double ftu = A_m * Lb[P::F_FVU * P::GPAD + q] - B_m * Lb[P::F_GVU * P::GPAD + q];
    const double ftv = A_m * Lb[P::F_FVV * P::GPAD + q] - B_m * Lb[P::F_GVV * P::GPAD + q];
#pragma unroll
    for (int s = 0; s < NK; ++s) {
      r1[s] -= O::D(OFF + s, m) * ftu;
      r2[s] -= O::D(OFF + s, m) * ftv;
    }
  }
}

// streamed-node loops rolled (1) or unrolled (0) per configuration, measured
// (ms/stage, 1M elements, profiles/r02_ab_hl_roll.txt): inviscid N+1 = 6 1.461 ->
// 1.444, 7 2.365 -> 2.111, 10 4.440 -> 4.351; viscous N+1 = 8 6.02 -> 5.89,
// 9 8.51 -> 7.79, 10 11.56 -> 10.87, 14 25.2 -> 24.6, 15 33.2 -> 31.2, 16 39.8 ->
// 38.9; slower or neutral elsewhere (inviscid N+1 = 12: 7.47 -> 7.84, 16: 13.6 ->
// 14.1).  At N+1 = 9 the rolled loops replaced the transposed node phase (a
// thread-per-node node phase over the group, with the xi lines' accumulators and
// state handed over through shared memory), which had been the faster choice
// there unrolled: 4.37 -> 4.06 ms/stage.  SWDG_HL_XROLL > 0 rolls every N+1 >= it.
__host__ __device__ constexpr bool hl_roll(int n1, bool visc) {
  return SWDG_HL_XROLL > 0 ? n1 >= SWDG_HL_XROLL
         : visc ? (n1 >= 8 && n1 <= 10) || n1 >= 14 : (n1 == 6 || n1 == 7 || n1 == 9 || n1 == 10);
}

// The node-data bulk copies and the next-group claim (an atomic round trip) are
// issued by one thread per group: the first xi-X lane, or (true) a lane of the
// last eta-Y warp, which idles during the node phase.  Measured per configuration
// (ms/stage, profiles/r02_ab_hl_issuer.txt): eta-Y faster at inviscid N+1 = 9
// (4.05 -> 3.95), 14..16 (1-2%), viscous 8..10 and 13..16 (1-4%: N+1 = 10 10.82 ->
// 10.40 ms); slower at inviscid N+1 = 5..8 and 11, 12 (2-4%), viscous 5..7, 11, 12.
__host__ __device__ constexpr bool hl_eta_issuer(int n1, bool visc) {
  return visc ? (n1 >= 8 && n1 != 11 && n1 != 12) : (n1 == 9 || n1 >= 14);
}

// resident CTAs the register allocation must allow: 4 (<= 128 registers) for
// N+1 = 5..7 (measured on B200, 1M elements: N=4 1.352 -> 1.132, N=5 1.635 ->
// 1.609, N=6 2.438 -> 2.374 ms/stage; at N+1 = 8 the 128-register cap spills 88
// bytes and runs 11% slower), 3 (<= 168 registers) up to N+1 = 10 (measured 22%
// faster at N+1 = 10); above, a 168-register cap spills (N+1 = 11, 13..16)
// The viscous variant keeps 3 at N+1 = 6, 7 (measured: N=5 3.566 vs 3.721, N=6
// 5.180 vs 5.547 ms/stage with 4) and takes 4 at N+1 = 5 (2.777 -> 2.559).
__host__ __device__ constexpr int hl_min_blocks(int n1, bool visc) {
  return n1 == 5 ? SWDG_HL_MB5 : (n1 == 6 && !visc) ? SWDG_HL_MB6
         : (n1 == 7 && !visc) ? SWDG_HL_MB7 : n1 <= 10 ? 3 : 1;
}

// One min-height atomic per CTA instead of one per element (1M same-address
// atomics per launch): viscous N=3 2.08 -> 1.58, N=2 1.29 -> 1.22 ms/stage.
// Inviscid per CTA too at N+1 = 9, 15 (round 2: 3.956 -> 3.924, 12.77 -> 12.65
// ms/stage); elsewhere per element: within +-1.5% at N = 4, 5, 7, 10, and the extra
// register pushed N+1 = 7 (128-register cap) from 48 to 60 B of spills (N=6
// 2.375 -> 2.520 ms)
__host__ __device__ constexpr bool hl_blockmin(int n1, bool visc) {
  return SWDG_HL_BLOCKMIN >= 0 ? SWDG_HL_BLOCKMIN != 0 : visc || n1 == 9 || n1 == 15;
}

template <int N1, bool FORCE, bool VISC>
__global__ void __launch_bounds__(HL<N1, VISC>::THREADS, hl_min_blocks(N1, VISC))
    k_stage_hl(Mesh M, Phys Ph, StageArgs A, Flags* F) {
  using P = HL<N1, VISC>;
  using O = Ops<N1>;
  constexpr int NP = N1 * N1, H = P::H, NB0 = P::NB0, PAD = P::PAD;
  constexpr int S = (H > N1 - H) ? H : N1 - H;  // register slots per thread
  extern __shared__ __align__(16) double sm[];
  uint64_t* bar_node = reinterpret_cast<uint64_t*>(sm + P::BAR);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int role = warp / P::WR;               // 0 xi-X, 1 xi-Y, 2 eta-X, 3 eta-Y
  const int part = role & 1;                   // 0: X (A half), 1: Y (B half)
  const bool xi = role < 2;
  const int lr = (warp % P::WR) * 32 + lane;   // el * (N+1) + li within the role
  const bool line_ok = lr < P::E * N1;
  const int el = lr / N1, li = lr - el * N1;
  const int line = (xi ? 0 : P::WR * 32) + lr;  // exchange/reduction slot of the line
  const int k0 = part ? H : 0;                  // first node of this thread's half
  const int nk = part ? N1 - H : H;             // nodes held
  const int ngroups = (M.n_owned - M.e_lo + P::E - 1) / P::E;
  const double g = Ph.g, h_des = Ph.h_des, inv2g = 1.0 / (2.0 * g), iw0 = 1.0 / M.w0;
  const double g2 = 2.0 * g;

  if (tid == 0) {
    mbar_init(bar_node, 1);
    fence_mbar_init();
  }
  if ((int)blockIdx.x >= ngroups) return;
  hl_prefetch_line<N1, VISC>(sm, M, A.in, A, blockIdx.x, tid, 0);
  cp_async_commit();
  uint32_t ph_node = 0;
  int buf = 0;

  __shared__ int s_next;  // the next group, claimed by thread 0
  int pending = -1;       // SWDG_HL_CLAIM_AHEAD: the issuer's claim one group ahead
  unsigned long long kmin = ~0ull;  // min height key of this thread's elements
  // With HL::XI_SPLIT the group loop is instantiated per line direction (xi is
  // warp-uniform): the metric selection (y_eta, x_eta) / -(y_xi, x_xi), the padded
  // addressing and the xi-only node phase become compile-time.  Every
  // instantiation passes the same barriers in the same order.
  auto group_loop = [&](auto xi_c) {
  const bool xi = xi_c;  // a compile-time constant when xi_c is std::integral_constant
  // padded in-element offset of node k of this line
  auto pidx = [&](int k) { return xi ? k * PAD + li : li * PAD + k; };
  for (int grp = blockIdx.x; grp < ngroups; grp = s_next, buf = P::DB ? buf ^ 1 : 0) {
    const int e0 = M.e_lo + grp * P::E, ne = min(P::E, M.n_owned - e0);
    const bool active = line_ok && el < ne;
    const int e = e0 + el;
    cp_async_wait_all();
    __syncthreads();  // line(g) and connectivity(g) resident for every thread
    if (tid == (hl_eta_issuer(N1, VISC) ? P::THREADS - 32 : 0)) {
      fence_proxy_async();
      hl_issue_node<N1, VISC>(sm, M, A, grp, bar_node);
      if constexpr (SWDG_HL_CLAIM_AHEAD || (N1 == 8 && !VISC)) {
        // the atomic's result is used a group later (measured: N=7 2.420 -> 2.406
        // ms/stage; N=6 2.11 -> 2.31, others within +-1.5%,
        // profiles/r02_ab_hl_issuer.txt)
        if (pending < 0) pending = next_group(A.gctr, grp);
        s_next = pending;
        if (pending < ngroups) pending = next_group(A.gctr, pending);
      } else {
        s_next = next_group(A.gctr, grp);  // read by all threads after the next barrier
      }
    }

    // ---- own half -> registers, gathers for the own endpoint
    double h[S], u[S], v[S], hu[S], hv[S], Am[S], Bm[S], r0[S], r1[S], r2[S];
    const double* Lb = sm + P::LINE + buf * P::LBUF + el * P::EPAD;
#pragma unroll
    for (int s = 0; s < S; ++s) {
      r0[s] = r1[s] = r2[s] = 0.0;
      h[s] = hu[s] = hv[s] = Am[s] = Bm[s] = u[s] = v[s] = 0.0;
      if (s < nk && active) {
        const int q = pidx(k0 + s);
        h[s] = Lb[P::F_H * P::GPAD + q];
        hu[s] = Lb[P::F_HU * P::GPAD + q];
        hv[s] = Lb[P::F_HV * P::GPAD + q];
        Am[s] = xi ? Lb[P::F_YE * P::GPAD + q] : -Lb[P::F_YX * P::GPAD + q];
        Bm[s] = xi ? Lb[P::F_XE * P::GPAD + q] : -Lb[P::F_XX * P::GPAD + q];
        vel(h[s], hu[s], hv[s], h_des, u[s], v[s]);
      }
    }
    const int face = xi ? (part ? 1 : 3) : (part ? 2 : 0);
    int efy = 0;
    // trace slots are component-major ([8][E][4][N+1]): consecutive lanes hit
    // consecutive words (no bank conflicts)
    constexpr int TRS = P::E * 4 * N1;
    double* tr = sm + P::TR + (el * 4 + face) * N1 + li;
    if (active) {
      const int4 ef = reinterpret_cast<const int4*>(sm + P::EFO)[(buf * P::E + el) * 4 + face];
      efy = ef.y;
      const long long own = (long long)e * NP + face_node(N1, face, li);
      cp_async8(tr + 6 * TRS, M.b + own);
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
        if constexpr (VISC) {  // the neighbour's viscous flux pairs for the penalty
          cp_async8(tr + 7 * TRS, A.fvu + nb);
          cp_async8(tr + 8 * TRS, A.gvu + nb);
          cp_async8(tr + 9 * TRS, A.fvv + nb);
          cp_async8(tr + 10 * TRS, A.gvv + nb);
        }
      }
    }
    cp_async_commit();
    if constexpr (P::DB) {  // next group's line data into the other buffer, now
      __syncthreads();
      const int gn = s_next;
      if (gn < ngroups) hl_prefetch_line<N1, VISC>(sm, M, A.in, A, gn, tid, buf ^ 1);
      cp_async_commit();
    }

    // ---- volume: pairs inside the own half (+ the corner diagonal); part is
    // warp-uniform, so each warp runs one fully unrolled, constant-operand body
    if (part == 0)
      hl_intra<N1, 0>(h, u, v, hu, hv, Am, Bm, r0, r1, r2, g2);
    else
      hl_intra<N1, 1>(h, u, v, hu, hv, Am, Bm, r0, r1, r2, g2);
    // ---- cross pairs: X streams B0 = [H, H+NB0), Y streams A = [0, H)
    // exchange slots are slot-major ([XS][LP]): consecutive lanes, consecutive words
    double* xch_base = sm + P::XCH + line;
    auto xch = [&](int slot) -> double& { return xch_base[slot * P::LP]; };
    // the streamed-node loops stay rolled where that measured faster (hl_roll: less
    // code for the instruction cache, fewer live registers; the inner loops over the
    // register-held half stay unrolled, the operator entries become warp-uniform
    // constant loads)
    constexpr int XU = hl_roll(N1, VISC) ? 1 : 32;
    if (part == 0) {
#pragma unroll(XU)
      for (int s = 0; s < NB0; ++s) {
        const int q = pidx(H + s);
        const double hb = Lb[P::F_H * P::GPAD + q], hub = Lb[P::F_HU * P::GPAD + q],
                     hvb = Lb[P::F_HV * P::GPAD + q];
        const double Ab = xi ? Lb[P::F_YE * P::GPAD + q] : -Lb[P::F_YX * P::GPAD + q];
        const double Bb = xi ? Lb[P::F_XE * P::GPAD + q] : -Lb[P::F_XX * P::GPAD + q];
        double ub, vb;
        vel(hb, hub, hvb, h_des, ub, vb);
        double c0 = 0.0, c1 = 0.0, c2 = 0.0;
#pragma unroll
        for (int a = 0; a < H; ++a) {
          double F0, T1, T2;
          pair_flux(h[a], u[a], v[a], hu[a], hv[a], Am[a], Bm[a], hb, ub, vb, hub, hvb, Ab, Bb,
                    g2, F0, T1, T2);
          r0[a] += O::D4(a, H + s) * F0;
          r1[a] += O::D8(a, H + s) * T1;
          r2[a] += O::D8(a, H + s) * T2;
          c0 += O::D4(H + s, a) * F0;
          c1 += O::D8(H + s, a) * T1;
          c2 += O::D8(H + s, a) * T2;
        }
        xch(3 * s + 0) = c0;
        xch(3 * s + 1) = c1;
        xch(3 * s + 2) = c2;
      }
    } else {
#pragma unroll(XU)
      for (int a = 0; a < H; ++a) {
        const int q = pidx(a);
        const double ha = Lb[P::F_H * P::GPAD + q], hua = Lb[P::F_HU * P::GPAD + q],
                     hva = Lb[P::F_HV * P::GPAD + q];
        const double Aa = xi ? Lb[P::F_YE * P::GPAD + q] : -Lb[P::F_YX * P::GPAD + q];
        const double Ba = xi ? Lb[P::F_XE * P::GPAD + q] : -Lb[P::F_XX * P::GPAD + q];
        double ua, va;
        vel(ha, hua, hva, h_des, ua, va);
        double c0 = 0.0, c1 = 0.0, c2 = 0.0;
#pragma unroll
        for (int s = NB0; s < N1 - H; ++s) {
          double F0, T1, T2;
          pair_flux(ha, ua, va, hua, hva, Aa, Ba, h[s], u[s], v[s], hu[s], hv[s], Am[s], Bm[s],
                    g2, F0, T1, T2);
          r0[s] += O::D4(H + s, a) * F0;
          r1[s] += O::D8(H + s, a) * T1;
          r2[s] += O::D8(H + s, a) * T2;
          c0 += O::D4(a, H + s) * F0;
          c1 += O::D8(a, H + s) * T1;
          c2 += O::D8(a, H + s) * T2;
        }
        xch(3 * NB0 + 3 * a + 0) = c0;
        xch(3 * NB0 + 3 * a + 1) = c1;
        xch(3 * NB0 + 3 * a + 2) = c2;
      }
    }
    // ---- viscous divergence along the line, own endpoint flux pairs kept for the
    // penalty (the line buffer is recycled after the next barrier)
    double fvo[4] = {0.0, 0.0, 0.0, 0.0};
    if constexpr (VISC) {
      if (part == 0)
        hl_visc_div<N1, 0, VISC>(Lb, li, xi, Am, Bm, r1, r2);
      else
        hl_visc_div<N1, 1, VISC>(Lb, li, xi, Am, Bm, r1, r2);
      const int qe = pidx(part ? N1 - 1 : 0);
      fvo[0] = Lb[P::F_FVU * P::GPAD + qe];
      fvo[1] = Lb[P::F_GVU * P::GPAD + qe];
      fvo[2] = Lb[P::F_FVV * P::GPAD + qe];
      fvo[3] = Lb[P::F_GVV * P::GPAD + qe];
    }
    __syncthreads();  // cross contributions published; line buffer free
    // the partner half's exchange slots: X (line's A) gets Y's, Y gets X's
    if (part == 0) {
#pragma unroll
      for (int a = 0; a < H; ++a) {
        r0[a] += xch(3 * NB0 + 3 * a + 0);
        r1[a] += xch(3 * NB0 + 3 * a + 1);
        r2[a] += xch(3 * NB0 + 3 * a + 2);
      }
    } else {
#pragma unroll
      for (int s = 0; s < NB0; ++s) {
        r0[s] += xch(3 * s + 0);
        r1[s] += xch(3 * s + 1);
        r2[s] += xch(3 * s + 2);
      }
    }
    if constexpr (!P::DB) {  // single buffer: prefetch behind the rest of this group
      const int gn = s_next;
      if (gn < ngroups) hl_prefetch_line<N1, VISC>(sm, M, A.in, A, gn, tid, 0);
      cp_async_commit();
    }

    // ---- interface flux at the own endpoint (dg_rhs.hpp:202-252)
    asm volatile("cp.async.wait_group 1;" ::: "memory");  // gathers(g); line(g+1) may fly
    if (active && (efy & EF_PRESENT)) {
      constexpr int SY = (N1 - H) - 1;  // Y's endpoint slot (node N); X's is slot 0
      const double hs = part ? h[SY] : h[0], hus = part ? hu[SY] : hu[0];
      const double hvs = part ? hv[SY] : hv[0];
      const double As = part ? Am[SY] : Am[0], Bs = part ? Bm[SY] : Bm[0];
      const double om0 = xi ? As : -As, om1 = xi ? Bs : -Bs;
      const double bo = tr[6 * TRS];
      // own velocities from the volume phase (the same vel() the neighbour
      // applies to the gathered trace: both sides see identical bits)
      const double us = part ? u[SY] : u[0], vs = part ? v[SY] : v[0];
      const double cs = wave_c(g, hs);
      double hn, hun, hvn, bn, un, vn, nx, ny, js, sgn = 1.0;
      if (efy & EF_MINUS) {
        face_normal(face, om0, om1, nx, ny, js);
        if (efy & EF_WALL) {  // exterior_state (mesh.hpp:382-386)
          const double mn = hus * nx + hvs * ny;
          hn = hs;
          hun = hus - 2.0 * mn * nx;
          hvn = hvs - 2.0 * mn * ny;
          bn = bo;
        } else {
          hn = tr[0 * TRS];
          hun = tr[1 * TRS];
          hvn = tr[2 * TRS];
          bn = tr[3 * TRS];
        }
      } else {
        face_normal(efy & EF_NBR_FACE_MASK, tr[4 * TRS], tr[5 * TRS], nx, ny, js);
        hn = tr[0 * TRS];
        hun = tr[1 * TRS];
        hvn = tr[2 * TRS];
        bn = tr[3 * TRS];
        sgn = -1.0;
      }
      vel(hn, hun, hvn, h_des, un, vn);
      const double cn = wave_c(g, hn);
      double f0, f1, f2;
      if (sgn > 0.0)
        es_flux_pre(hs, us, vs, cs, hn, un, vn, cn, bo, bn, nx, ny, g, inv2g, f0, f1, f2);
      else
        es_flux_pre(hn, un, vn, cn, hs, us, vs, cs, bn, bo, nx, ny, g, inv2g, f0, f1, f2);
      const double c = sgn * js * iw0;
      if constexpr (VISC) {
        // viscous interface penalty (viscosity.hpp:224-246): with the minus-side
        // normal, du = (phi+ - phi-)/2 lands on both sides; walls take 0 - phi-
        const double pu_o = nx * fvo[0] + ny * fvo[1], pv_o = nx * fvo[2] + ny * fvo[3];
        double du, dv;
        if (efy & EF_WALL) {
          du = -pu_o;
          dv = -pv_o;
        } else {
          const double pu_n = nx * tr[7 * TRS] + ny * tr[8 * TRS];
          const double pv_n = nx * tr[9 * TRS] + ny * tr[10 * TRS];
          const double sg = (efy & EF_MINUS) ? 1.0 : -1.0;  // (plus - minus)
          du = 0.5 * sg * (pu_n - pu_o);
          dv = 0.5 * sg * (pv_n - pv_o);
        }
        f1 -= du / sgn;  // folded below as c * f: c = sgn js / w0
        f2 -= dv / sgn;
      }
      if (part) {
        r0[SY] += c * f0;
        r1[SY] += c * f1;
        r2[SY] += c * f2;
      } else {
        r0[0] += c * f0;
        r1[0] += c * f1;
        r2[0] += c * f2;
      }
    }
    // eta-line threads hand their accumulators to the xi-line owners
    if constexpr (P::PRE) {
      // the eta lines finish their half of each node before handing it over:
      // split source (dg_rhs.hpp:154-183) and the -1/J scaling, so the xi-line
      // node phase (the longer one) is one FMA per component
      if (active && !xi) {
        mbar_wait(bar_node, ph_node);
        double* acc = sm + P::ACC + el * P::EPAD;
        const double* Nd = sm + P::NODE + (int)(((long long)e0 * NP) & 1) + el * NP;
#pragma unroll
        for (int s = 0; s < S; ++s)
          if (s < nk) {
            const int q = li * N1 + k0 + s, qp = pidx(k0 + s);
            const double ij = -1.0 / Nd[P::N_JAC * P::GNP + q], hg2 = 0.5 * g * h[s];
            const long long n = (long long)e * NP + q;
            const double sxv = P::kSxGlobal ? __ldg(M.sx + n) : Nd[P::N_SX * P::GNP + q];
            const double syv = P::kSxGlobal ? __ldg(M.sy + n) : Nd[P::N_SY * P::GNP + q];
            acc[0 * P::GPAD + qp] = r0[s] * ij;
            acc[1 * P::GPAD + qp] = (r1[s] + hg2 * sxv) * ij;
            acc[2 * P::GPAD + qp] = (r2[s] + hg2 * syv) * ij;
            acc[3 * P::GPAD + qp] = ij;
          }
      }
    }
    if (active && !P::PRE && !xi) {
      double* acc = sm + P::ACC + el * P::EPAD;
#pragma unroll
      for (int s = 0; s < S; ++s)
        if (s < nk) {
          const int q = pidx(k0 + s);
          acc[0 * P::GPAD + q] = r0[s];
          acc[1 * P::GPAD + q] = r1[s];
          acc[2 * P::GPAD + q] = r2[s];
        }
    }
    __syncthreads();
    mbar_wait(bar_node, ph_node);
    ph_node ^= 1;

    // ---- node phase on the xi-line threads: nodes (k, li), k in the own half
    double pv[5] = {0.0, 0.0, 0.0, 0.0, 1.0e300};  // element partials of this thread
    if (xi && active) {
      const double* acc = sm + P::ACC + el * P::EPAD;
      const double* Nd = sm + P::NODE + (int)(((long long)e0 * NP) & 1) + el * NP;
      double s_area = 0.0, s0 = 0.0, s1 = 0.0, s2 = 0.0, mmin = 1.0e300;
      const double wj = O::w(li);
#pragma unroll
      for (int s = 0; s < S; ++s) {
        if (s >= nk) continue;
        const int k = k0 + s, q = k * N1 + li, qp = k * PAD + li;
        const long long n = (long long)e * NP + q;
        const double jac = Nd[P::N_JAC * P::GNP + q];
        double rh, rhu, rhv;
        if constexpr (P::PRE) {
          const double ij = acc[3 * P::GPAD + qp];  // -1/J from the eta line
          rh = __fma_rn(r0[s], ij, acc[0 * P::GPAD + qp]);
          rhu = __fma_rn(r1[s], ij, acc[1 * P::GPAD + qp]);
          rhv = __fma_rn(r2[s], ij, acc[2 * P::GPAD + qp]);
        } else {
          const double ij = -1.0 / jac, hg2 = 0.5 * g * h[s];
          const double sxv = P::kSxGlobal ? __ldg(M.sx + n) : Nd[P::N_SX * P::GNP + q];
          const double syv = P::kSxGlobal ? __ldg(M.sy + n) : Nd[P::N_SY * P::GNP + q];
          rh = (acc[0 * P::GPAD + qp] + r0[s]) * ij;
          rhu = (acc[1 * P::GPAD + qp] + r1[s] + hg2 * sxv) * ij;
          rhv = (acc[2 * P::GPAD + qp] + r2[s] + hg2 * syv) * ij;
        }
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
        double sh = h[s] + A.dt * rh;
        double shu = hu[s] + A.dt * rhu;
        double shv = hv[s] + A.dt * rhv;
        if (A.stage > 0 && A.update) {
          sh = A.ca * Nd[P::N_WH * P::GNP + q] + A.cb * sh;
          shu = A.ca * Nd[P::N_WHU * P::GNP + q] + A.cb * shu;
          shv = A.ca * Nd[P::N_WHV * P::GNP + q] + A.cb * shv;
        }
        h[s] = sh;
        hu[s] = shu;
        hv[s] = shv;
        const double wq = O::w(k) * wj * jac;
        s_area += wq;
        s0 += wq * sh;
        s1 += wq * shu;
        s2 += wq * shv;
        mmin = smin(mmin, sh);
      }
      pv[0] = s_area;
      pv[1] = s0;
      pv[2] = s1;
      pv[3] = s2;
      pv[4] = mmin;
    }
    // element partial sums: segmented shuffle reduction over the xi lanes of each
    // element inside the warp (fixed tree: reproducible), one piece per (warp,
    // element) to shared memory; an element whose lines straddle two warps of
    // its role has two pieces
    if (xi && (32 % N1 == 0)) {
      // N+1 divides 32: each element's lines are an aligned lane segment of
      // N+1 lanes; an xor butterfly leaves the segment sum on all of them
#pragma unroll
      for (int o = N1 / 2; o > 0; o >>= 1) {
#pragma unroll
        for (int c = 0; c < 4; ++c) pv[c] += __shfl_xor_sync(0xffffffffu, pv[c], o);
        pv[4] = smin(pv[4], __shfl_xor_sync(0xffffffffu, pv[4], o));
      }
      if (line_ok && li == 0 && active) {
        double* rr = sm + P::RED + ((part * P::E + el) * 2) * 5;
#pragma unroll
        for (int c = 0; c < 5; ++c) rr[c] = pv[c];
      }
    } else if (xi) {
      const int seg = line_ok ? lr / N1 : -1 - lane;  // element of this lane
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int seg2 = __shfl_down_sync(0xffffffffu, seg, o);
        double t[5];
#pragma unroll
        for (int c = 0; c < 5; ++c) t[c] = __shfl_down_sync(0xffffffffu, pv[c], o);
        if (lane + o < 32 && seg2 == seg) {
#pragma unroll
          for (int c = 0; c < 4; ++c) pv[c] += t[c];
          pv[4] = smin(pv[4], t[4]);
        }
      }
      const bool head = line_ok && (lane == 0 || li == 0);
      if (head && active) {
        double* rr = sm + P::RED + ((part * P::E + el) * 2 + (li == 0 ? 0 : 1)) * 5;
#pragma unroll
        for (int c = 0; c < 5; ++c) rr[c] = pv[c];
      }
    }
    __syncthreads();

    // ---- limiter (limit_element, limiter.hpp:43-84) and write-out, xi threads
    bool lim = xi && active && A.update;
    if (lim) {
      // pieces in a fixed order: part X (first piece, continuation), part Y
      const bool split = (el * N1) / 32 != (el * N1 + N1 - 1) / 32;
      double area = 0.0, a0 = 0.0, a1 = 0.0, a2 = 0.0, mmin = 1.0e300;
#pragma unroll
      for (int pp = 0; pp < 2; ++pp)
#pragma unroll
        for (int pc = 0; pc < 2; ++pc) {
          if (pc == 1 && !split) continue;
          const double* rr = sm + P::RED + ((pp * P::E + el) * 2 + pc) * 5;
          area += rr[0];
          a0 += rr[1];
          a1 += rr[2];
          a2 += rr[3];
          mmin = smin(mmin, rr[4]);
        }
      const double inv = 1.0 / area;
      const double avg0 = inv * a0, avg1 = inv * a1, avg2 = inv * a2;
      const bool lead = part == 0 && li == 0;  // one thread per element
      if (avg0 < 0.0) {  // reject (timeloop.hpp:205-209): nothing written
        if (lead) {
          atomicExch(&F->reject, 1);
          if (!Ph.limiter) atomicExch(&F->abort, 1);
        }
        lim = false;
      }
      double theta = 1.0;
      if (lim && Ph.limiter && mmin < 0.0) {
        const double denom = avg0 - mmin;
        theta = denom < 1e-14 ? 1.0 : smin(1.0, avg0 / denom);
      }
      if (lim && !Ph.limiter && mmin < 0.0 && lead) atomicExch(&F->abort, 1);
      if (lim) {
#pragma unroll
        for (int s = 0; s < S; ++s) {
          if (s >= nk) continue;
          const long long n = (long long)e * NP + (k0 + s) * N1 + li;
          double sh = h[s], shu = hu[s], shv = hv[s];
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
        if (lead) {
          // the limited heights are a monotone map of the unlimited ones: the
          // element's minimum after limiting is the map of its minimum
          const double m = theta < 1.0 ? smax(theta * (mmin - avg0) + avg0, 0.0) : mmin;
          if (hl_blockmin(N1, VISC)) {
            const unsigned long long k = order_key(m);
            kmin = k < kmin ? k : kmin;
          } else {
            atomicMin(&F->min_h_key, order_key(m));
          }
          if (theta < 1.0) atomicAdd(&F->n_limited, 1);
        }
      }
    }
  }
  };
  if constexpr (P::XI_SPLIT) {
    if (role < 2)
      group_loop(std::true_type{});
    else
      group_loop(std::false_type{});
  } else {
    group_loop(role < 2);
  }
  cp_async_wait_all();
  if (hl_blockmin(N1, VISC)) {  // one atomic per CTA for the whole launch
    const unsigned long long bmin = block_min_key(kmin);
    if (tid == 0 && bmin != ~0ull) atomicMin(&F->min_h_key, bmin);
  }
}

// ===========================================================================
// Element-per-thread kernel for the smallest degrees (N+1 <= 3, inviscid).  An
// element is (N+1)^2 <= 9 nodes: one thread loads all of it (vectorised,
// coalesced across the warp), its neighbours' face traces (L2 hits) and does the
// whole stage in registers — volume pairs, source, the 4(N+1) interface
// fluxes, -1/J, SSPRK3 update, element mean, limiter — with no shared memory
// and no barriers.  At these degrees the stage is a stream (HBM bound); what
// matters is many independent loads in flight, which this gives at full
// occupancy.
// element data of one field: NP consecutive doubles, 16-byte vectors when the
// element block is 16-byte aligned (NP even)
template <int NP>
__device__ __forceinline__ void ld_elem(const double* __restrict__ p, long long base,
                                        double (&o)[NP]) {
  if constexpr ((NP & 1) == 0) {
    const double2* v = reinterpret_cast<const double2*>(p + base);
#pragma unroll
    for (int k = 0; k < NP / 2; ++k) {
      const double2 t = __ldg(v + k);
      o[2 * k] = t.x;
      o[2 * k + 1] = t.y;
    }
  } else {
#pragma unroll
    for (int k = 0; k < NP; ++k) o[k] = __ldg(p + base + k);
  }
}

template <int NP>
__device__ __forceinline__ void st_elem(double* __restrict__ p, long long base,
                                        const double (&o)[NP]) {
  if constexpr ((NP & 1) == 0) {
    double2* v = reinterpret_cast<double2*>(p + base);
#pragma unroll
    for (int k = 0; k < NP / 2; ++k) v[k] = make_double2(o[2 * k], o[2 * k + 1]);
  } else {
#pragma unroll
    for (int k = 0; k < NP; ++k) p[base + k] = o[k];
  }
}

template <int N1, bool FORCE>
__global__ void __launch_bounds__(128) k_stage_elem(Mesh M, Phys Ph, StageArgs A, Flags* F) {
  using O = Ops<N1>;
  constexpr int NP = N1 * N1;
  const int e = M.e_lo + blockIdx.x * blockDim.x + threadIdx.x;
  const bool active = e < M.n_owned;
  const long long base = (long long)(active ? e : 0) * NP;
  const double g = Ph.g, h_des = Ph.h_des, inv2g = 1.0 / (2.0 * g), iw0 = 1.0 / M.w0;
  double h[NP], hu[NP], hv[NP], u[NP], v[NP], ye[NP], xe[NP], yx[NP], xx[NP];
  double r0[NP], r1[NP], r2[NP];
  ld_elem<NP>(A.in.h, base, h);
  ld_elem<NP>(A.in.hu, base, hu);
  ld_elem<NP>(A.in.hv, base, hv);
  ld_elem<NP>(M.ye, base, ye);
  ld_elem<NP>(M.xe, base, xe);
  ld_elem<NP>(M.yx, base, yx);
  ld_elem<NP>(M.xx, base, xx);
  int4 efs[4];
#pragma unroll
  for (int face = 0; face < 4; ++face) efs[face] = M.ef[(active ? e : 0) * 4 + face];
#pragma unroll
  for (int q = 0; q < NP; ++q) {
    r0[q] = r1[q] = r2[q] = 0.0;
    vel(h[q], hu[q], hv[q], h_des, u[q], v[q]);
  }
  const double g2 = 2.0 * g;
  // volume: xi-lines (j fixed, metrics (y_eta, x_eta)) and eta-lines (i fixed, -(y_xi, x_xi))
#pragma unroll
  for (int dir = 0; dir < 2; ++dir)
#pragma unroll
    for (int l = 0; l < N1; ++l)
#pragma unroll
      for (int a = 0; a < N1; ++a)
#pragma unroll
        for (int b = a; b < N1; ++b) {
          if (a == b && a != 0 && a != N1 - 1) continue;
          const int qa = dir == 0 ? a * N1 + l : l * N1 + a;
          const int qb = dir == 0 ? b * N1 + l : l * N1 + b;
          const double Aa = dir == 0 ? ye[qa] : -yx[qa], Ba = dir == 0 ? xe[qa] : -xx[qa];
          const double Ab = dir == 0 ? ye[qb] : -yx[qb], Bb = dir == 0 ? xe[qb] : -xx[qb];
          double F0, T1, T2;
          pair_flux(h[qa], u[qa], v[qa], hu[qa], hv[qa], Aa, Ba, h[qb], u[qb], v[qb], hu[qb],
                    hv[qb], Ab, Bb, g2, F0, T1, T2);
          r0[qa] += O::D4(a, b) * F0;
          r1[qa] += O::D8(a, b) * T1;
          r2[qa] += O::D8(a, b) * T2;
          if (a != b) {
            r0[qb] += O::D4(b, a) * F0;
            r1[qb] += O::D8(b, a) * T1;
            r2[qb] += O::D8(b, a) * T2;
          }
        }
  // interface fluxes at the 4 (N+1) face nodes; own velocities reused, one
  // reciprocal and one square root per neighbour trace node
  double bo[NP];
  ld_elem<NP>(M.b, base, bo);
#pragma unroll
  for (int face = 0; face < 4; ++face) {
    const int4 ef = efs[face];
    if (!active || !(ef.y & EF_PRESENT)) continue;
    const int nf = ef.y & EF_NBR_FACE_MASK;
#pragma unroll
    for (int t = 0; t < N1; ++t) {
      const int q = face == 0 ? t * N1 : face == 1 ? (N1 - 1) * N1 + t
                  : face == 2 ? t * N1 + (N1 - 1) : t;
      const bool ew = face == 1 || face == 3;
      const double co = wave_c(g, h[q]);
      double hn, hun, hvn, bn, un = 0.0, vn = 0.0, nx, ny, js, sgn = 1.0;
      if ((ef.y & EF_MINUS) && (ef.y & EF_WALL)) {  // exterior_state (mesh.hpp:382-386)
        face_normal(face, ew ? ye[q] : yx[q], ew ? xe[q] : xx[q], nx, ny, js);
        const double mn = hu[q] * nx + hv[q] * ny;
        hn = h[q];
        hun = hu[q] - 2.0 * mn * nx;
        hvn = hv[q] - 2.0 * mn * ny;
        bn = bo[q];
        vel(hn, hun, hvn, h_des, un, vn);
      } else {
        const int tp = (ef.y & EF_REVERSED) ? N1 - 1 - t : t;
        const long long nb = (long long)ef.x * NP + face_node(N1, nf, tp);
        hn = __ldg(A.in.h + nb);
        hun = __ldg(A.in.hu + nb);
        hvn = __ldg(A.in.hv + nb);
        bn = __ldg(M.b + nb);
        vel(hn, hun, hvn, h_des, un, vn);
        if (ef.y & EF_MINUS) {
          face_normal(face, ew ? ye[q] : yx[q], ew ? xe[q] : xx[q], nx, ny, js);
        } else {
          const bool new_ = nf == 1 || nf == 3;
          face_normal(nf, __ldg((new_ ? M.ye : M.yx) + nb), __ldg((new_ ? M.xe : M.xx) + nb),
                      nx, ny, js);
          sgn = -1.0;
        }
      }
      const double cn = wave_c(g, hn);
      double f0, f1, f2;
      if (sgn > 0.0)
        es_flux_pre(h[q], u[q], v[q], co, hn, un, vn, cn, bo[q], bn, nx, ny, g, inv2g, f0, f1, f2);
      else
        es_flux_pre(hn, un, vn, cn, h[q], u[q], v[q], co, bn, bo[q], nx, ny, g, inv2g, f0, f1, f2);
      const double c = sgn * js * iw0;
      r0[q] += c * f0;
      r1[q] += c * f1;
      r2[q] += c * f2;
    }
  }
  // node phase + element mean (no early returns: warp-collective reductions follow)
  double jac[NP], sxa[NP], sya[NP];
  ld_elem<NP>(M.jac, base, jac);
  ld_elem<NP>(M.sx, base, sxa);
  ld_elem<NP>(M.sy, base, sya);
  const bool comb = A.stage > 0 && A.update;
  double area = 1.0, a0 = 0.0, a1 = 0.0, a2 = 0.0, mmin = 1.0e300;
  if (active) {
    area = 0.0;
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      const long long n = base + q;
      const double ij = -frcp(jac[q]), hg2 = 0.5 * g * h[q];
      double rh = r0[q] * ij;
      double rhu = (r1[q] + hg2 * sxa[q]) * ij;
      double rhv = (r2[q] + hg2 * sya[q]) * ij;
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
      h[q] = h[q] + A.dt * rh;
      hu[q] = hu[q] + A.dt * rhu;
      hv[q] = hv[q] + A.dt * rhv;
    }
    if (comb) {
      double wh[NP], whu[NP], whv[NP];
      ld_elem<NP>(A.wn.h, base, wh);
      ld_elem<NP>(A.wn.hu, base, whu);
      ld_elem<NP>(A.wn.hv, base, whv);
#pragma unroll
      for (int q = 0; q < NP; ++q) {
        h[q] = A.ca * wh[q] + A.cb * h[q];
        hu[q] = A.ca * whu[q] + A.cb * hu[q];
        hv[q] = A.ca * whv[q] + A.cb * hv[q];
      }
    }
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      const double wq = O::w(q / N1) * O::w(q % N1) * jac[q];
      area += wq;
      a0 += wq * h[q];
      a1 += wq * hu[q];
      a2 += wq * hv[q];
      mmin = smin(mmin, h[q]);
    }
  }
  bool lim = active && A.update;
  const double inv = frcp(area);
  const double avg0 = inv * a0, avg1 = inv * a1, avg2 = inv * a2;
  if (lim && avg0 < 0.0) {
    atomicExch(&F->reject, 1);
    if (!Ph.limiter) atomicExch(&F->abort, 1);
    lim = false;
  }
  double theta = 1.0;
  if (lim && Ph.limiter && mmin < 0.0) {
    const double denom = avg0 - mmin;
    theta = denom < 1e-14 ? 1.0 : smin(1.0, avg0 / denom);
  }
  if (lim && !Ph.limiter && mmin < 0.0) atomicExch(&F->abort, 1);
  unsigned long long key = ~0ull;
  if (lim) {
    double mine = 1.0e300;
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      double sh = h[q], shu = hu[q], shv = hv[q];
      if (theta < 1.0) {
        sh = smax(theta * (sh - avg0) + avg0, 0.0);
        shu = theta * (shu - avg1) + avg1;
        shv = theta * (shv - avg2) + avg2;
      }
      if (Ph.limiter && sh < Ph.h_tol) {
        shu = 0.0;
        shv = 0.0;
      }
      h[q] = sh;
      hu[q] = shu;
      hv[q] = shv;
      mine = smin(mine, sh);
    }
    st_elem<NP>(A.out.h, base, h);
    st_elem<NP>(A.out.hu, base, hu);
    st_elem<NP>(A.out.hv, base, hv);
    key = order_key(mine);
  }
  // one atomic per warp for the limited count and the min height
  const unsigned limited = __ballot_sync(0xffffffffu, lim && theta < 1.0);
  key = warp_min_key(key);
  if ((threadIdx.x & 31) == 0) {
    if (limited) atomicAdd(&F->n_limited, __popc(limited));
    atomicMin(&F->min_h_key, key);
  }
}

template <int N1, bool FORCE>
static void launch_elem(const Mesh& M, const Phys& P, const StageArgs& A, Flags* F,
                        cudaStream_t st) {
  k_stage_elem<N1, FORCE><<<(M.n_owned - M.e_lo + 127) / 128, 128, 0, st>>>(M, P, A, F);
}

// Node-per-thread kernel for the smallest degrees (N+1 <= 4, inviscid).  A warp
// holds EPW = 32 / (N+1)^2 whole elements, lane = one node: every load and store
// is one coalesced 8-byte-per-lane stream (the element-per-thread kernel strides
// its lanes by a whole element and runs out of registers for loads in flight).
// The line partners of a node are the lanes of its xi- and eta-line: their
// state, velocity and metrics arrive by warp shuffles, partner k of node i being
// node (i + k) mod (N+1), so no lane idles and no shared memory or barrier is
// needed.  Each lane evaluates its own row of the ordered pairs (the flux is
// symmetric, so the value equals the element kernel's), then the interface
// fluxes of its (at most two) faces — slot s = the node's s-th face, so every
// lane runs the same code — the node update, and the element mean / limiter by
// a segmented shuffle reduction (fixed tree, broadcast from the element's first
// lane: every lane of an element sees the same bits).  Persistent grid-stride
// warps; one flag atomic per block.
template <int N1>
__device__ __forceinline__ double seg_sum(double x, int q, int base_lane) {
  constexpr int NP = N1 * N1;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    if (off >= NP) continue;
    const double o = __shfl_down_sync(0xffffffffu, x, off);
    if (q + off < NP) x += o;
  }
  return __shfl_sync(0xffffffffu, x, base_lane);
}
template <int N1>
__device__ __forceinline__ double seg_min(double x, int q, int base_lane) {
  constexpr int NP = N1 * N1;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    if (off >= NP) continue;
    const double o = __shfl_down_sync(0xffffffffu, x, off);
    if (q + off < NP) x = smin(x, o);
  }
  return __shfl_sync(0xffffffffu, x, base_lane);
}

// shared-memory plan of the node-per-thread kernel (doubles): STAGES groups of
// G = 8 warps x EPW elements in flight, each as 14 node fields of G (N+1)^2
// doubles (+ slack for a one-double shift when the group's first node is at an
// odd index: bulk copies need 16-byte aligned sources) and the group's
// element-face records
template <int N1, bool V = false>
struct NodePlan {
  // warps per CTA (16 / WARPS CTAs per SM): 4 inviscid (N=3 0.853 -> 0.845 ms/stage
  // against 8), 8 viscous (N=2 1.016 vs 1.032 with 4)
  static constexpr int NP = N1 * N1, EPW = 32 / NP, WARPS = V ? 8 : 4, THREADS = 32 * WARPS;
  static constexpr int G = WARPS * EPW, GN = G * NP, GNS = (GN + 3) & ~1;
  // the viscous variant streams the four physical viscous flux pairs too
  enum { F_H, F_HU, F_HV, F_YE, F_XE, F_YX, F_XX, F_B, F_JAC, F_SX, F_SY, F_WH, F_WHU, F_WHV,
         F_FVU, F_GVU, F_FVV, F_GVV };
  static constexpr int kFields = V ? 18 : 14;
  static constexpr int EF = kFields * GNS;     // int4 [G][4] = 2 doubles each
  static constexpr int STAGE = EF + G * 4 * 2;  // doubles per stage
  static constexpr int STAGES = 3;
  static constexpr int BAR = STAGES * STAGE;    // STAGES mbarriers
  static constexpr int GIDX = BAR + STAGES;     // STAGES group ids (ints)
  static constexpr int TOTAL = GIDX + STAGES;
  static constexpr size_t bytes = TOTAL * sizeof(double);
};

// thread 0: stream group g's node fields and face records into stage buffer sb
template <int N1, bool V>
__device__ __forceinline__ void node_issue(double* sb, uint64_t* bar, const Mesh& M,
                                           const StageArgs& A, int g, bool comb) {
  using P = NodePlan<N1, V>;
  const int e0 = M.e_lo + g * P::G, ne = min(P::G, M.n_owned - e0);
  const long long n0 = (long long)e0 * P::NP;
  const int shift = (int)(n0 & 1);
  const uint32_t fb = round16((size_t)(ne * P::NP + shift) * sizeof(double));
  const uint32_t eb = (uint32_t)(ne * 4 * sizeof(int4));
  const int nf = (comb ? 14 : P::F_WH) + (V ? 4 : 0);
  mbar_expect_tx(bar, nf * fb + eb);
  const double* src[18] = {A.in.h, A.in.hu, A.in.hv, M.ye, M.xe, M.yx, M.xx,
                           M.b, M.jac, M.sx, M.sy, A.wn.h, A.wn.hu, A.wn.hv,
                           A.fvu, A.gvu, A.fvv, A.gvv};
#pragma unroll
  for (int f = 0; f < P::kFields; ++f)
    if (f >= P::F_FVU || comb || f < P::F_WH) bulk_g2s(sb + f * P::GNS, src[f] + n0 - shift, fb, bar);
  bulk_g2s(sb + P::EF, M.ef + (long long)e0 * 4, eb, bar);
}

template <int N1, bool FORCE, bool VISC>
__global__ void __launch_bounds__(NodePlan<N1, VISC>::THREADS, 16 / NodePlan<N1, VISC>::WARPS) k_stage_node(Mesh M, Phys Ph, StageArgs A, Flags* F) {
  using P = NodePlan<N1, VISC>;
  constexpr int NP = N1 * N1, EPW = P::EPW;
  extern __shared__ __align__(16) double sm[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + P::BAR);
  int* gidx = reinterpret_cast<int*>(sm + P::GIDX);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int le = lane / NP, q = lane - le * NP, i = q / N1, j = q - i * N1;
  const int base_lane = le * NP;
  const bool lane_ok = le < EPW;
  // this lane's D~ rows, rotated: slot k holds column (i + k) mod (N+1) (xi
  // line) and (j + k) mod (N+1) (eta line).  The pair sums accumulate D~ F and
  // are scaled by 1/4, 1/8 afterwards: power-of-two scaling commutes with
  // rounding, so this is bitwise (D~/4) F summed.
  double dx[N1], de[N1];
#pragma unroll
  for (int k = 0; k < N1; ++k) {
    dx[k] = __ldg(M.Dt + i * N1 + (i + k) % N1);
    de[k] = __ldg(M.Dt + j * N1 + (j + k) % N1);
  }
  // viscous: the plain D rows, same rotation (strong divergence, viscosity.hpp:195-223)
  double vx[VISC ? N1 : 1], ve[VISC ? N1 : 1];
  if constexpr (VISC) {
#pragma unroll
    for (int k = 0; k < N1; ++k) {
      vx[k] = __ldg(M.D + i * N1 + (i + k) % N1);
      ve[k] = __ldg(M.D + j * N1 + (j + k) % N1);
    }
  }
  const double wij = __ldg(M.w + i) * __ldg(M.w + j);
  const double g = Ph.g, h_des = Ph.h_des, inv2g = 1.0 / (2.0 * g), iw0 = 1.0 / M.w0;
  const double g2 = 2.0 * g;
  const bool comb = A.stage > 0 && A.update;
  int fid0 = -1, fid1 = -1;  // smallest and second-smallest face id touching the node
#pragma unroll
  for (int f = 3; f >= 0; --f) {
    const bool on = f == 0 ? j == 0 : f == 1 ? i == N1 - 1 : f == 2 ? j == N1 - 1 : i == 0;
    if (on && lane_ok) {
      fid1 = fid0;
      fid0 = f;
    }
  }
  const int ngroups = (M.n_owned - M.e_lo + P::G - 1) / P::G;
  if (threadIdx.x == 0) {
    for (int s = 0; s < P::STAGES; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
    int grp = blockIdx.x;
    for (int s = 0; s < P::STAGES; ++s) {
      gidx[s] = grp < ngroups ? grp : -1;
      if (grp < ngroups) node_issue<N1, VISC>(sm + s * P::STAGE, &bars[s], M, A, grp, comb);
      if (s + 1 < P::STAGES) grp = grp < ngroups ? next_group(A.gctr, grp) : ngroups;
    }
  }
  __syncthreads();
  unsigned long long kmin = ~0ull;
  int nlim = 0;
  for (int it = 0;; ++it) {
    // gidx[s] was written by thread 0 before the barrier that ended iteration
    // it - STAGES + 1 (or before the prologue barrier)
    const int s = it % P::STAGES;
    const int grp = gidx[s];
    if (grp < 0) break;  // CTA-uniform
    mbar_wait(&bars[s], (it / P::STAGES) & 1);
    const double* sb = sm + s * P::STAGE;
    const int e0 = M.e_lo + grp * P::G;
    const int shift = (int)(((long long)e0 * NP) & 1);
    const int el = warp * EPW + le;  // element within the group
    const int e = e0 + el;
    const bool active = lane_ok && e < M.n_owned;
    const int ln = (lane_ok ? el * NP + q : 0) + shift;
    const long long n = (long long)e * NP + q;
    double h = sb[P::F_H * P::GNS + ln], hu = sb[P::F_HU * P::GNS + ln],
           hv = sb[P::F_HV * P::GNS + ln];
    const double ye = sb[P::F_YE * P::GNS + ln], xe = sb[P::F_XE * P::GNS + ln],
                 yx = sb[P::F_YX * P::GNS + ln], xx = sb[P::F_XX * P::GNS + ln];
    const double bo = sb[P::F_B * P::GNS + ln];
    double u, v;
    vel(h, hu, hv, h_des, u, v);
    double r0 = 0.0, r1 = 0.0, r2 = 0.0;
    // volume: xi line (b, j), metrics (y_eta, x_eta); eta line (i, b), -(y_xi, x_xi)
#pragma unroll
    for (int dir = 0; dir < 2; ++dir) {
      const double Aa = dir == 0 ? ye : -yx, Ba = dir == 0 ? xe : -xx;
#pragma unroll
      for (int k = 0; k < N1; ++k) {
        double hb = h, ub = u, vb = v, hub = hu, hvb = hv, Ab = Aa, Bb = Ba;
        if (k > 0) {
          const int src = dir == 0 ? base_lane + ((i + k) % N1) * N1 + j
                                   : base_lane + i * N1 + (j + k) % N1;
          hb = __shfl_sync(0xffffffffu, h, src);
          ub = __shfl_sync(0xffffffffu, u, src);
          vb = __shfl_sync(0xffffffffu, v, src);
          hub = __shfl_sync(0xffffffffu, hu, src);
          hvb = __shfl_sync(0xffffffffu, hv, src);
          Ab = __shfl_sync(0xffffffffu, Aa, src);
          Bb = __shfl_sync(0xffffffffu, Ba, src);
        }
        double F0, T1, T2;
        pair_flux(h, u, v, hu, hv, Aa, Ba, hb, ub, vb, hub, hvb, Ab, Bb, g2, F0, T1, T2);
        const double c = dir == 0 ? dx[k] : de[k];
        r0 += c * F0;
        r1 += c * T1;
        r2 += c * T2;
      }
    }
    r0 *= 0.25;
    r1 *= 0.125;
    r2 *= 0.125;
    double fvo[4] = {0.0, 0.0, 0.0, 0.0};  // own physical viscous flux pairs
    if constexpr (VISC) {
      // strong divergence of the contravariant viscous fluxes along both lines
      // (viscous_lhs viscosity.hpp:195-223): xi lines (y_eta, x_eta), eta lines
      // -(y_xi, x_xi), the same metrics as the volume pairs
      fvo[0] = sb[P::F_FVU * P::GNS + ln];
      fvo[1] = sb[P::F_GVU * P::GNS + ln];
      fvo[2] = sb[P::F_FVV * P::GNS + ln];
      fvo[3] = sb[P::F_GVV * P::GNS + ln];
#pragma unroll
      for (int dir = 0; dir < 2; ++dir) {
        const double Aa = dir == 0 ? ye : -yx, Ba = dir == 0 ? xe : -xx;
        const double tu = Aa * fvo[0] - Ba * fvo[1], tv = Aa * fvo[2] - Ba * fvo[3];
#pragma unroll
        for (int k = 0; k < N1; ++k) {
          double tub = tu, tvb = tv;
          if (k > 0) {
            const int src = dir == 0 ? base_lane + ((i + k) % N1) * N1 + j
                                     : base_lane + i * N1 + (j + k) % N1;
            tub = __shfl_sync(0xffffffffu, tu, src);
            tvb = __shfl_sync(0xffffffffu, tv, src);
          }
          const double d = dir == 0 ? vx[k] : ve[k];
          r1 -= d * tub;
          r2 -= d * tvb;
        }
      }
    }
    // interface fluxes: slot s is the node's s-th face
    const double co = wave_c(g, h);
    const int4* efs = reinterpret_cast<const int4*>(sb + P::EF);
#pragma unroll
    for (int sl = 0; sl < 2; ++sl) {
      const int face = sl == 0 ? fid0 : fid1;
      if (!active || face < 0) continue;
      const int t = (face == 0 || face == 2) ? i : j;
      const int4 ef = efs[el * 4 + face];
      if (!(ef.y & EF_PRESENT)) continue;
      const int nf = ef.y & EF_NBR_FACE_MASK;
      const bool minus = ef.y & EF_MINUS, wall = minus && (ef.y & EF_WALL);
      const bool ew = face == 1 || face == 3;
      double hn = h, hun = hu, hvn = hv, bn = bo, m0, m1;
      double fvn[4] = {0.0, 0.0, 0.0, 0.0};  // neighbour's viscous flux pairs
      long long nb = 0;
      if (!wall) {
        const int tp = (ef.y & EF_REVERSED) ? N1 - 1 - t : t;
        nb = (long long)ef.x * NP + face_node(N1, nf, tp);
        hn = __ldg(A.in.h + nb);
        hun = __ldg(A.in.hu + nb);
        hvn = __ldg(A.in.hv + nb);
        bn = __ldg(M.b + nb);
        if constexpr (VISC) {
          fvn[0] = __ldg(A.fvu + nb);
          fvn[1] = __ldg(A.gvu + nb);
          fvn[2] = __ldg(A.fvv + nb);
          fvn[3] = __ldg(A.gvv + nb);
        }
      }
      if (minus) {
        m0 = ew ? ye : yx;
        m1 = ew ? xe : xx;
      } else {
        const bool new_ = nf == 1 || nf == 3;
        m0 = __ldg((new_ ? M.ye : M.yx) + nb);
        m1 = __ldg((new_ ? M.xe : M.xx) + nb);
      }
      double nx, ny, js;
      face_normal(minus ? face : nf, m0, m1, nx, ny, js);
      if (wall) {  // exterior_state (mesh.hpp:382-386)
        const double mn = hu * nx + hv * ny;
        hun = hu - 2.0 * mn * nx;
        hvn = hv - 2.0 * mn * ny;
      }
      double un, vn;
      vel(hn, hun, hvn, h_des, un, vn);
      const double cn = wave_c(g, hn);
      double f0, f1, f2;
      if (minus)
        es_flux_pre(h, u, v, co, hn, un, vn, cn, bo, bn, nx, ny, g, inv2g, f0, f1, f2);
      else
        es_flux_pre(hn, un, vn, cn, h, u, v, co, bn, bo, nx, ny, g, inv2g, f0, f1, f2);
      if constexpr (VISC) {
        // viscous interface penalty (viscosity.hpp:224-246): with the minus-side
        // normal, (phi+ - phi-)/2 lands on both sides; walls take 0 - phi-
        const double pu_o = nx * fvo[0] + ny * fvo[1], pv_o = nx * fvo[2] + ny * fvo[3];
        double du, dv;
        if (wall) {
          du = -pu_o;
          dv = -pv_o;
        } else {
          const double pu_n = nx * fvn[0] + ny * fvn[1], pv_n = nx * fvn[2] + ny * fvn[3];
          const double sg = minus ? 1.0 : -1.0;  // (plus - minus)
          du = 0.5 * sg * (pu_n - pu_o);
          dv = 0.5 * sg * (pv_n - pv_o);
        }
        // folded into the flux: c = sgn js / w0
        f1 -= minus ? du : -du;
        f2 -= minus ? dv : -dv;
      }
      const double c = (minus ? 1.0 : -1.0) * js * iw0;
      r0 += c * f0;
      r1 += c * f1;
      r2 += c * f2;
    }
    // node update (assemble_rhs tail, axpy, SSPRK3 combination)
    const double jac = sb[P::F_JAC * P::GNS + ln];
    {
      const double ij = -frcp(jac), hg2 = 0.5 * g * h;
      double rh = r0 * ij;
      double rhu = (r1 + hg2 * sb[P::F_SX * P::GNS + ln]) * ij;
      double rhv = (r2 + hg2 * sb[P::F_SY * P::GNS + ln]) * ij;
      if (FORCE && active) {
        rh += A.fh[n];
        rhu += A.fhu[n];
        rhv += A.fhv[n];
      }
      if (A.rhs.h && active) {
        A.rhs.h[n] = rh;
        A.rhs.hu[n] = rhu;
        A.rhs.hv[n] = rhv;
      }
      h = h + A.dt * rh;
      hu = hu + A.dt * rhu;
      hv = hv + A.dt * rhv;
      if (comb) {
        h = A.ca * sb[P::F_WH * P::GNS + ln] + A.cb * h;
        hu = A.ca * sb[P::F_WHU * P::GNS + ln] + A.cb * hu;
        hv = A.ca * sb[P::F_WHV * P::GNS + ln] + A.cb * hv;
      }
    }
    if (A.update) {  // kernel-uniform
      // element mean and minimum (limiter.hpp:24-37, 43-84)
      const double wq = wij * jac;
      const double area = seg_sum<N1>(wq, q, base_lane);
      const double a0 = seg_sum<N1>(wq * h, q, base_lane);
      const double a1 = seg_sum<N1>(wq * hu, q, base_lane);
      const double a2 = seg_sum<N1>(wq * hv, q, base_lane);
      const double mmin = seg_min<N1>(h, q, base_lane);
      bool lim = active;
      const double inv = frcp(area);
      const double avg0 = inv * a0, avg1 = inv * a1, avg2 = inv * a2;
      if (lim && avg0 < 0.0) {
        if (q == 0) {
          atomicExch(&F->reject, 1);
          if (!Ph.limiter) atomicExch(&F->abort, 1);
        }
        lim = false;
      }
      double theta = 1.0;
      if (lim && Ph.limiter && mmin < 0.0) {
        const double denom = avg0 - mmin;
        theta = denom < 1e-14 ? 1.0 : smin(1.0, avg0 / denom);
      }
      if (lim && !Ph.limiter && mmin < 0.0 && q == 0) atomicExch(&F->abort, 1);
      if (lim) {
        if (theta < 1.0) {
          h = smax(theta * (h - avg0) + avg0, 0.0);
          hu = theta * (hu - avg1) + avg1;
          hv = theta * (hv - avg2) + avg2;
          nlim += q == 0;
        }
        if (Ph.limiter && h < Ph.h_tol) {
          hu = 0.0;
          hv = 0.0;
        }
        A.out.h[n] = h;
        A.out.hu[n] = hu;
        A.out.hv[n] = hv;
        const unsigned long long key = order_key(h);
        kmin = key < kmin ? key : kmin;
      }
    }
    // stage s consumed by every warp: thread 0 refills it.  (A barrier-free
    // refill by the last warp to finish, handing the group id over through an
    // atomic counter, measured 0.863 vs 0.853 ms/stage at N+1 = 4 and is opaque
    // to compute-sanitizer racecheck.)
    __syncthreads();
    if (threadIdx.x == 0) {
      const int nx_ = next_group(A.gctr, grp);
      gidx[s] = nx_ < ngroups ? nx_ : -1;
      if (nx_ < ngroups) {
        fence_proxy_async();
        node_issue<N1, VISC>(sm + s * P::STAGE, &bars[s], M, A, nx_, comb);
      }
    }
  }
  // one atomic per block for the min height, per warp (rare) for the count
  const unsigned long long bmin = block_min_key(kmin);
  if (threadIdx.x == 0 && bmin != ~0ull) atomicMin(&F->min_h_key, bmin);
  const int wl = __reduce_add_sync(0xffffffffu, nlim);
  if (lane == 0 && wl) atomicAdd(&F->n_limited, wl);
}

template <int N1, bool FORCE, bool VISC>
static void launch_node(const Mesh& M, const Phys& P, const StageArgs& A, Flags* F,
                        cudaStream_t st) {
  using PL = NodePlan<N1, VISC>;
  static int cache[kMaxDevices] = {};
  auto kern = k_stage_node<N1, FORCE, VISC>;
  const int groups = (M.n_owned - M.e_lo + PL::G - 1) / PL::G;
  const int grid = grid_for(kern, PL::THREADS, PL::bytes, groups, cache, A.reserve_sms);
  if (grid > 0) kern<<<grid, PL::THREADS, PL::bytes, st>>>(M, P, A, F);
}

#include "visc_lines.cuh"

// geometry-only split-source coefficients (dg_rhs.hpp:159-176), one thread per node
__global__ void k_source_geometry(Mesh M, double* sx, double* sy) {
  const long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (n >= (long long)M.K * M.np) return;
  const int n1 = M.n1, np = M.np;
  const int loc = (int)(n % np), i = loc / n1, j = loc % n1;
  const long long base = n - loc;
  double db_xi = 0.0, db_eta = 0.0, dye = 0.0, dyx = 0.0, dxe = 0.0, dxx = 0.0;
  for (int m = 0; m < n1; ++m) {
    const double di = M.D[i * n1 + m], dj = M.D[j * n1 + m];
    const long long qx = base + m * n1 + j, qe = base + i * n1 + m;
    db_xi += di * M.b[qx];
    db_eta += dj * M.b[qe];
    dye += di * (M.ye[qx] * M.b[qx]);
    dxe += di * (M.xe[qx] * M.b[qx]);
    dyx += dj * (M.yx[qe] * M.b[qe]);
    dxx += dj * (M.xx[qe] * M.b[qe]);
  }
  sx[n] = M.ye[n] * db_xi + dye - M.yx[n] * db_eta - dyx;
  sy[n] = M.xx[n] * db_eta + dxx - M.xe[n] * db_xi - dxe;
}

}  // namespace

int SWDG_EXPORT(launch_source_geometry)(const Mesh& M, double* sx, double* sy, cudaStream_t st) {
  const long long nn = (long long)M.K * M.np;
  k_source_geometry<<<(unsigned)((nn + 255) / 256), 256, 0, st>>>(M, sx, sy);
  return 1;
}

// ---------------------------------------------------------------------------
// the operator tables live in __constant__ memory, one copy per device: the
// upload is tracked per device; the host image pins what every device holds
static bool g_ops_set[kMaxDevices][17];
static bool g_ops_known[17];
static double g_ops_host[kOpsTotal];

int SWDG_EXPORT(upload_fast_ops)(int n1, const double* D, const double* Dt, const double* Dh,
                    const double* Vinv, const double* w) {
  const int base = ops_offset(n1), np = n1 * n1;
  double tab[5 * 256 + 16];
  for (int k = 0; k < np; ++k) {
    tab[k] = D[k];
    tab[np + k] = 0.25 * Dt[k];
    tab[2 * np + k] = 0.125 * Dt[k];
    tab[3 * np + k] = Dh[k];
    tab[4 * np + k] = Vinv[k];
  }
  for (int k = 0; k < n1; ++k) tab[5 * np + k] = w[k];
  const int len = 5 * np + n1;
  if (g_ops_known[n1] && std::memcmp(tab, g_ops_host + base, len * sizeof(double)) != 0)
    return -1;
  const int dev = current_device();
  if (dev < 0) return -2;
  if (g_ops_set[dev][n1]) return 0;
  if (upload_ops_local(base, tab, len) != 0) return -2;
  std::memcpy(g_ops_host + base, tab, len * sizeof(double));
  g_ops_known[n1] = true;
  g_ops_set[dev][n1] = true;
  return 0;
}


// half-line kernel (N+1 >= 5 inviscid, N+1 >= 4 viscous)
template <int N1, bool FORCE, bool VISC>
static void launch_half(const Mesh& M, const Phys& P, const StageArgs& A, Flags* F,
                        cudaStream_t st) {
  using PL = HL<N1, VISC>;
  static int cache[kMaxDevices] = {};
  auto kern = k_stage_hl<N1, FORCE, VISC>;
  const int grid = grid_for(kern, PL::THREADS, PL::bytes, (M.n_owned - M.e_lo + PL::E - 1) / PL::E,
                            cache, A.reserve_sms);
  kern<<<grid, PL::THREADS, PL::bytes, st>>>(M, P, A, F);
}

// Kernel choice per degree, measured on B200 (1M elements, profiles/r01_sweep_variants.txt,
// r01_node_variants.txt): inviscid element-per-thread at N+1 <= 3 (0.185 / 0.483 vs node
// 0.197 / 0.552 ms/stage), node-per-thread at N+1 = 4 (0.853 vs full-line 0.926 vs
// half-line 1.65), half-line above; viscous node-per-thread at N+1 = 3 (1.013 vs 1.224),
// half-line above (N+1 = 4: 1.585 vs node 1.798).
template <int N1>
static void launch_n(const Mesh& M, const Phys& P, const StageArgs& A, Flags* F,
                     cudaStream_t st) {
  if constexpr (N1 >= 3) {
    if (A.fvu) {
      if constexpr (N1 <= SWDG_VISC_NODE_MAX) {
        if (A.fh) launch_node<N1, true, true>(M, P, A, F, st);
        else launch_node<N1, false, true>(M, P, A, F, st);
      } else {
        if (A.fh) launch_half<N1, true, true>(M, P, A, F, st);
        else launch_half<N1, false, true>(M, P, A, F, st);
      }
      return;
    }
  }
  if constexpr (N1 <= 3) {
    if (A.fh) launch_elem<N1, true>(M, P, A, F, st);
    else launch_elem<N1, false>(M, P, A, F, st);
  } else if constexpr (N1 == 4) {
    if (A.fh) launch_node<N1, true, false>(M, P, A, F, st);
    else launch_node<N1, false, false>(M, P, A, F, st);
  } else {
    if (A.fh) launch_half<N1, true, false>(M, P, A, F, st);
    else launch_half<N1, false, false>(M, P, A, F, st);
  }
}

int SWDG_EXPORT(launch_fast_visc_pre)(const Mesh& M, const Phys& P, CState S, double* eps,
                                      double* fvu, double* fvv, double* gvu, double* gvv,
                                      Flags* F, cudaStream_t st) {
  // line-based pre-kernel at every degree (one velocity component at a time:
  // ~5 (N+1) doubles per thread); measured faster than a node-per-thread kernel
  // at every N once the eps maximum went to one atomic per CTA (N=14: 50.4 -> 35.9
  // ms/stage)
  switch (M.n1) {
#define SWDG_VL(n)                                                                \
  case n:                                                                         \
    if constexpr (n >= SWDG_N1_LO && n <= SWDG_N1_HI)                             \
      launch_visc_lines_n<n>(M, P, S, eps, fvu, fvv, gvu, gvv, F, st);            \
    else                                                                          \
      return 0;                                                                   \
    break;
    SWDG_VL(3) SWDG_VL(4) SWDG_VL(5) SWDG_VL(6) SWDG_VL(7) SWDG_VL(8) SWDG_VL(9) SWDG_VL(10)
    SWDG_VL(11) SWDG_VL(12) SWDG_VL(13) SWDG_VL(14) SWDG_VL(15) SWDG_VL(16)
#undef SWDG_VL
    default: return 0;
  }
  return 1;
}

int SWDG_EXPORT(launch_fast_stage)(const Mesh& M, const Phys& P, const StageArgs& A, Flags* F,
                                   cudaStream_t st) {
  switch (M.n1) {
#define SWDG_ST(n)                                                                \
  case n:                                                                         \
    if constexpr (n >= SWDG_N1_LO && n <= SWDG_N1_HI)                             \
      launch_n<n>(M, P, A, F, st);                                                \
    else                                                                          \
      return 0;                                                                   \
    break;
    SWDG_ST(2) SWDG_ST(3) SWDG_ST(4) SWDG_ST(5) SWDG_ST(6) SWDG_ST(7) SWDG_ST(8) SWDG_ST(9)
    SWDG_ST(10) SWDG_ST(11) SWDG_ST(12) SWDG_ST(13) SWDG_ST(14) SWDG_ST(15) SWDG_ST(16)
#undef SWDG_ST
    default: return 0;
  }
  return 1;
}

}  // namespace swdg_dev
