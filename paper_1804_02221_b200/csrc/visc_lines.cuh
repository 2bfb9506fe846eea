// visc_lines.cuh — line-based viscous pre-kernel (fast mode), included inside
// kernels_fast.cu's anonymous namespace (uses Ops<>, vel, smin/smax).
//
// Per element: the modal shock indicator and viscosity coefficient
// (shock_indicator / viscosity_coefficient, viscosity.hpp:35-78), the BR1
// lifted velocity gradients (br1_gradients, viscosity.hpp:95-168) and the
// physical viscous flux pairs h eps grad (viscous_lhs, viscosity.hpp:187-194),
// written per node for the stage kernel.
//
// The node-per-thread version reads 2(N+1) neighbours x 4 fields from shared
// memory for every node (shared-memory bandwidth bound: 2.9 ms at N=7, 1M
// elements).  Here a thread owns a line: xi-line threads (column j) apply the
// 1D operators along i with the line in registers and constant-bank
// coefficients, eta-line threads (row i) along j, so each node's data is read
// from shared memory once per direction:
//   xi:  tmp = V^-1 h (first modal pass), the xi terms of the BR1 sums
//        (D-hat of y_eta u, x_eta u, y_eta v, x_eta v) and the E/W face
//        corrections at the line's endpoints;
//   eta: the eta terms (D-hat of y_xi u, ...), the S/N face corrections, and —
//        after the barrier — the second modal pass along j and the row's shell
//        energies (segmented warp-shuffle reduction per element).
// Both directions leave their four partials per node in shared memory; the
// final phase is one thread per node (balanced, coalesced stores).
#pragma once

template <int N1>
struct VLP {
  static constexpr int NP = N1 * N1, N = N1 - 1;
// elements per CTA: two warps per CTA (more independent CTAs per SM hide the
// staging latency better: viscous N=7 6.54 -> 6.35 ms/stage against 128 threads)
#ifndef VL_THREADS
#define VL_THREADS 64
#endif
  static constexpr int E = (VL_THREADS / (2 * N1)) > 1 ? VL_THREADS / (2 * N1) : 1;
  static constexpr int LPD = E * N1;                 // lines per direction
  static constexpr int LS = (LPD + 31) / 32 * 32;     // lane slots per direction
  static constexpr int THREADS = 2 * LS;
  static constexpr int PAD = N1 | 1, EPAD = N1 * PAD, GPAD = E * EPAD;
  static constexpr int PMAX = (LPD + 31) / 32 + 1;
  // shared fields [E][N1][PAD]: state, the first modal pass, and the four BR1
  // partials of each direction.  The metrics are read from global memory by the
  // line threads (each is used by one direction only): 12 instead of 16 fields
  // per node, so more CTAs share an SM
  enum { H, U, V, TMP, XU1, XU2, XV1, XV2, EU1, EU2, EV1, EV2, kF };
  // asynchronous (LDGSTS) staging of the state from N+1 = 4 on (measured with the
  // metrics out of shared memory: viscous N=3..6 1-4% faster than synchronous
  // staging, neutral at 7, 8, profiles/r02_ab_visc_pre_staging.txt; with the
  // metrics staged too it had measured slower at N+1 <= 8); N+1 = 3 stages
  // synchronously with every node's loads issued first (N=2 0.957 -> 0.931)
#ifndef VL_PREFETCH_AHEAD
#define VL_PREFETCH_AHEAD 592  // measured (profiles/r02_ab_visc_pre_prefetch.txt): viscous N=7 5.88 -> 5.66, N=12 20.5 -> 19.6 ms/stage
#endif
#ifndef VL_SYNC_BATCH
#define VL_SYNC_BATCH 1
#endif
#ifndef VL_ASYNC_MIN
#define VL_ASYNC_MIN 4
#endif
  static constexpr bool kAsync = N1 >= VL_ASYNC_MIN;
  static constexpr int RED = kF * GPAD;             // [E][PMAX][4] shell-energy pieces
  static constexpr int EPS = RED + E * PMAX * 4;
  static constexpr int TOTAL = EPS + E;
  static constexpr size_t bytes = TOTAL * sizeof(double);
};

template <int N1>
__global__ void __launch_bounds__(VLP<N1>::THREADS)
    k_visc_lines(Mesh M, Phys Ph, CState S, double* eps_out, double* fvu, double* fvv,
                 double* gvu, double* gvv, Flags* F) {
  using P = VLP<N1>;
  using O = Ops<N1>;
  constexpr int NP = P::NP, N = P::N, PAD = P::PAD, GP = P::GPAD, LPD = P::LPD;
  extern __shared__ __align__(16) double sm[];
  const int tid = threadIdx.x, lane = tid & 31;
  const bool xi = tid < P::LS;
  const int ls = xi ? tid : tid - P::LS;  // line slot within the direction
  const bool line_ok = ls < LPD;
  const int el = line_ok ? ls / N1 : 0, li = line_ok ? ls - (ls / N1) * N1 : 0;
  const int e0 = M.e_lo + blockIdx.x * P::E, ne = min(P::E, M.n_owned - e0);
  const bool active = line_ok && el < ne;
  const int e = e0 + el;
  const double h_des = Ph.h_des, iw0 = 1.0 / M.w0;

  const long long base = (long long)e0 * NP;
  // L2 prefetch of the state, metrics and J of the CTA that is dispatched about
  // one CTA lifetime later (blockIdx + VL_PREFETCH_AHEAD): its loads then hit L2
  if constexpr (VL_PREFETCH_AHEAD > 0) {
    if (tid == 0 && blockIdx.x + VL_PREFETCH_AHEAD < gridDim.x) {
      const long long pb = base + (long long)VL_PREFETCH_AHEAD * P::E * NP;
      const long long lim = (long long)M.n_owned * NP;
      const long long lo = pb & ~1ll;  // 16-byte aligned start
      long long hi = pb + (long long)P::E * NP;
      if (hi > lim) hi = lim;
      if (hi > lo) {
        const uint32_t bytes = (uint32_t)(((hi - lo) * 8) & ~15ll);
        if (bytes) {
          const double* f[8] = {S.h, S.hu, S.hv, M.ye, M.xe, M.yx, M.xx, M.jac};
#pragma unroll
          for (int q = 0; q < 8; ++q) bulk_prefetch_l2(f[q] + lo, bytes);
        }
      }
    }
  }
  // this thread's nodes of the final (flux-pair) phase: J prefetched now
  constexpr int R = (P::E * NP + P::THREADS - 1) / P::THREADS;
  double jr[R];
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const int r = tid + k * P::THREADS;
    jr[k] = r < ne * NP ? __ldg(M.jac + base + r) : 1.0;
  }
  if constexpr (P::kAsync) {
    // the group's state and metrics go to shared memory by asynchronous 8-byte
    // copies (LDGSTS), in flight together with the connectivity and neighbour
    // gathers below (hu, hv land in the x-partial slots, free until the line
    // phase)
    for (int r = tid; r < ne * NP; r += P::THREADS) {
      const int el2 = r / NP, q = r - el2 * NP, i = q / N1, j = q - i * N1;
      double* d = sm + el2 * P::EPAD + i * PAD + j;
      const long long n = base + r;
      cp_async8(d + P::H * GP, S.h + n);
      cp_async8(d + P::XU1 * GP, S.hu + n);
      cp_async8(d + P::XU2 * GP, S.hv + n);
    }
    cp_async_commit();
  }
  // neighbour traces at this line's two endpoints
  int fy[2] = {0, 0};
  double nh[2] = {0.0, 0.0}, nhu[2] = {0.0, 0.0}, nhv[2] = {0.0, 0.0};
  if (active) {
#pragma unroll
    for (int end = 0; end < 2; ++end) {
      const int face = xi ? (end ? 1 : 3) : (end ? 2 : 0);
      const int4 ef = M.ef[e * 4 + face];
      fy[end] = ef.y;
      if ((ef.y & EF_PRESENT) && !(ef.y & EF_WALL)) {
        const int nf = ef.y & EF_NBR_FACE_MASK;
        const int tp = (ef.y & EF_REVERSED) ? N - li : li;
        const long long nb = (long long)ef.x * NP + face_node(N1, nf, tp);
        nh[end] = __ldg(S.h + nb);
        nhu[end] = __ldg(S.hu + nb);
        nhv[end] = __ldg(S.hv + nb);
      }
    }
  }
  // this line's metrics, straight from global memory (in flight with the staging):
  // node k of the line is (k, li) on xi lines, (li, k) on eta lines
  double A[N1], B[N1];
  {
    const double* ga = xi ? M.ye : M.yx;
    const double* gb = xi ? M.xe : M.xx;
    const long long g0 = (long long)(active ? e : e0) * NP + (xi ? li : li * N1);
    const int gs = xi ? N1 : 1;
#pragma unroll
    for (int k = 0; k < N1; ++k) {
      A[k] = __ldg(ga + g0 + k * gs);
      B[k] = __ldg(gb + g0 + k * gs);
    }
  }
  if constexpr (P::kAsync) {
    // velocities of the staged state (each thread reads the words its own copies
    // wrote: no barrier needed before this pass)
    cp_async_wait_all();
    for (int r = tid; r < ne * NP; r += P::THREADS) {
      const int el2 = r / NP, q = r - el2 * NP, i = q / N1, j = q - i * N1;
      double* d = sm + el2 * P::EPAD + i * PAD + j;
      double u, v;
      vel(d[P::H * GP], d[P::XU1 * GP], d[P::XU2 * GP], h_des, u, v);
      d[P::U * GP] = u;
      d[P::V * GP] = v;
    }
  } else if constexpr (VL_SYNC_BATCH) {
    // stage the group's state (+ velocities), one thread per node: every node's
    // loads issued before the first velocity (one memory round trip per CTA)
    double th[R], thu[R], thv[R];
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const int r = tid + k * P::THREADS;
      const long long n = base + (r < ne * NP ? r : 0);
      th[k] = __ldg(S.h + n);
      thu[k] = __ldg(S.hu + n);
      thv[k] = __ldg(S.hv + n);
    }
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const int r = tid + k * P::THREADS;
      if (r >= ne * NP) break;
      const int el2 = r / NP, q = r - el2 * NP, i = q / N1, j = q - i * N1;
      double* d = sm + el2 * P::EPAD + i * PAD + j;
      double u, v;
      vel(th[k], thu[k], thv[k], h_des, u, v);
      d[P::H * GP] = th[k];
      d[P::U * GP] = u;
      d[P::V * GP] = v;
    }
  } else {
    // stage the group's state (+ velocities), one thread per node
    for (int r = tid; r < ne * NP; r += P::THREADS) {
      const int el2 = r / NP, q = r - el2 * NP, i = q / N1, j = q - i * N1;
      double* d = sm + el2 * P::EPAD + i * PAD + j;
      const long long n = base + r;
      const double h = S.h[n], hu = S.hu[n], hv = S.hv[n];
      double u, v;
      vel(h, hu, hv, h_des, u, v);
      d[P::H * GP] = h;
      d[P::U * GP] = u;
      d[P::V * GP] = v;
    }
  }
  __syncthreads();

  // ---- line phase: node k of this line at off0 + k*st
  const int off0 = el * P::EPAD + (xi ? li : li * PAD), st = xi ? PAD : 1;
  if (active) {
    if (xi) {  // first modal pass along i: tmp(a, j) = sum_k Vinv(a, k) h(k, j)
      double hh[N1];
#pragma unroll
      for (int k = 0; k < N1; ++k) hh[k] = sm[P::H * GP + off0 + k * st];
#pragma unroll
      for (int a = 0; a < N1; ++a) {
        double t = 0.0;
#pragma unroll
        for (int k = 0; k < N1; ++k) t += O::Vinv(a, k) * hh[k];
        sm[P::TMP * GP + off0 + a * st] = t;
      }
    }
    // neighbour velocities at the endpoints (interface U* = <u>, walls u-)
    double nu[2] = {0.0, 0.0}, nv[2] = {0.0, 0.0};
#pragma unroll
    for (int end = 0; end < 2; ++end)
      if ((fy[end] & EF_PRESENT) && !(fy[end] & EF_WALL))
        vel(nh[end], nhu[end], nhv[end], h_des, nu[end], nv[end]);
    // BR1 weak D-hat sums along the line (viscosity.hpp:114-126), one velocity
    // component at a time (register footprint ~5 (N+1) doubles): xi lines give
    // +Dh(y_eta w), -Dh(x_eta w); eta lines -Dh(y_xi w), +Dh(x_xi w); then the
    // interface corrections at the endpoints (viscosity.hpp:127-160), face
    // metrics W: -(y_eta, x_eta), E: +(y_eta, x_eta), S: +(y_xi, x_xi), N: -(y_xi, x_xi)
    const double sg = xi ? 1.0 : -1.0;
    const int f0 = xi ? P::XU1 : P::EU1;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      double w[N1], Aw[N1], Bw[N1];
#pragma unroll
      for (int m = 0; m < N1; ++m) {
        w[m] = sm[(c ? P::V : P::U) * GP + off0 + m * st];
        Aw[m] = A[m] * w[m];
        Bw[m] = B[m] * w[m];
      }
      double* o1 = sm + (f0 + 2 * c) * GP + off0;      // u1 / v1 partial
      double* o2 = sm + (f0 + 2 * c + 1) * GP + off0;  // u2 / v2 partial
#pragma unroll
      for (int a = 0; a < N1; ++a) {
        double s1 = 0.0, s2 = 0.0;
#pragma unroll
        for (int m = 0; m < N1; ++m) {
          const double d = O::Dh(a, m);
          s1 += d * Aw[m];
          s2 += d * Bw[m];
        }
        double p1 = sg * s1, p2 = -sg * s2;
        if (a == 0 || a == N) {
          const int end = a == N ? 1 : 0;
          if (fy[end] & EF_PRESENT) {
            const double nb = c ? nv[end] : nu[end];
            const double ws = (fy[end] & EF_WALL) ? w[a] : 0.5 * (w[a] + nb);
            const double s = (xi == (end == 1)) ? 1.0 : -1.0;
            p1 += (s * A[a] * iw0) * ws;
            p2 -= (s * B[a] * iw0) * ws;
          }
        }
        o1[a * st] = p1;
        o2[a * st] = p2;
      }
    }
  }
  __syncthreads();  // first modal pass and both directions' partials published

  // ---- eta lines: second modal pass along j and the row's shell energies
  if (!xi) {
    double c[4] = {0.0, 0.0, 0.0, 0.0};
    if (active) {
      double tr[N1];
      const int i = li;
#pragma unroll
      for (int k = 0; k < N1; ++k) tr[k] = sm[P::TMP * GP + off0 + k];
#pragma unroll
      for (int b = 0; b < N1; ++b) {
        double mo = 0.0;
#pragma unroll
        for (int k = 0; k < N1; ++k) mo += tr[k] * O::Vinv(b, k);
        const double m2 = mo * mo;
        // shells (viscosity.hpp:44-57): all; i,b < N; top (i or b = N); N-1
        c[0] += m2;
        if (i < N && b < N) c[1] += m2;
        if (i == N || b == N) c[2] += m2;
        if ((i == N - 1 && b <= N - 1) || (b == N - 1 && i <= N - 1)) c[3] += m2;
      }
    }
    const int seg = active ? el : -1 - lane;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int seg2 = __shfl_down_sync(0xffffffffu, seg, o);
      double t[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) t[k] = __shfl_down_sync(0xffffffffu, c[k], o);
      if (lane + o < 32 && seg2 == seg) {
#pragma unroll
        for (int k = 0; k < 4; ++k) c[k] += t[k];
      }
    }
    const int w0 = (el * N1) >> 5;  // first warp (of the eta half) of the element
    if (active && (lane == 0 || li == 0)) {
      double* rr = sm + P::RED + (el * P::PMAX + (ls >> 5) - w0) * 4;
#pragma unroll
      for (int k = 0; k < 4; ++k) rr[k] = c[k];
    }
  }
  __syncthreads();
  // ---- eps per element (viscosity_coefficient, viscosity.hpp:60-78)
  if (tid < ne) {
    const int el2 = tid;
    const int w0 = (el2 * N1) >> 5, npc = ((el2 * N1 + N1 - 1) >> 5) - w0 + 1;
    double den1 = 0.0, den2 = 0.0, num1 = 0.0, num2 = 0.0;
    for (int pc = 0; pc < npc; ++pc) {
      const double* rr = sm + P::RED + (el2 * P::PMAX + pc) * 4;
      den1 += rr[0];
      den2 += rr[1];
      num1 += rr[2];
      num2 += rr[3];
    }
    const double floor_abs = 1e-28 * den1 + 1e-300;
    double eps = 0.0;
    if (!(den1 <= 1e-300)) {
      const double r1 = num1 > floor_abs ? num1 / den1 : 0.0;
      const double r2 = (num2 > floor_abs && den2 > floor_abs) ? num2 / den2 : 0.0;
      const double r = smax(r1, r2);
      if (r > 0.0) {
        const double sigma = log10(r);
        if (sigma >= Ph.sigma_max) {
          eps = Ph.epsilon0;
        } else if (!(sigma < Ph.sigma_min)) {
          eps = 0.5 * Ph.epsilon0 *
                (1.0 + sin(M_PI * (sigma - 0.5 * (Ph.sigma_max + Ph.sigma_min)) /
                           (Ph.sigma_max - Ph.sigma_min)));
        }
      }
    }
    sm[P::EPS + el2] = eps;
    eps_out[e0 + el2] = eps;
  }
  // max eps: one atomic per CTA (E <= 32 elements, all in warp 0); one per
  // element put 1M same-address atomics into every launch
  if (tid < 32) {
    unsigned long long k = tid < ne ? order_key(sm[P::EPS + tid]) : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long t = __shfl_xor_sync(0xffffffffu, k, o);
      k = t > k ? t : k;
    }
    if (tid == 0) atomicMax(&F->max_eps_key, k);
  }
  __syncthreads();
  // ---- viscous flux pairs, one thread per node (coalesced)
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const int r = tid + k * P::THREADS;
    if (r >= ne * NP) break;
    const int el2 = r / NP, q = r - el2 * NP, i = q / N1, j = q - i * N1;
    const int pq = el2 * P::EPAD + i * PAD + j;
    const long long n = base + r;
    const double u1 = sm[P::XU1 * GP + pq] + sm[P::EU1 * GP + pq];
    const double u2 = sm[P::XU2 * GP + pq] + sm[P::EU2 * GP + pq];
    const double v1 = sm[P::XV1 * GP + pq] + sm[P::EV1 * GP + pq];
    const double v2 = sm[P::XV2 * GP + pq] + sm[P::EV2 * GP + pq];
    const double he = sm[P::H * GP + pq] * sm[P::EPS + el2] * (1.0 / jr[k]);
    fvu[n] = he * u1;
    fvv[n] = he * v1;
    gvu[n] = he * u2;
    gvv[n] = he * v2;
  }
}

template <int N1>
void launch_visc_lines_n(const Mesh& M, const Phys& P, CState S, double* eps, double* fvu,
                         double* fvv, double* gvu, double* gvv, Flags* F, cudaStream_t st) {
  using PL = VLP<N1>;
  static bool attr[kMaxDevices] = {};
  const int dev = current_device();
  if (dev < 0) return;
  if (!attr[dev]) {
    cudaFuncSetAttribute(k_visc_lines<N1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)PL::bytes);
    attr[dev] = true;
  }
  if (M.n_owned <= M.e_lo) return;
  const int grid = (M.n_owned - M.e_lo + PL::E - 1) / PL::E;
  k_visc_lines<N1><<<grid, PL::THREADS, PL::bytes, st>>>(M, P, S, eps, fvu, fvv, gvu, gvv, F);
}
