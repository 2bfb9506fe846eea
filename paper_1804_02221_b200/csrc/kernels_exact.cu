// kernels_exact.cu — bitwise-parity stage kernels (SWDG_MODE_EXACT), sm_100a FP64.
//
// Compiled with --fmad=false: no FMA contraction and no reassociation, so every
// expression below rounds exactly like the reference built at its Release
// flags.  The kernels replay the reference expression trees and, per node,
// its accumulation order: volume xi-sum then eta-sum into one accumulator,
// then -source, then the surface contributions in global face-list order,
// then -viscous, then *(-1/J) (dg_rhs.hpp:267-303).  The reference scatters
// each face flux once to both sides (dg_rhs.hpp:199-252); here each side
// re-evaluates the same flux from the minus side's data (normal, J_surf,
// trace order), which is bitwise the same number, so no face buffer and no
// atomics are needed.  One thread per node (or per element for the serial
// element reductions); throughput is the job of kernels_fast.cu.
#include <cuda_runtime.h>

#include "swdg_device.cuh"
#include "swdg_launch.h"

namespace swdg_dev {
namespace {

__device__ __forceinline__ double smin(double a, double b) { return (b < a) ? b : a; }
__device__ __forceinline__ double smax(double a, double b) { return (a < b) ? b : a; }

// phys::velocity (physics.hpp:23-36)
__device__ __forceinline__ void velocity(double h, double hu, double hv, double h_des,
                                         double& u, double& v) {
  if (h >= h_des) {
    u = hu / h;
    v = hv / h;
  } else {
    u = 0.0;
    v = 0.0;
  }
}

// fluxes::es_surface_flux_normal (fluxes.hpp:136-166): rotated EC flux minus
// 1/2 R|Lambda|R^T [[q]] (make_dissipation 96-108, apply_dissipation 111-118,
// including the literal products with the 0/1 entries of R), unrotated.
__device__ void es_flux(double hm, double hum, double hvm, double hp, double hup, double hvp,
                        double bm, double bp, double nx, double ny, double g, double h_des,
                        double& f0, double& f1, double& f2) {
  double um, vm, up, vp;
  velocity(hm, hum, hvm, h_des, um, vm);
  velocity(hp, hup, hvp, h_des, up, vp);
  const double unm = nx * um + ny * vm, utm = -ny * um + nx * vm;
  const double unp = nx * up + ny * vp, utp = -ny * up + nx * vp;
  const double havg = 0.5 * (hm + hp);
  const double h2avg = 0.5 * (hm * hm + hp * hp);
  const double uavg = 0.5 * (unm + unp);
  const double vavg = 0.5 * (utm + utp);
  const double cavg = 0.5 * (sqrt(g * smax(hm, 0.0)) + sqrt(g * smax(hp, 0.0)));
  double a0 = havg * uavg;
  double a1 = havg * uavg * uavg + 0.5 * g * h2avg;
  double a2 = havg * uavg * vavg;
  const double x0 = g * ((hp + bp) - (hm + bm)) - 0.5 * (unp * unp - unm * unm) -
                    0.5 * (utp * utp - utm * utm);
  const double x1 = unp - unm, x2 = utp - utm;
  const double r10 = uavg + cavg, r12 = uavg - cavg;
  const double s = 1.0 / (2.0 * g);
  const double l0 = s * fabs(uavg + cavg), l1 = fabs(havg * uavg), l2 = s * fabs(uavg - cavg);
  const double y0 = l0 * (1.0 * x0 + r10 * x1 + vavg * x2);
  const double y1 = l1 * (0.0 * x0 + 0.0 * x1 + 1.0 * x2);
  const double y2 = l2 * (1.0 * x0 + r12 * x1 + vavg * x2);
  const double d0 = 1.0 * y0 + 0.0 * y1 + 1.0 * y2;
  const double d1 = r10 * y0 + 0.0 * y1 + r12 * y2;
  const double d2 = vavg * y0 + 1.0 * y1 + vavg * y2;
  a0 -= 0.5 * d0;
  a1 -= 0.5 * d1;
  a2 -= 0.5 * d2;
  f0 = a0;
  f1 = nx * a1 - ny * a2;
  f2 = ny * a1 + nx * a2;
}

// phys::physical_flux (physics.hpp:39-45)
__device__ __forceinline__ void phys_flux(double h, double hu, double hv, double g,
                                          double h_des, double* fx, double* fy) {
  double u, v;
  velocity(h, hu, hv, h_des, u, v);
  const double pr = 0.5 * g * h * h;
  fx[0] = h * u;
  fx[1] = h * u * u + pr;
  fx[2] = h * u * v;
  fy[0] = h * v;
  fy[1] = h * u * v;
  fy[2] = h * v * v + pr;
}

// fluxes::llf_surface_flux (fluxes.hpp:192-202) with phys::max_wave_speed
// (physics.hpp:101-112): central flux minus (lambda_max / 2) [[w]]
__device__ void llf_flux(double hm, double hum, double hvm, double hp, double hup, double hvp,
                         double nx, double ny, double g, double h_des, double& f0, double& f1,
                         double& f2) {
  double fxm[3], fym[3], fxp[3], fyp[3];
  phys_flux(hm, hum, hvm, g, h_des, fxm, fym);
  phys_flux(hp, hup, hvp, g, h_des, fxp, fyp);
  double um, vm, up, vp;
  velocity(hm, hum, hvm, h_des, um, vm);
  velocity(hp, hup, hvp, h_des, up, vp);
  const double unm = nx * um + ny * vm, unp = nx * up + ny * vp;
  const double cm = sqrt(g * smax(hm, 0.0)), cp = sqrt(g * smax(hp, 0.0));
  const double lmax = smax(fabs(unm) + cm, fabs(unp) + cp);
  const double wm[3] = {hm, hum, hvm}, wp[3] = {hp, hup, hvp};
  double f[3];
  for (int c = 0; c < 3; ++c) {
    f[c] = 0.5 * (nx * fxm[c] + ny * fym[c] + nx * fxp[c] + ny * fyp[c]);
    f[c] -= 0.5 * lmax * (wp[c] - wm[c]);
  }
  f0 = f[0];
  f1 = f[1];
  f2 = f[2];
}

// Face visiting order at a node: up to two faces sorted by global ordinal.
// `minus_first` picks the side order inside one FaceInfo (surface_terms and
// viscous_lhs scatter minus then plus; br1_gradients plus then minus).
struct NodeFaces {
  int n, face[2], t[2];
};

__device__ __forceinline__ NodeFaces sorted_faces(const Mesh& M, int e, int i, int j,
                                                  bool minus_first) {
  NodeFaces nf;
  int fa[2], ta[2];
  const int c = node_faces(M.n1, i, j, fa, ta);
  int k = 0;
  for (int q = 0; q < c; ++q) {
    const int4 ef = M.ef[e * 4 + fa[q]];
    if (!(ef.y & EF_PRESENT)) continue;
    nf.face[k] = fa[q];
    nf.t[k] = ta[q];
    ++k;
  }
  nf.n = k;
  if (k == 2) {
    const int4 e0 = M.ef[e * 4 + nf.face[0]], e1 = M.ef[e * 4 + nf.face[1]];
    // key = ordinal*2 + side rank
    const int r0 = ((e0.y & EF_MINUS) != 0) == minus_first ? 0 : 1;
    const int r1 = ((e1.y & EF_MINUS) != 0) == minus_first ? 0 : 1;
    const long long k0 = 2ll * e0.z + r0, k1 = 2ll * e1.z + r1;
    if (k1 < k0) {
      int tf = nf.face[0], tt = nf.t[0];
      nf.face[0] = nf.face[1];
      nf.t[0] = nf.t[1];
      nf.face[1] = tf;
      nf.t[1] = tt;
    }
  }
  return nf;
}

// Global node index of the neighbour partner of (e, face, t) and the index of
// the minus side's face-array entry.
__device__ __forceinline__ void partner_of(const Mesh& M, int e, int face, int t, int4 ef,
                                           long long& nbr_node, long long& minus_fidx) {
  const int nf = ef.y & EF_NBR_FACE_MASK;
  const int tp = (ef.y & EF_REVERSED) ? M.degree - t : t;
  nbr_node = (long long)ef.x * M.np + face_node(M.n1, nf, tp);
  minus_fidx = (ef.y & EF_MINUS) ? ((long long)e * 4 + face) * M.n1 + t
                                 : ((long long)ef.x * 4 + nf) * M.n1 + tp;
}

// ------------------------------------------------------------------------
// shock_indicator (viscosity.hpp:35-65) up to the log10: writes r = max(r1,r2)
// or -1 for the sentinel.  The host finishes sigma = log10(r) and the ramp
// (viscosity.hpp:69-78) with the same libm as the reference.
__global__ void k_indicator(Mesh M, CState S, double* r_out) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= M.K) return;
  const int n1 = M.n1, N = M.degree;
  const double* f = S.h + (long long)e * M.np;
  double tmp[256];
  for (int i = 0; i < n1; ++i)
    for (int j = 0; j < n1; ++j) {
      double s = 0.0;
      for (int k = 0; k < n1; ++k) s += M.Vinv[i * n1 + k] * f[k * n1 + j];
      tmp[i * n1 + j] = s;
    }
  double den1 = 0.0, den2 = 0.0, num1 = 0.0, num2 = 0.0;
  // modal(i,j) = sum_k tmp(i,k) Vinv(j,k); accumulate the shells in the
  // reference's orders: den1 over all (i,j) row-major, den2 over i,j<N,
  // num1 = m(N,N) + sum_i [m(i,N) + m(N,i)], num2 likewise at N-1.
  auto modal = [&](int i, int j) {
    double s = 0.0;
    for (int k = 0; k < n1; ++k) s += tmp[i * n1 + k] * M.Vinv[j * n1 + k];
    return s * s;
  };
  for (int i = 0; i < n1; ++i)
    for (int j = 0; j < n1; ++j) den1 += modal(i, j);
  for (int i = 0; i < n1 - 1; ++i)
    for (int j = 0; j < n1 - 1; ++j) den2 += modal(i, j);
  num1 = modal(N, N);
  num2 = modal(N - 1, N - 1);
  for (int i = 0; i < N; ++i) num1 += modal(i, N) + modal(N, i);
  for (int i = 0; i < N - 1; ++i) num2 += modal(i, N - 1) + modal(N - 1, i);
  const double floor_abs = 1e-28 * den1 + 1e-300;
  double r = -1.0;
  if (!(den1 <= 1e-300)) {
    const double r1 = num1 > floor_abs ? num1 / den1 : 0.0;
    const double r2 = (num2 > floor_abs && den2 > floor_abs) ? num2 / den2 : 0.0;
    const double rr = smax(r1, r2);
    if (!(rr <= 0.0)) r = rr;
  }
  r_out[e] = r;
}

// ------------------------------------------------------------------------
// BR1 lifted gradients (viscosity.hpp:95-168) and the viscous flux pairs of
// viscous_lhs (viscosity.hpp:187-194), one thread per node.
__global__ void k_grad(Mesh M, Phys P, CState S, const double* eps, double* fvu, double* fvv,
                       double* gvu, double* gvv) {
  const long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (n >= (long long)M.n_owned * M.np) return;
  const int n1 = M.n1, np = M.np;
  const int e = (int)(n / np), loc = (int)(n % np), i = loc / n1, j = loc % n1;
  const long long base = (long long)e * np;
  const double* Dh = M.Dh;
  // volume parts: pu = metric*f, s = sum_m Dhat * pu
  double sye_u = 0.0, syx_u = 0.0, sxe_u = 0.0, sxx_u = 0.0;
  double sye_v = 0.0, syx_v = 0.0, sxe_v = 0.0, sxx_v = 0.0;
  for (int m = 0; m < n1; ++m) {
    const long long qx = base + m * n1 + j, qe = base + i * n1 + m;
    double ux, vx, ue, ve;
    velocity(S.h[qx], S.hu[qx], S.hv[qx], P.h_des, ux, vx);
    velocity(S.h[qe], S.hu[qe], S.hv[qe], P.h_des, ue, ve);
    const double di = Dh[i * n1 + m], dj = Dh[j * n1 + m];
    sye_u += di * (M.ye[qx] * ux);
    syx_u += dj * (M.yx[qe] * ue);
    sxe_u += di * (M.xe[qx] * ux);
    sxx_u += dj * (M.xx[qe] * ue);
    sye_v += di * (M.ye[qx] * vx);
    syx_v += dj * (M.yx[qe] * ve);
    sxe_v += di * (M.xe[qx] * vx);
    sxx_v += dj * (M.xx[qe] * ve);
  }
  double u1 = 0.0, u2 = 0.0, v1 = 0.0, v2 = 0.0;
  u1 += 1.0 * sye_u;
  u1 += -1.0 * syx_u;
  u2 += -1.0 * sxe_u;
  u2 += 1.0 * sxx_u;
  v1 += 1.0 * sye_v;
  v1 += -1.0 * syx_v;
  v2 += -1.0 * sxe_v;
  v2 += 1.0 * sxx_v;
  // interface corrections, plus side before minus side inside one face
  double uo, vo;
  velocity(S.h[n], S.hu[n], S.hv[n], P.h_des, uo, vo);
  const NodeFaces nf = sorted_faces(M, e, i, j, /*minus_first=*/false);
  for (int q = 0; q < nf.n; ++q) {
    const int face = nf.face[q], t = nf.t[q];
    const int4 ef = M.ef[e * 4 + face];
    double us = uo, vs = vo;
    if (!(ef.y & EF_WALL)) {
      long long nb, fidx;
      partner_of(M, e, face, t, ef, nb, fidx);
      double ub, vb;
      velocity(S.h[nb], S.hu[nb], S.hv[nb], P.h_des, ub, vb);
      if (ef.y & EF_MINUS) {
        us = 0.5 * (uo + ub);
        vs = 0.5 * (vo + vb);
      } else {
        us = 0.5 * (ub + uo);
        vs = 0.5 * (vb + vo);
      }
    }
    double cy, cx;
    switch (face) {
      case 1: cy = M.ye[n] / M.w0; cx = M.xe[n] / M.w0; break;
      case 3: cy = -M.ye[n] / M.w0; cx = -M.xe[n] / M.w0; break;
      case 2: cy = -M.yx[n] / M.w0; cx = -M.xx[n] / M.w0; break;
      default: cy = M.yx[n] / M.w0; cx = M.xx[n] / M.w0; break;
    }
    u1 += cy * us;
    u2 -= cx * us;
    v1 += cy * vs;
    v2 -= cx * vs;
  }
  const double inv_j = 1.0 / M.jac[n];
  u1 *= inv_j;
  u2 *= inv_j;
  v1 *= inv_j;
  v2 *= inv_j;
  const double he = S.h[n] * eps[e];
  fvu[n] = he * u1;
  fvv[n] = he * v1;
  gvu[n] = he * u2;
  gvv[n] = he * v2;
}

// ------------------------------------------------------------------------
// One RK stage, one thread per node: dW/dt (assemble_rhs dg_rhs.hpp:267-303
// with the viscous operator viscous_lhs viscosity.hpp:195-246 and optional
// forcing), then StateVec::axpy/combine (timeloop.hpp:114-127).
template <bool VISC, bool FORCE>
__global__ void k_rhs_stage(Mesh M, Phys P, StageArgs A) {
  const long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (n >= (long long)M.n_owned * M.np) return;
  const int n1 = M.n1, np = M.np;
  const int e = (int)(n / np), loc = (int)(n % np), i = loc / n1, j = loc % n1;
  const long long base = (long long)e * np;
  const double g = P.g, h_des = P.h_des, half = 0.5;
  const double *h = A.in.h, *hu = A.in.hu, *hv = A.in.hv;

  const double hn = h[n], hun = hu[n], hvn = hv[n];
  double un, vn;
  velocity(hn, hun, hvn, h_des, un, vn);

  // split_volume_element (dg_rhs.hpp:23-71) with volume_flux_pair (fluxes.hpp:21-39),
  // or standard_volume_element (dg_rhs.hpp:75-117): pointwise contravariant
  // fluxes (recomputed per partner node: bitwise the reference's ft/gt) and D
  double ah = 0.0, ahu = 0.0, ahv = 0.0;
  if (P.standard) {
    for (int m = 0; m < n1; ++m) {
      const double di = M.D[i * n1 + m], dj = M.D[j * n1 + m];
      const long long qx = base + m * n1 + j, qe = base + i * n1 + m;
      double fx[3], fy[3], ex[3], ey[3];
      phys_flux(h[qx], hu[qx], hv[qx], g, h_des, fx, fy);
      phys_flux(h[qe], hu[qe], hv[qe], g, h_des, ex, ey);
      double ft[3], gt[3];
      for (int c = 0; c < 3; ++c) {
        ft[c] = M.ye[qx] * fx[c] - M.xe[qx] * fy[c];
        gt[c] = M.xx[qe] * ey[c] - M.yx[qe] * ex[c];
      }
      ah += di * ft[0] + dj * gt[0];
      ahu += di * ft[1] + dj * gt[1];
      ahv += di * ft[2] + dj * gt[2];
    }
  }
  for (int dir = 0; dir < (P.standard ? 0 : 2); ++dir)
    for (int m = 0; m < n1; ++m) {
      const long long q = dir == 0 ? base + m * n1 + j : base + i * n1 + m;
      const double hq = h[q], huq = hu[q], hvq = hv[q];
      double uq, vq;
      velocity(hq, huq, hvq, h_des, uq, vq);
      const double havg = half * (hn + hq);
      const double uavg = half * (un + uq);
      const double vavg = half * (vn + vq);
      const double huavg = half * (hun + huq);
      const double hvavg = half * (hvn + hvq);
      const double h2avg = half * (hn * hn + hq * hq);
      const double press = g * havg * havg - half * g * h2avg;
      const double fs0 = huavg, fs1 = huavg * uavg + press, fs2 = huavg * vavg;
      const double gs0 = hvavg, gs1 = hvavg * uavg, gs2 = hvavg * vavg + press;
      if (dir == 0) {
        const double a = half * (M.ye[n] + M.ye[q]);
        const double b = half * (M.xe[n] + M.xe[q]);
        const double d = M.Dt[i * n1 + m];
        ah += d * (a * fs0 - b * gs0);
        ahu += d * (a * fs1 - b * gs1);
        ahv += d * (a * fs2 - b * gs2);
      } else {
        const double a = half * (M.yx[n] + M.yx[q]);
        const double b = half * (M.xx[n] + M.xx[q]);
        const double d = M.Dt[j * n1 + m];
        ah += d * (b * gs0 - a * fs0);
        ahu += d * (b * gs1 - a * fs1);
        ahv += d * (b * gs2 - a * fs2);
      }
    }
  double rh = 0.0, rhu = 0.0, rhv = 0.0;
  rh += ah;
  rhu += ahu;
  rhv += ahv;

  // source_terms (dg_rhs.hpp:154-183); b*metric products as sample_bathymetry
  // defines them (mesh.hpp:227-230)
  {
    double db_xi = 0.0, db_eta = 0.0, dbye_xi = 0.0, dbyx_eta = 0.0, dbxe_xi = 0.0,
           dbxx_eta = 0.0;
    for (int m = 0; m < n1; ++m) {
      const double di = M.D[i * n1 + m], dj = M.D[j * n1 + m];
      const long long qx = base + m * n1 + j, qe = base + i * n1 + m;
      const double bx = M.b[qx], be = M.b[qe];
      db_xi += di * bx;
      db_eta += dj * be;
      dbye_xi += di * (M.ye[qx] * bx);
      dbyx_eta += dj * (M.yx[qe] * be);
      dbxe_xi += di * (M.xe[qx] * bx);
      dbxx_eta += dj * (M.xx[qe] * be);
    }
    const double hg2 = 0.5 * g * hn;
    const double src_hu = -hg2 * (M.ye[n] * db_xi + dbye_xi - M.yx[n] * db_eta - dbyx_eta);
    const double src_hv = -hg2 * (M.xx[n] * db_eta + dbxx_eta - M.xe[n] * db_xi - dbxe_xi);
    rhu -= src_hu;
    rhv -= src_hv;
  }

  // surface_terms (dg_rhs.hpp:202-252), es mode: this node's share of every
  // face flux touching it, in face-list order (minus before plus)
  {
    const NodeFaces nf = sorted_faces(M, e, i, j, /*minus_first=*/true);
    for (int q = 0; q < nf.n; ++q) {
      const int face = nf.face[q], t = nf.t[q];
      const int4 ef = M.ef[e * 4 + face];
      double f0, f1, f2, js, snx, sny;
      if (ef.y & EF_WALL) {
        const long long fi = ((long long)e * 4 + face) * n1 + t;
        const double nx = M.fnx[fi], ny = M.fny[fi];
        js = M.fjs[fi];
        // exterior_state (mesh.hpp:382-386)
        const double mn = hun * nx + hvn * ny;
        const double hup = hun - 2.0 * mn * nx, hvp = hvn - 2.0 * mn * ny;
        const double bn = M.b[n];
        if (P.standard)
          llf_flux(hn, hun, hvn, hn, hup, hvp, nx, ny, g, h_des, f0, f1, f2);
        else
          es_flux(hn, hun, hvn, hn, hup, hvp, bn, bn, nx, ny, g, h_des, f0, f1, f2);
        snx = nx;
        sny = ny;
      } else {
        long long nb, fi;
        partner_of(M, e, face, t, ef, nb, fi);
        const double nx = M.fnx[fi], ny = M.fny[fi];
        js = M.fjs[fi];
        snx = nx;
        sny = ny;
        if (P.standard) {
          if (ef.y & EF_MINUS)
            llf_flux(hn, hun, hvn, h[nb], hu[nb], hv[nb], nx, ny, g, h_des, f0, f1, f2);
          else
            llf_flux(h[nb], hu[nb], hv[nb], hn, hun, hvn, nx, ny, g, h_des, f0, f1, f2);
        } else if (ef.y & EF_MINUS) {
          es_flux(hn, hun, hvn, h[nb], hu[nb], hv[nb], M.b[n], M.b[nb], nx, ny, g, h_des, f0,
                  f1, f2);
        } else {
          es_flux(h[nb], hu[nb], hv[nb], hn, hun, hvn, M.b[nb], M.b[n], nx, ny, g, h_des, f0,
                  f1, f2);
        }
      }
      double c0 = js * f0, c1 = js * f1, c2 = js * f2;
      if (P.standard) {
        // strong form: minus the node's own normal physical flux (dg_rhs.hpp:228-246;
        // the plus side's exterior trace is its own state)
        double fx[3], fy[3];
        phys_flux(hn, hun, hvn, g, h_des, fx, fy);
        c0 -= js * (snx * fx[0] + sny * fy[0]);
        c1 -= js * (snx * fx[1] + sny * fy[1]);
        c2 -= js * (snx * fx[2] + sny * fy[2]);
      }
      if (ef.y & EF_MINUS) {
        rh += c0 / M.w0;
        rhu += c1 / M.w0;
        rhv += c2 / M.w0;
      } else {
        rh -= c0 / M.w0;
        rhu -= c1 / M.w0;
        rhv -= c2 / M.w0;
      }
    }
  }

  if (VISC) {
    // viscous_lhs (viscosity.hpp:195-246): strong-form divergence of the
    // contravariant viscous fluxes, then the averaged normal-flux penalties
    const double* D = M.D;
    double su = 0.0, sv = 0.0;
    for (int m = 0; m < n1; ++m) {
      const long long qx = base + m * n1 + j, qe = base + i * n1 + m;
      const double ftu = M.ye[qx] * A.fvu[qx] - M.xe[qx] * A.gvu[qx];
      const double ftv = M.ye[qx] * A.fvv[qx] - M.xe[qx] * A.gvv[qx];
      const double gtu = -M.yx[qe] * A.fvu[qe] + M.xx[qe] * A.gvu[qe];
      const double gtv = -M.yx[qe] * A.fvv[qe] + M.xx[qe] * A.gvv[qe];
      su += D[i * n1 + m] * ftu + D[j * n1 + m] * gtu;
      sv += D[i * n1 + m] * ftv + D[j * n1 + m] * gtv;
    }
    const NodeFaces nf = sorted_faces(M, e, i, j, /*minus_first=*/true);
    for (int q = 0; q < nf.n; ++q) {
      const int face = nf.face[q], t = nf.t[q];
      const int4 ef = M.ef[e * 4 + face];
      if (ef.y & EF_WALL) {
        const long long fi = ((long long)e * 4 + face) * n1 + t;
        const double nx = M.fnx[fi], ny = M.fny[fi], js = M.fjs[fi];
        const double phim_u = nx * A.fvu[n] + ny * A.gvu[n];
        const double phim_v = nx * A.fvv[n] + ny * A.gvv[n];
        su += js * (0.0 - phim_u) / M.w0;
        sv += js * (0.0 - phim_v) / M.w0;
        continue;
      }
      long long nb, fi;
      partner_of(M, e, face, t, ef, nb, fi);
      const double nx = M.fnx[fi], ny = M.fny[fi], js = M.fjs[fi];
      const long long nm = (ef.y & EF_MINUS) ? n : nb, npl = (ef.y & EF_MINUS) ? nb : n;
      const double phim_u = nx * A.fvu[nm] + ny * A.gvu[nm];
      const double phim_v = nx * A.fvv[nm] + ny * A.gvv[nm];
      const double phip_u = nx * A.fvu[npl] + ny * A.gvu[npl];
      const double phip_v = nx * A.fvv[npl] + ny * A.gvv[npl];
      const double du = 0.5 * (phip_u - phim_u);
      const double dv = 0.5 * (phip_v - phim_v);
      su += js * du / M.w0;
      sv += js * dv / M.w0;
    }
    rhu -= su;
    rhv -= sv;
  }

  const double inv_j = -1.0 / M.jac[n];
  rh *= inv_j;
  rhu *= inv_j;
  rhv *= inv_j;
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
  if (A.update) {
    double sh = hn, shu = hun, shv = hvn;
    sh += A.dt * rh;
    shu += A.dt * rhu;
    shv += A.dt * rhv;
    if (A.stage > 0) {
      sh = A.ca * A.wn.h[n] + A.cb * sh;
      shu = A.ca * A.wn.hu[n] + A.cb * shu;
      shv = A.ca * A.wn.hv[n] + A.cb * shv;
    }
    A.out.h[n] = sh;
    A.out.hu[n] = shu;
    A.out.hv[n] = shv;
  }
}

// ------------------------------------------------------------------------
// post_stage (timeloop.hpp:202-234) with element_average / limit_element
// (limiter.hpp:24-84), one thread per element (serial J w w sums keep the
// reference's summation order).  A rejected stage is discarded by the host,
// so limiting every element concurrently is equivalent to the reference's
// "check all means, then limit" two-pass loop.
__global__ void k_limit(Mesh M, Phys P, State S, Flags* F) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= M.n_owned) return;
  const int n1 = M.n1, np = M.np;
  const long long b = (long long)e * np;
  double area = 0.0, a0 = 0.0, a1 = 0.0, a2 = 0.0;
  for (int i = 0; i < n1; ++i)
    for (int j = 0; j < n1; ++j) {
      const long long n = b + i * n1 + j;
      const double w = M.jac[n] * M.w[i] * M.w[j];
      area += w;
      a0 += w * S.h[n];
      a1 += w * S.hu[n];
      a2 += w * S.hv[n];
    }
  const double inv = 1.0 / area;
  const double avg0 = inv * a0, avg1 = inv * a1, avg2 = inv * a2;
  if (avg0 < 0.0) {
    atomicExch(&F->reject, 1);
    if (!P.limiter) atomicExch(&F->abort, 1);
    return;
  }
  double mn;
  if (!P.limiter) {
    mn = S.h[b];
    for (int n = 0; n < np; ++n) {
      if (S.h[b + n] < 0.0) atomicExch(&F->abort, 1);
      mn = smin(mn, S.h[b + n]);
    }
    atomicMin(&F->min_h_key, order_key(mn));
    return;
  }
  double mmin = S.h[b];
  for (int n = 1; n < np; ++n) mmin = smin(mmin, S.h[b + n]);
  double theta = 1.0;
  if (mmin < 0.0) {
    const double denom = avg0 - mmin;
    theta = denom < 1e-14 ? 1.0 : smin(1.0, avg0 / denom);
  }
  if (theta < 1.0) {
    atomicAdd(&F->n_limited, 1);
    for (int n = 0; n < np; ++n) {
      double h = theta * (S.h[b + n] - avg0) + avg0;
      S.hu[b + n] = theta * (S.hu[b + n] - avg1) + avg1;
      S.hv[b + n] = theta * (S.hv[b + n] - avg2) + avg2;
      S.h[b + n] = smax(h, 0.0);
    }
  }
  mn = S.h[b];
  for (int n = 0; n < np; ++n) {
    const double h = S.h[b + n];
    if (h < P.h_tol) {
      S.hu[b + n] = 0.0;
      S.hv[b + n] = 0.0;
    }
    mn = smin(mn, h);
  }
  atomicMin(&F->min_h_key, order_key(mn));
}

}  // namespace

// ---------------------------------------------------------------------------
// launchers (host)
int launch_exact_indicator(const Mesh& M, CState S, double* r, cudaStream_t st) {
  k_indicator<<<(M.K + 127) / 128, 128, 0, st>>>(M, S, r);
  return 1;
}

int launch_exact_grad(const Mesh& M, const Phys& P, CState S, const double* eps, double* fvu,
                      double* fvv, double* gvu, double* gvv, cudaStream_t st) {
  const long long nn = (long long)M.n_owned * M.np;
  k_grad<<<(unsigned)((nn + 255) / 256), 256, 0, st>>>(M, P, S, eps, fvu, fvv, gvu, gvv);
  return 1;
}

int launch_exact_rhs_stage(const Mesh& M, const Phys& P, const StageArgs& A, cudaStream_t st) {
  const long long nn = (long long)M.n_owned * M.np;
  const unsigned grid = (unsigned)((nn + 255) / 256);
  const bool visc = A.fvu != nullptr, force = A.fh != nullptr;
  if (visc && force) k_rhs_stage<true, true><<<grid, 256, 0, st>>>(M, P, A);
  else if (visc) k_rhs_stage<true, false><<<grid, 256, 0, st>>>(M, P, A);
  else if (force) k_rhs_stage<false, true><<<grid, 256, 0, st>>>(M, P, A);
  else k_rhs_stage<false, false><<<grid, 256, 0, st>>>(M, P, A);
  return 1;
}

int launch_exact_limit(const Mesh& M, const Phys& P, State S, Flags* F, cudaStream_t st) {
  k_limit<<<(M.n_owned + 127) / 128, 128, 0, st>>>(M, P, S, F);
  return 1;
}


}  // namespace swdg_dev
