/* oracle/swdg_port.c — TEST INFRASTRUCTURE ONLY (parity checker, never the product).
 *
 * Plain-C restatement of the reference stage path; see swdg_port.h.  Compile
 * with -ffp-contract=off (oracle/Makefile): every expression below keeps the
 * reference's evaluation order, so the results are bitwise those of the
 * reference built at its Release flags.  Comments give the reference
 * file:line each block restates (paths under proj/include/swdg/).
 */
#define _DEFAULT_SOURCE /* M_PI */
#include "swdg_port.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static char g_err[256];
const char* port_last_error(void) { return g_err; }
static int set_err(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

/* std::min / std::max semantics (first argument wins ties and NaN cases). */
static inline double smin(double a, double b) { return (b < a) ? b : a; }
static inline double smax(double a, double b) { return (a < b) ? b : a; }

/* node_index / face_node_index (core.hpp:42-61) */
static inline int face_node(int n1, int face, int t) {
  switch (face) {
    case 0: return t * n1;                /* south: (t, 0) */
    case 1: return (n1 - 1) * n1 + t;     /* east:  (N, t) */
    case 2: return t * n1 + (n1 - 1);     /* north: (t, N) */
    default: return t;                    /* west:  (0, t) */
  }
}
static inline int partner(const swdg_face* f, int degree, int t) {
  return f->reversed ? degree - t : t; /* mesh.hpp:51-53 */
}
static inline int owned(const swdg_mesh_view* m) {
  return m->n_owned > 0 ? m->n_owned : m->n_elem;
}

/* phys::velocity (physics.hpp:23-36) */
static inline void velocity(double h, double hu, double hv, double h_des, double* u,
                            double* v) {
  if (h >= h_des) {
    *u = hu / h;
    *v = hv / h;
  } else {
    *u = 0.0;
    *v = 0.0;
  }
}

/* fluxes::volume_flux_pair (fluxes.hpp:21-39) */
static inline void volume_pair(double ha, double ua, double va, double hua, double hva,
                               double hb, double ub, double vb, double hub, double hvb,
                               double g, double* fs, double* gs) {
  const double half = 0.5;
  const double havg = half * (ha + hb);
  const double uavg = half * (ua + ub);
  const double vavg = half * (va + vb);
  const double huavg = half * (hua + hub);
  const double hvavg = half * (hva + hvb);
  const double h2avg = half * (ha * ha + hb * hb);
  const double press = g * havg * havg - half * g * h2avg;
  fs[0] = huavg;
  fs[1] = huavg * uavg + press;
  fs[2] = huavg * vavg;
  gs[0] = hvavg;
  gs[1] = hvavg * uavg;
  gs[2] = hvavg * vavg + press;
}

/* fluxes::es_surface_flux_normal (fluxes.hpp:136-166) with make_dissipation
 * (96-108), apply_dissipation (111-118), phys::rotate/unrotate (physics.hpp:78-98). */
static int es_flux(const double* wm, const double* wp, double bm, double bp, double nx,
                   double ny, double g, double h_des, double* out) {
  if (fabs(sqrt(nx * nx + ny * ny) - 1.0) > 1e-10)
    return set_err(SWDG_ERR_INPUT, "normal vector is not unit length");
  double um, vm, up, vp;
  velocity(wm[0], wm[1], wm[2], h_des, &um, &vm);
  velocity(wp[0], wp[1], wp[2], h_des, &up, &vp);
  const double unm = nx * um + ny * vm, utm = -ny * um + nx * vm;
  const double unp = nx * up + ny * vp, utp = -ny * up + nx * vp;
  const double havg = 0.5 * (wm[0] + wp[0]);
  const double h2avg = 0.5 * (wm[0] * wm[0] + wp[0] * wp[0]);
  const double uavg = 0.5 * (unm + unp);
  const double vavg = 0.5 * (utm + utp);
  const double cavg = 0.5 * (sqrt(g * smax(wm[0], 0.0)) + sqrt(g * smax(wp[0], 0.0)));
  double f0 = havg * uavg;
  double f1 = havg * uavg * uavg + 0.5 * g * h2avg;
  double f2 = havg * uavg * vavg;
  const double x0 = g * ((wp[0] + bp) - (wm[0] + bm)) - 0.5 * (unp * unp - unm * unm) -
                    0.5 * (utp * utp - utm * utm);
  const double x1 = unp - unm, x2 = utp - utm;
  /* R = [[1,0,1],[u+c,0,u-c],[v,1,v]], |Lambda| = (s|u+c|, |h u|, s|u-c|) */
  const double r10 = uavg + cavg, r12 = uavg - cavg;
  const double s = 1.0 / (2.0 * g);
  const double l0 = s * fabs(uavg + cavg), l1 = fabs(havg * uavg), l2 = s * fabs(uavg - cavg);
  const double y0 = l0 * (1.0 * x0 + r10 * x1 + vavg * x2);
  const double y1 = l1 * (0.0 * x0 + 0.0 * x1 + 1.0 * x2);
  const double y2 = l2 * (1.0 * x0 + r12 * x1 + vavg * x2);
  const double d0 = 1.0 * y0 + 0.0 * y1 + 1.0 * y2;
  const double d1 = r10 * y0 + 0.0 * y1 + r12 * y2;
  const double d2 = vavg * y0 + 1.0 * y1 + vavg * y2;
  f0 -= 0.5 * d0;
  f1 -= 0.5 * d1;
  f2 -= 0.5 * d2;
  out[0] = f0;
  out[1] = nx * f1 - ny * f2;
  out[2] = ny * f1 + nx * f2;
  return 0;
}

int port_es_flux(const double* wm, const double* wp, double bm, double bp, double nx,
                 double ny, double g, double h_des, double* out3) {
  return es_flux(wm, wp, bm, bp, nx, ny, g, h_des, out3);
}

/* exterior_state (mesh.hpp:382-386): wall mirror */
static inline void wall_mirror(const double* w, double nx, double ny, double* out) {
  const double mn = w[1] * nx + w[2] * ny;
  out[0] = w[0];
  out[1] = w[1] - 2.0 * mn * nx;
  out[2] = w[2] - 2.0 * mn * ny;
}

/* -------------------------------------------------------------------------- */
/* assemble_rhs (dg_rhs.hpp:267-303)                                           */
/* -------------------------------------------------------------------------- */
int port_assemble_rhs(const swdg_mesh_view* m, const swdg_params* p, const double* h,
                      const double* hu, const double* hv, const double* visc_hu,
                      const double* visc_hv, const double* f_h, const double* f_hu,
                      const double* f_hv, double* rh, double* rhu, double* rhv) {
  const int n1 = m->degree + 1, np = n1 * n1, K = m->n_elem;
  const int64_t nn = (int64_t)K * np;
  const double g = p->g, h_des = p->h_des, half = 0.5;
  const double* Dt = m->deriv_modified;
  const double* D = m->deriv;
  double* u = malloc(sizeof(double) * np);
  double* v = malloc(sizeof(double) * np);
  for (int64_t n = 0; n < nn; ++n) rh[n] = rhu[n] = rhv[n] = 0.0;

  for (int e = 0; e < K; ++e) {
    const int64_t base = (int64_t)e * np;
    const double *eh = h + base, *ehu = hu + base, *ehv = hv + base;
    const double *ye = m->y_eta + base, *xe = m->x_eta + base;
    const double *yx = m->y_xi + base, *xx = m->x_xi + base;
    /* split_volume_element (dg_rhs.hpp:23-71) */
    for (int n = 0; n < np; ++n) velocity(eh[n], ehu[n], ehv[n], h_des, &u[n], &v[n]);
    for (int i = 0; i < n1; ++i)
      for (int j = 0; j < n1; ++j) {
        const int n = i * n1 + j;
        double ah = 0.0, ahu = 0.0, ahv = 0.0;
        for (int mm = 0; mm < n1; ++mm) { /* xi: (i,j) with (m,j) */
          const int q = mm * n1 + j;
          double fs[3], gs[3];
          volume_pair(eh[n], u[n], v[n], ehu[n], ehv[n], eh[q], u[q], v[q], ehu[q], ehv[q], g,
                      fs, gs);
          const double a = half * (ye[n] + ye[q]);
          const double b = half * (xe[n] + xe[q]);
          const double d = Dt[i * n1 + mm];
          ah += d * (a * fs[0] - b * gs[0]);
          ahu += d * (a * fs[1] - b * gs[1]);
          ahv += d * (a * fs[2] - b * gs[2]);
        }
        for (int mm = 0; mm < n1; ++mm) { /* eta: (i,j) with (i,m) */
          const int q = i * n1 + mm;
          double fs[3], gs[3];
          volume_pair(eh[n], u[n], v[n], ehu[n], ehv[n], eh[q], u[q], v[q], ehu[q], ehv[q], g,
                      fs, gs);
          const double a = half * (yx[n] + yx[q]);
          const double b = half * (xx[n] + xx[q]);
          const double d = Dt[j * n1 + mm];
          ah += d * (b * gs[0] - a * fs[0]);
          ahu += d * (b * gs[1] - a * fs[1]);
          ahv += d * (b * gs[2] - a * fs[2]);
        }
        rh[base + n] += ah;
        rhu[base + n] += ahu;
        rhv[base + n] += ahv;
      }
    /* source_terms (dg_rhs.hpp:154-183); b*metric products as in
     * sample_bathymetry (mesh.hpp:227-230) */
    const double* eb = m->b + base;
    for (int i = 0; i < n1; ++i)
      for (int j = 0; j < n1; ++j) {
        const int n = i * n1 + j;
        double db_xi = 0.0, db_eta = 0.0, dbye_xi = 0.0, dbyx_eta = 0.0, dbxe_xi = 0.0,
               dbxx_eta = 0.0;
        for (int mm = 0; mm < n1; ++mm) {
          const double di = D[i * n1 + mm], dj = D[j * n1 + mm];
          const int qx = mm * n1 + j, qe = i * n1 + mm;
          db_xi += di * eb[qx];
          db_eta += dj * eb[qe];
          dbye_xi += di * (ye[qx] * eb[qx]);
          dbyx_eta += dj * (yx[qe] * eb[qe]);
          dbxe_xi += di * (xe[qx] * eb[qx]);
          dbxx_eta += dj * (xx[qe] * eb[qe]);
        }
        const double hg2 = 0.5 * g * eh[n];
        const double src_hu = -hg2 * (ye[n] * db_xi + dbye_xi - yx[n] * db_eta - dbyx_eta);
        const double src_hv = -hg2 * (xx[n] * db_eta + dbxx_eta - xe[n] * db_xi - dbxe_xi);
        rhu[base + n] -= src_hu;
        rhv[base + n] -= src_hv;
      }
  }
  free(u);
  free(v);

  /* surface_terms (dg_rhs.hpp:202-252), es mode: one flux per face node,
   * scattered with opposite signs in face-list order */
  const double w0 = m->weights[0];
  for (int fi = 0; fi < m->n_faces; ++fi) {
    const swdg_face* f = &m->faces[fi];
    for (int t = 0; t < n1; ++t) {
      const int64_t fm = ((int64_t)f->elem_minus * 4 + f->face_minus) * n1 + t;
      const double nx = m->face_nx[fm], ny = m->face_ny[fm], js = m->face_jsurf[fm];
      const int64_t nm = (int64_t)f->elem_minus * np + face_node(n1, f->face_minus, t);
      const double wm[3] = {h[nm], hu[nm], hv[nm]};
      double wp[3];
      const double bm = m->b[nm];
      double bp = bm;
      int64_t npl = -1;
      if (f->tag == SWDG_TAG_WALL) {
        wall_mirror(wm, nx, ny, wp);
      } else {
        npl = (int64_t)f->elem_plus * np + face_node(n1, f->face_plus, partner(f, m->degree, t));
        wp[0] = h[npl];
        wp[1] = hu[npl];
        wp[2] = hv[npl];
        bp = m->b[npl];
      }
      double fl[3];
      const int rc = es_flux(wm, wp, bm, bp, nx, ny, g, h_des, fl);
      if (rc) return rc;
      const double c0 = js * fl[0], c1 = js * fl[1], c2 = js * fl[2];
      rh[nm] += c0 / w0;
      rhu[nm] += c1 / w0;
      rhv[nm] += c2 / w0;
      if (npl >= 0) {
        rh[npl] -= c0 / w0;
        rhu[npl] -= c1 / w0;
        rhv[npl] -= c2 / w0;
      }
    }
  }

  if (visc_hu)
    for (int64_t n = 0; n < nn; ++n) {
      rhu[n] -= visc_hu[n];
      rhv[n] -= visc_hv[n];
    }
  for (int64_t n = 0; n < nn; ++n) {
    const double inv_j = -1.0 / m->jac[n];
    rh[n] *= inv_j;
    rhu[n] *= inv_j;
    rhv[n] *= inv_j;
  }
  if (f_h)
    for (int64_t n = 0; n < nn; ++n) {
      rh[n] += f_h[n];
      rhu[n] += f_hu[n];
      rhv[n] += f_hv[n];
    }
  return 0;
}

/* -------------------------------------------------------------------------- */
/* viscosity (viscosity.hpp)                                                   */
/* -------------------------------------------------------------------------- */
double port_shock_indicator(int degree, const double* vinv, const double* field, int* err) {
  const int n1 = degree + 1, np = n1 * n1;
  if (degree < 2) {
    *err = set_err(SWDG_ERR_INPUT, "shock_indicator: requires degree >= 2");
    return 0.0;
  }
  double tmp[256], modal[256];
  /* nodal_to_modal (operators.hpp:191-206): modal = V^-1 nodal V^-T */
  for (int i = 0; i < n1; ++i)
    for (int j = 0; j < n1; ++j) {
      double s = 0.0;
      for (int k = 0; k < n1; ++k) s += vinv[i * n1 + k] * field[k * n1 + j];
      tmp[i * n1 + j] = s;
    }
  for (int i = 0; i < n1; ++i)
    for (int j = 0; j < n1; ++j) {
      double s = 0.0;
      for (int k = 0; k < n1; ++k) s += tmp[i * n1 + k] * vinv[j * n1 + k];
      modal[i * n1 + j] = s;
    }
  (void)np;
#define M2(i, j) (modal[(i) * n1 + (j)] * modal[(i) * n1 + (j)])
  double den1 = 0.0, den2 = 0.0;
  for (int i = 0; i < n1; ++i)
    for (int j = 0; j < n1; ++j) den1 += M2(i, j);
  for (int i = 0; i < n1 - 1; ++i)
    for (int j = 0; j < n1 - 1; ++j) den2 += M2(i, j);
  double num1 = M2(degree, degree), num2 = M2(degree - 1, degree - 1);
  for (int i = 0; i < degree; ++i) num1 += M2(i, degree) + M2(degree, i);
  for (int i = 0; i < degree - 1; ++i) num2 += M2(i, degree - 1) + M2(degree - 1, i);
#undef M2
  const double floor_abs = 1e-28 * den1 + 1e-300;
  if (den1 <= 1e-300) return -INFINITY;
  const double r1 = num1 > floor_abs ? num1 / den1 : 0.0;
  const double r2 = (num2 > floor_abs && den2 > floor_abs) ? num2 / den2 : 0.0;
  const double r = smax(r1, r2);
  if (r <= 0.0) return -INFINITY;
  return log10(r);
}

double port_viscosity_coefficient(double sigma, const swdg_params* p, int* err) {
  if (!(p->sigma_min < p->sigma_max)) {
    *err = set_err(SWDG_ERR_INPUT, "viscosity: sigma_min must be < sigma_max");
    return 0.0;
  }
  if (p->epsilon0 < 0.0) {
    *err = set_err(SWDG_ERR_INPUT, "viscosity: epsilon0 must be >= 0");
    return 0.0;
  }
  if (sigma < p->sigma_min) return 0.0;
  if (sigma >= p->sigma_max) return p->epsilon0;
  const double delta =
      1.0 + sin(M_PI * (sigma - 0.5 * (p->sigma_max + p->sigma_min)) / (p->sigma_max - p->sigma_min));
  return 0.5 * p->epsilon0 * delta;
}

int port_compute_viscosity(const swdg_mesh_view* m, const swdg_params* p, const double* h,
                           double* eps) {
  const int np = (m->degree + 1) * (m->degree + 1);
  for (int e = 0; e < m->n_elem; ++e) eps[e] = 0.0;
  if (!p->visc_enabled) return 0;
  for (int e = 0; e < m->n_elem; ++e) {
    int err = 0;
    const double sigma = port_shock_indicator(m->degree, m->vandermonde_inv, h + (int64_t)e * np, &err);
    if (err) return err;
    eps[e] = port_viscosity_coefficient(sigma, p, &err);
    if (err) return err;
  }
  return 0;
}

void port_velocities(const swdg_mesh_view* m, const swdg_params* p, const double* h,
                     const double* hu, const double* hv, double* u, double* v) {
  const int64_t nn = (int64_t)m->n_elem * (m->degree + 1) * (m->degree + 1);
  for (int64_t n = 0; n < nn; ++n) velocity(h[n], hu[n], hv[n], p->h_des, &u[n], &v[n]);
}

/* one BR1 volume_part (viscosity.hpp:103-112): out += sign * Dhat-sum(metric*f) */
static void br1_volume(int n1, const double* Dh, const double* metric, const double* f,
                       int xi_dir, double sign, double* pu, double* out) {
  const int np = n1 * n1;
  for (int n = 0; n < np; ++n) pu[n] = metric[n] * f[n];
  for (int i = 0; i < n1; ++i)
    for (int j = 0; j < n1; ++j) {
      double s = 0.0;
      for (int mm = 0; mm < n1; ++mm)
        s += xi_dir ? Dh[i * n1 + mm] * pu[mm * n1 + j] : Dh[j * n1 + mm] * pu[i * n1 + mm];
      out[i * n1 + j] += sign * s;
    }
}

int port_br1_gradients(const swdg_mesh_view* m, const double* u, const double* v, double* u1,
                       double* u2, double* v1, double* v2) {
  const int n1 = m->degree + 1, np = n1 * n1;
  const int64_t nn = (int64_t)m->n_elem * np;
  for (int64_t n = 0; n < nn; ++n) u1[n] = u2[n] = v1[n] = v2[n] = 0.0;
  double pu[256];
  const double* Dh = m->deriv_weak;
  for (int e = 0; e < m->n_elem; ++e) {
    const int64_t b = (int64_t)e * np;
    br1_volume(n1, Dh, m->y_eta + b, u + b, 1, 1.0, pu, u1 + b);
    br1_volume(n1, Dh, m->y_xi + b, u + b, 0, -1.0, pu, u1 + b);
    br1_volume(n1, Dh, m->x_eta + b, u + b, 1, -1.0, pu, u2 + b);
    br1_volume(n1, Dh, m->x_xi + b, u + b, 0, 1.0, pu, u2 + b);
    br1_volume(n1, Dh, m->y_eta + b, v + b, 1, 1.0, pu, v1 + b);
    br1_volume(n1, Dh, m->y_xi + b, v + b, 0, -1.0, pu, v1 + b);
    br1_volume(n1, Dh, m->x_eta + b, v + b, 1, -1.0, pu, v2 + b);
    br1_volume(n1, Dh, m->x_xi + b, v + b, 0, 1.0, pu, v2 + b);
  }
  /* interface corrections (viscosity.hpp:114-160) */
  const double w0 = m->weights[0];
  for (int fi = 0; fi < m->n_faces; ++fi) {
    const swdg_face* f = &m->faces[fi];
    for (int t = 0; t < n1; ++t) {
      const int64_t nm = (int64_t)f->elem_minus * np + face_node(n1, f->face_minus, t);
      double us = u[nm], vs = v[nm];
      for (int side = 0; side < 2; ++side) {
        /* plus side scattered first (viscosity.hpp:155-157), then minus */
        int64_t n;
        int face;
        if (side == 0) {
          if (f->tag != SWDG_TAG_INTERIOR) continue;
          const int tp = partner(f, m->degree, t);
          n = (int64_t)f->elem_plus * np + face_node(n1, f->face_plus, tp);
          us = 0.5 * (u[nm] + u[n]);
          vs = 0.5 * (v[nm] + v[n]);
          face = f->face_plus;
        } else {
          n = nm;
          face = f->face_minus;
        }
        double cy, cx;
        switch (face) {
          case 1: cy = m->y_eta[n] / w0; cx = m->x_eta[n] / w0; break;
          case 3: cy = -m->y_eta[n] / w0; cx = -m->x_eta[n] / w0; break;
          case 2: cy = -m->y_xi[n] / w0; cx = -m->x_xi[n] / w0; break;
          default: cy = m->y_xi[n] / w0; cx = m->x_xi[n] / w0; break;
        }
        u1[n] += cy * us;
        u2[n] -= cx * us;
        v1[n] += cy * vs;
        v2[n] -= cx * vs;
      }
    }
  }
  for (int64_t n = 0; n < nn; ++n) {
    const double inv_j = 1.0 / m->jac[n];
    u1[n] *= inv_j;
    u2[n] *= inv_j;
    v1[n] *= inv_j;
    v2[n] *= inv_j;
  }
  return 0;
}

int port_viscous_fluxes(const swdg_mesh_view* m, const double* h, const double* u1,
                        const double* u2, const double* v1, const double* v2, const double* eps,
                        double* fvu, double* fvv, double* gvu, double* gvv) {
  const int np = (m->degree + 1) * (m->degree + 1);
  for (int e = 0; e < m->n_elem; ++e)
    if (eps[e] < 0.0) return set_err(SWDG_ERR_INPUT, "viscous_lhs: negative viscosity coefficient");
  for (int e = 0; e < m->n_elem; ++e)
    for (int n = 0; n < np; ++n) {
      const int64_t k = (int64_t)e * np + n;
      const double he = h[k] * eps[e];
      fvu[k] = he * u1[k];
      fvv[k] = he * v1[k];
      gvu[k] = he * u2[k];
      gvv[k] = he * v2[k];
    }
  return 0;
}

int port_viscous_lhs(const swdg_mesh_view* m, const double* fvu, const double* fvv,
                     const double* gvu, const double* gvv, double* out_hu, double* out_hv) {
  const int n1 = m->degree + 1, np = n1 * n1;
  const double* D = m->deriv;
  double ftu[256], ftv[256], gtu[256], gtv[256];
  for (int e = 0; e < m->n_elem; ++e) {
    const int64_t b = (int64_t)e * np;
    for (int n = 0; n < np; ++n) {
      const int64_t k = b + n;
      ftu[n] = m->y_eta[k] * fvu[k] - m->x_eta[k] * gvu[k];
      ftv[n] = m->y_eta[k] * fvv[k] - m->x_eta[k] * gvv[k];
      gtu[n] = -m->y_xi[k] * fvu[k] + m->x_xi[k] * gvu[k];
      gtv[n] = -m->y_xi[k] * fvv[k] + m->x_xi[k] * gvv[k];
    }
    for (int i = 0; i < n1; ++i)
      for (int j = 0; j < n1; ++j) {
        double su = 0.0, sv = 0.0;
        for (int mm = 0; mm < n1; ++mm) {
          su += D[i * n1 + mm] * ftu[mm * n1 + j] + D[j * n1 + mm] * gtu[i * n1 + mm];
          sv += D[i * n1 + mm] * ftv[mm * n1 + j] + D[j * n1 + mm] * gtv[i * n1 + mm];
        }
        out_hu[b + i * n1 + j] = su;
        out_hv[b + i * n1 + j] = sv;
      }
  }
  const double w0 = m->weights[0];
  for (int fi = 0; fi < m->n_faces; ++fi) {
    const swdg_face* f = &m->faces[fi];
    for (int t = 0; t < n1; ++t) {
      const int64_t fm = ((int64_t)f->elem_minus * 4 + f->face_minus) * n1 + t;
      const double nx = m->face_nx[fm], ny = m->face_ny[fm], js = m->face_jsurf[fm];
      const int64_t nm = (int64_t)f->elem_minus * np + face_node(n1, f->face_minus, t);
      const double phim_u = nx * fvu[nm] + ny * gvu[nm];
      const double phim_v = nx * fvv[nm] + ny * gvv[nm];
      if (f->tag == SWDG_TAG_WALL) {
        out_hu[nm] += js * (0.0 - phim_u) / w0;
        out_hv[nm] += js * (0.0 - phim_v) / w0;
        continue;
      }
      const int64_t npl =
          (int64_t)f->elem_plus * np + face_node(n1, f->face_plus, partner(f, m->degree, t));
      const double phip_u = nx * fvu[npl] + ny * gvu[npl];
      const double phip_v = nx * fvv[npl] + ny * gvv[npl];
      const double du = 0.5 * (phip_u - phim_u);
      const double dv = 0.5 * (phip_v - phim_v);
      out_hu[nm] += js * du / w0;
      out_hv[nm] += js * dv / w0;
      out_hu[npl] += js * du / w0;
      out_hv[npl] += js * dv / w0;
    }
  }
  return 0;
}

int port_evaluate_rhs(const swdg_mesh_view* m, const swdg_params* p, const double* h,
                      const double* hu, const double* hv, const double* f_h,
                      const double* f_hu, const double* f_hv, double* rh, double* rhu,
                      double* rhv, double* eps) {
  if (!p->visc_enabled)
    return port_assemble_rhs(m, p, h, hu, hv, NULL, NULL, f_h, f_hu, f_hv, rh, rhu, rhv);
  const int64_t nn = (int64_t)m->n_elem * (m->degree + 1) * (m->degree + 1);
  double* buf = malloc(sizeof(double) * nn * 12);
  double *u = buf, *v = buf + nn, *u1 = buf + 2 * nn, *u2 = buf + 3 * nn, *v1 = buf + 4 * nn,
         *v2 = buf + 5 * nn, *fvu = buf + 6 * nn, *fvv = buf + 7 * nn, *gvu = buf + 8 * nn,
         *gvv = buf + 9 * nn, *vhu = buf + 10 * nn, *vhv = buf + 11 * nn;
  int rc = port_compute_viscosity(m, p, h, eps);
  if (!rc) {
    port_velocities(m, p, h, hu, hv, u, v);
    rc = port_br1_gradients(m, u, v, u1, u2, v1, v2);
  }
  if (!rc) rc = port_viscous_fluxes(m, h, u1, u2, v1, v2, eps, fvu, fvv, gvu, gvv);
  if (!rc) rc = port_viscous_lhs(m, fvu, fvv, gvu, gvv, vhu, vhv);
  if (!rc) rc = port_assemble_rhs(m, p, h, hu, hv, vhu, vhv, f_h, f_hu, f_hv, rh, rhu, rhv);
  free(buf);
  return rc;
}

/* -------------------------------------------------------------------------- */
/* limiter (limiter.hpp) and SSPRK3 (timeloop.hpp)                             */
/* -------------------------------------------------------------------------- */
void port_element_average(const swdg_mesh_view* m, const double* h, const double* hu,
                          const double* hv, int e, double* avg3, double* area_out) {
  const int n1 = m->degree + 1, np = n1 * n1;
  double area = 0.0, a0 = 0.0, a1 = 0.0, a2 = 0.0;
  for (int i = 0; i < n1; ++i)
    for (int j = 0; j < n1; ++j) {
      const int64_t n = (int64_t)e * np + i * n1 + j;
      const double w = m->jac[n] * m->weights[i] * m->weights[j];
      area += w;
      a0 += w * h[n];
      a1 += w * hu[n];
      a2 += w * hv[n];
    }
  if (area_out) *area_out = area;
  const double inv = 1.0 / area;
  avg3[0] = inv * a0;
  avg3[1] = inv * a1;
  avg3[2] = inv * a2;
}

double port_limit_element(const swdg_mesh_view* m, const swdg_params* p, double* h, double* hu,
                          double* hv, int e, int zero_dry, int* err) {
  const int np = (m->degree + 1) * (m->degree + 1);
  const int64_t b = (int64_t)e * np;
  double avg[3];
  port_element_average(m, h, hu, hv, e, avg, NULL);
  double mmin = h[b];
  for (int n = 1; n < np; ++n) mmin = smin(mmin, h[b + n]);
  if (avg[0] < 0.0) {
    *err = set_err(SWDG_ERR_INPUT, "limiter: negative element mean water height");
    return 1.0;
  }
  double theta = 1.0;
  if (mmin < 0.0) {
    const double denom = avg[0] - mmin;
    theta = denom < 1e-14 ? 1.0 : smin(1.0, avg[0] / denom);
  }
  if (theta < 1.0)
    for (int n = 0; n < np; ++n) {
      h[b + n] = theta * (h[b + n] - avg[0]) + avg[0];
      hu[b + n] = theta * (hu[b + n] - avg[1]) + avg[1];
      hv[b + n] = theta * (hv[b + n] - avg[2]) + avg[2];
      h[b + n] = smax(h[b + n], 0.0);
    }
  if (zero_dry)
    for (int n = 0; n < np; ++n)
      if (h[b + n] < p->h_tol) {
        hu[b + n] = 0.0;
        hv[b + n] = 0.0;
      }
  return theta;
}

static double min_height_owned(const swdg_mesh_view* m, const double* h) {
  const int64_t nn = (int64_t)owned(m) * (m->degree + 1) * (m->degree + 1);
  double mn = nn ? h[0] : 0.0;
  for (int64_t n = 0; n < nn; ++n) mn = smin(mn, h[n]);
  return mn;
}

int port_post_stage(const swdg_mesh_view* m, const swdg_params* p, double* h, double* hu,
                    double* hv, int* n_limited, double* min_stage_h) {
  const int np = (m->degree + 1) * (m->degree + 1), K = owned(m);
  for (int e = 0; e < K; ++e) {
    double avg[3];
    port_element_average(m, h, hu, hv, e, avg, NULL);
    if (avg[0] < 0.0) {
      if (!p->limiter_enabled) {
        set_err(SWDG_ERR_ABORT, "negative element mean water height without limiter");
        return -1;
      }
      return 0;
    }
  }
  if (!p->limiter_enabled) {
    for (int64_t n = 0; n < (int64_t)K * np; ++n)
      if (h[n] < 0.0) {
        set_err(SWDG_ERR_ABORT, "negative water height without limiter");
        return -1;
      }
    *min_stage_h = smin(*min_stage_h, min_height_owned(m, h));
    return 1;
  }
  *n_limited = 0;
  for (int e = 0; e < K; ++e) {
    int err = 0;
    const double theta = port_limit_element(m, p, h, hu, hv, e, 1, &err);
    if (theta < 1.0) ++*n_limited;
  }
  *min_stage_h = smin(*min_stage_h, min_height_owned(m, h));
  return 1;
}

static void wave_forcing(const swdg_mesh_view* m, const double* fp, double t, double* fh,
                         double* fhu, double* fhv) {
  const double h0 = fp[0], amp = fp[1], u0 = fp[2], v0 = fp[3], k = fp[4], g = fp[5];
  const double omega = k * (u0 + v0);
  const int64_t nn = (int64_t)m->n_elem * (m->degree + 1) * (m->degree + 1);
  for (int64_t n = 0; n < nn; ++n) {
    const double x = m->x[n], y = m->y[n];
    const double hx = amp * k * cos(k * (x + y) - omega * t);
    const double hh = h0 + amp * sin(k * (x + y) - omega * t);
    fh[n] = 0.0;
    fhu[n] = g * hh * hx;
    fhv[n] = g * hh * hx;
  }
}

int port_try_step(const swdg_mesh_view* m, const swdg_params* p, double* h, double* hu,
                  double* hv, double t, double dt, int forcing_kind, const double* fparams,
                  swdg_step_info* info) {
  static const double ca[3] = {0.0, 3.0 / 4.0, 1.0 / 3.0};
  static const double cb[3] = {1.0, 1.0 / 4.0, 2.0 / 3.0};
  static const double ct[3] = {0.0, 1.0, 0.5};
  const int64_t nn = (int64_t)m->n_elem * (m->degree + 1) * (m->degree + 1);
  if (p->visc_enabled && m->degree < 2)
    return set_err(SWDG_ERR_INPUT, "artificial viscosity requires polynomial degree >= 2");
  double* buf = malloc(sizeof(double) * nn * 9);
  double *sh = buf, *shu = buf + nn, *shv = buf + 2 * nn;
  double *rh = buf + 3 * nn, *rhu = buf + 4 * nn, *rhv = buf + 5 * nn;
  double *fh = buf + 6 * nn, *fhu = buf + 7 * nn, *fhv = buf + 8 * nn;
  double* eps = malloc(sizeof(double) * (m->n_elem + 1));
  memcpy(sh, h, sizeof(double) * nn);
  memcpy(shu, hu, sizeof(double) * nn);
  memcpy(shv, hv, sizeof(double) * nn);
  info->n_limited = 0;
  info->max_eps = 0.0;
  info->min_stage_h = INFINITY;
  info->accepted = 0;
  int rc = 0;
  for (int k = 0; k < 3 && !rc; ++k) {
    const int forced = forcing_kind == 1;
    if (forced) wave_forcing(m, fparams, t + ct[k] * dt, fh, fhu, fhv);
    rc = port_evaluate_rhs(m, p, sh, shu, shv, forced ? fh : NULL, forced ? fhu : NULL,
                           forced ? fhv : NULL, rh, rhu, rhv, eps);
    if (rc) break;
    if (p->visc_enabled)
      for (int e = 0; e < m->n_elem; ++e) info->max_eps = smax(info->max_eps, eps[e]);
    for (int64_t n = 0; n < nn; ++n) { /* StateVec::axpy (timeloop.hpp:114-120) */
      sh[n] += dt * rh[n];
      shu[n] += dt * rhu[n];
      shv[n] += dt * rhv[n];
    }
    if (k > 0)
      for (int64_t n = 0; n < nn; ++n) { /* StateVec::combine (timeloop.hpp:121-127) */
        sh[n] = ca[k] * h[n] + cb[k] * sh[n];
        shu[n] = ca[k] * hu[n] + cb[k] * shu[n];
        shv[n] = ca[k] * hv[n] + cb[k] * shv[n];
      }
    const int ok = port_post_stage(m, p, sh, shu, shv, &info->n_limited, &info->min_stage_h);
    if (ok < 0) rc = SWDG_ERR_ABORT;
    else if (ok == 0) break;
    else if (k == 2) info->accepted = 1;
  }
  if (!rc && info->accepted) {
    memcpy(h, sh, sizeof(double) * nn);
    memcpy(hu, shu, sizeof(double) * nn);
    memcpy(hv, shv, sizeof(double) * nn);
  }
  free(buf);
  free(eps);
  return rc;
}

int port_compute_dt(const swdg_mesh_view* m, const swdg_params* p, const double* h,
                    const double* hu, const double* hv, double cfl, double* dt_out) {
  if (!(cfl > 0.0) || cfl > 1.0) return set_err(SWDG_ERR_INPUT, "compute_dt: cfl must be in (0, 1]");
  const double order = 2.0 * m->degree + 1.0;
  double dt = INFINITY, min_len = INFINITY;
  const int64_t nn = (int64_t)owned(m) * (m->degree + 1) * (m->degree + 1);
  for (int64_t n = 0; n < nn; ++n) {
    double u, v;
    velocity(h[n], hu[n], hv[n], p->h_des, &u, &v);
    const double c = sqrt(p->g * smax(h[n], 0.0));
    const double len_xi = 2.0 * m->jac[n] / hypot(m->x_eta[n], m->y_eta[n]);
    const double len_eta = 2.0 * m->jac[n] / hypot(m->x_xi[n], m->y_xi[n]);
    min_len = smin(min_len, smin(len_xi, len_eta));
    const double lx = fabs(u) + c, ly = fabs(v) + c;
    if (lx > 1e-14) dt = smin(dt, len_xi / (order * lx));
    if (ly > 1e-14) dt = smin(dt, len_eta / (order * ly));
  }
  if (!isfinite(dt)) dt = min_len / (order * sqrt(p->g * smax(p->h_ref, 1e-12)));
  *dt_out = cfl * dt;
  return 0;
}

/* positivity_dt_bounds (limiter.hpp:107-130) */
static void posdt_bounds(const double* wm, const double* wp, double nx, double ny, double w0,
                         double a_scale, const swdg_params* p, double* b1, double* b2) {
  double um, vm, up, vp;
  velocity(wm[0], wm[1], wm[2], p->h_des, &um, &vm);
  velocity(wp[0], wp[1], wp[2], p->h_des, &up, &vp);
  const double unm = nx * um + ny * vm, unp = nx * up + ny * vp;
  const double uavg = 0.5 * (unm + unp);
  const double cavg =
      0.5 * (sqrt(p->g * smax(wm[0], 0.0)) + sqrt(p->g * smax(wp[0], 0.0)));
  const double a = fabs(uavg + cavg) + fabs(uavg - cavg);
  const double b = fabs(uavg + cavg) - fabs(uavg - cavg);
  const double den1 = a + 2.0 * uavg;
  *b1 = den1 > 1e-300 ? w0 * a_scale / den1 : INFINITY;
  const double jump_un = unp - unm;
  *b2 = INFINITY;
  if (wm[0] > 0.0 && b * jump_un < 0.0)
    *b2 = fabs(w0 * a_scale * p->g * wm[0] / (cavg * b * jump_un));
}

int port_diagnostics(const swdg_mesh_view* m, const swdg_params* p, const double* h,
                     const double* hu, const double* hv, swdg_diagnostics* out) {
  const int n1 = m->degree + 1, np = n1 * n1, K = owned(m);
  double mass = 0.0, ent = 0.0;
  for (int e = 0; e < K; ++e)
    for (int i = 0; i < n1; ++i)
      for (int j = 0; j < n1; ++j) {
        const int64_t n = (int64_t)e * np + i * n1 + j;
        const double wi = m->weights[i], wj = m->weights[j];
        mass += h[n] * m->jac[n] * wi * wj;
        double u, v; /* phys::entropy_and_flux (physics.hpp:48-56) */
        velocity(h[n], hu[n], hv[n], p->h_des, &u, &v);
        const double k = 0.5 * h[n] * (u * u + v * v);
        const double e_n = k + 0.5 * p->g * h[n] * h[n] + p->g * h[n] * m->b[n];
        ent += e_n * m->jac[n] * wi * wj;
      }
  out->mass = mass;
  out->entropy = ent;
  out->min_h = min_height_owned(m, h);
  const double w0 = m->weights[0];
  double dt = INFINITY;
  for (int fi = 0; fi < m->n_faces; ++fi) {
    const swdg_face* f = &m->faces[fi];
    for (int t = 0; t < n1; ++t) {
      const int64_t fm = ((int64_t)f->elem_minus * 4 + f->face_minus) * n1 + t;
      const int64_t nm = (int64_t)f->elem_minus * np + face_node(n1, f->face_minus, t);
      const double nx = m->face_nx[fm], ny = m->face_ny[fm];
      const double wm[3] = {h[nm], hu[nm], hv[nm]};
      double wp[3], b1, b2;
      int64_t npl = -1;
      const int tp = partner(f, m->degree, t);
      if (f->tag == SWDG_TAG_WALL) {
        wall_mirror(wm, nx, ny, wp);
      } else {
        npl = (int64_t)f->elem_plus * np + face_node(n1, f->face_plus, tp);
        wp[0] = h[npl];
        wp[1] = hu[npl];
        wp[2] = hv[npl];
      }
      posdt_bounds(wm, wp, nx, ny, w0, m->face_a[fm], p, &b1, &b2);
      dt = smin(dt, smin(b1, b2));
      if (npl >= 0) {
        const int64_t fp = ((int64_t)f->elem_plus * 4 + f->face_plus) * n1 + tp;
        posdt_bounds(wp, wm, m->face_nx[fp], m->face_ny[fp], w0, m->face_a[fp], p, &b1, &b2);
        dt = smin(dt, smin(b1, b2));
      }
    }
  }
  out->positivity_dt = dt;
  return 0;
}
