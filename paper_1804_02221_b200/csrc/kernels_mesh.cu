// kernels_mesh.cu — device generation of the structured curvilinear meshes
// (mesh.hpp:114-232, 294-379) for the 1M-element throughput meshes (SURVEY §8d,
// C5): the transfinite blend of the four mapped edge curves sampled at the LGL
// nodes and the metrics by differentiating the nodal coordinate polynomials, in
// the reference's expression order.  Compiled with --fmad=false and free of
// device libm (the wavy map's sines come from a host table, glibc), so x, y,
// the metrics, J and the polynomial bathymetries are bitwise the reference's
// host build; the host (swdg_gpu.cu) finishes the hypot- and sin-dependent
// fields with glibc, as the reference does.
#include <cuda_runtime.h>

#include "swdg_device.cuh"
#include "swdg_mesh.h"

namespace swdg_dev {
namespace {

struct Pt {
  double x, y;
};

// su, sv: sin(2 pi u), sin(2 pi v) of this (u, v) from the host tables (wavy only)
__device__ Pt map_point(const MeshSpecDev& s, double u, double v, double su, double sv) {
  Pt p;
  switch (s.kind) {
    case 0:  // cartesian (mesh.hpp:342-349)
      p.x = s.x0 + u * (s.x1 - s.x0);
      p.y = s.y0 + v * (s.y1 - s.y0);
      break;
    case 1: {  // curved dam (mesh.hpp:352-366)
      p.y = s.y0 + v * (s.y1 - s.y0);
      const double xd = p.y * p.y / 25.0 - 0.25;
      if (u <= s.extra)
        p.x = s.x0 + (u / s.extra) * (xd - s.x0);
      else
        p.x = xd + ((u - s.extra) / (1.0 - s.extra)) * (s.x1 - xd);
      break;
    }
    default: {  // wavy (mesh.hpp:370-379)
      const double w = su * sv;
      p.x = s.x0 + (u + s.extra * w) * (s.x1 - s.x0);
      p.y = s.y0 + (v - 0.75 * s.extra * w) * (s.y1 - s.y0);
      break;
    }
  }
  return p;
}

// BoundaryCurve of structured_mesh (mesh.hpp:313-318): map(u0 + t (u1 - u0),
// v0 + t (v1 - v0)), t = (1 + r) / 2.  A curve varies u (south/north: su = the
// table entry of sample k, sv fixed) or v (west/east).
__device__ Pt curve(const MeshSpecDev& s, double u0, double v0, double u1, double v1, double r,
                    double su, double sv) {
  const double t = 0.5 * (1.0 + r);
  return map_point(s, u0 + t * (u1 - u0), v0 + t * (v1 - v0), su, sv);
}

// the closures of oracle/ref_capi.cpp ref_mesh_bathymetry without libm; kinds 4
// and 6 (sines) are sampled on the host
__device__ double bathymetry(const MeshSpecDev& s, double x, double y) {
  const double* p = s.bathy;
  switch (s.bathy_kind) {
    case 1: return p[0];
    case 2: return p[0] * x + p[1] * y + p[2];
    case 3: return p[0] * (x * x + y * y);
    case 5: return x < p[0] ? p[1] : p[2];
    default: return 0.0;
  }
}

// build_transfinite_element (mesh.hpp:114-159), one thread per node
__global__ void k_coords(MeshSpecDev s, const double* nodes, int n1, long long nn, double* x,
                         double* y) {
  const long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (n >= nn) return;
  const int np = n1 * n1;
  const int e = (int)(n / np), loc = (int)(n % np), i = loc / n1, j = loc % n1;
  const int eg = s.gid ? s.gid[e] : e;
  const int ex = eg % s.kx, ey = eg / s.kx;
  const double u0 = (double)ex / s.kx, u1 = (double)(ex + 1) / s.kx;
  const double v0 = (double)ey / s.ky, v1 = (double)(ey + 1) / s.ky;
  const double xi = nodes[i], eta = nodes[j];
  const bool wavy = s.kind == 2;
  const int n2 = n1 + 2;
  // table entries: u samples along south/north (k = i, corners n1, n1 + 1), the
  // fixed u0 / u1 of west/east; likewise v
  auto SU = [&](int k) { return wavy ? s.sin_u[ex * n2 + k] : 0.0; };
  auto SV = [&](int k) { return wavy ? s.sin_v[ey * n2 + k] : 0.0; };
  const double su0 = wavy ? s.sin_ue[ex] : 0.0, su1 = wavy ? s.sin_ue[ex + 1] : 0.0;
  const double sv0 = wavy ? s.sin_ve[ey] : 0.0, sv1 = wavy ? s.sin_ve[ey + 1] : 0.0;
  const Pt S = curve(s, u0, v0, u1, v0, xi, SU(i), sv0);
  const Pt Nn = curve(s, u0, v1, u1, v1, xi, SU(i), sv1);
  const Pt W = curve(s, u0, v0, u0, v1, eta, su0, SV(j));
  const Pt E = curve(s, u1, v0, u1, v1, eta, su1, SV(j));
  const Pt sw = curve(s, u0, v0, u1, v0, -1.0, SU(n1), sv0);
  const Pt se = curve(s, u0, v0, u1, v0, 1.0, SU(n1 + 1), sv0);
  const Pt nw = curve(s, u0, v1, u1, v1, -1.0, SU(n1), sv1);
  const Pt ne = curve(s, u0, v1, u1, v1, 1.0, SU(n1 + 1), sv1);
  const double a00 = 0.25 * (1.0 - xi) * (1.0 - eta), a10 = 0.25 * (1.0 + xi) * (1.0 - eta);
  const double a01 = 0.25 * (1.0 - xi) * (1.0 + eta), a11 = 0.25 * (1.0 + xi) * (1.0 + eta);
  x[n] = 0.5 * (1.0 - eta) * S.x + 0.5 * (1.0 + eta) * Nn.x + 0.5 * (1.0 - xi) * W.x +
         0.5 * (1.0 + xi) * E.x - (a00 * sw.x + a10 * se.x + a01 * nw.x + a11 * ne.x);
  y[n] = 0.5 * (1.0 - eta) * S.y + 0.5 * (1.0 + eta) * Nn.y + 0.5 * (1.0 - xi) * W.y +
         0.5 * (1.0 + xi) * E.y - (a00 * sw.y + a10 * se.y + a01 * nw.y + a11 * ne.y);
}

// compute_metrics nodal part (mesh.hpp:163-190) + sample_bathymetry (223-232)
// + the compute_dt lengths (timeloop.hpp:62-65)
__global__ void k_metrics(MeshSpecDev s, const double* D, int n1, long long nn, const double* x,
                          const double* y, MeshOut o) {
  const long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (n >= nn) return;
  const int np = n1 * n1;
  const int loc = (int)(n % np), i = loc / n1, j = loc % n1;
  const long long base = n - loc;
  double xxi = 0.0, xeta = 0.0, yxi = 0.0, yeta = 0.0;
  for (int m = 0; m < n1; ++m) {
    const double dxi = D[i * n1 + m], deta = D[j * n1 + m];
    xxi += dxi * x[base + m * n1 + j];
    yxi += dxi * y[base + m * n1 + j];
    xeta += deta * x[base + i * n1 + m];
    yeta += deta * y[base + i * n1 + m];
  }
  const double jac = xxi * yeta - xeta * yxi;
  o.x_xi[n] = xxi;
  o.x_eta[n] = xeta;
  o.y_xi[n] = yxi;
  o.y_eta[n] = yeta;
  o.jac[n] = jac;
  if (!bathy_needs_libm(s.bathy_kind)) o.b[n] = bathymetry(s, x[n], y[n]);
  if (!(jac > 0.0)) atomicExch(o.bad_jac, 1);
}

}  // namespace

int launch_structured_mesh(const MeshSpecDev& s, const double* nodes, const double* D, int n1,
                           const MeshOut& o, cudaStream_t st) {
  const long long nn = s.n_elem * n1 * n1;
  k_coords<<<(unsigned)((nn + 255) / 256), 256, 0, st>>>(s, nodes, n1, nn, o.x, o.y);
  k_metrics<<<(unsigned)((nn + 255) / 256), 256, 0, st>>>(s, D, n1, nn, o.x, o.y, o);
  return 2;
}

}  // namespace swdg_dev
