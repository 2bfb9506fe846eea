// kernels_mesh.cu — device generation of the structured curvilinear meshes
// (mesh.hpp:114-232, 294-379) straight into the context's geometry arrays, so
// the 1M-element throughput meshes never touch host memory.
// Same algorithm as the reference (transfinite blend of the four mapped edge
// curves sampled at LGL nodes, metrics by differentiating the nodal
// coordinate polynomials, normals/J_surf from the face metrics); FMA and CUDA
// libm make it agree with the host build to rounding, not bitwise — the
// parity tests use reference-built meshes.
#include <cuda_runtime.h>

#include "swdg_device.cuh"
#include "swdg_mesh.h"

namespace swdg_dev {
namespace {

struct Pt {
  double x, y;
};

__device__ Pt map_point(const MeshSpecDev& s, double u, double v) {
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
      const double w = sin(2.0 * M_PI * u) * sin(2.0 * M_PI * v);
      p.x = s.x0 + (u + s.extra * w) * (s.x1 - s.x0);
      p.y = s.y0 + (v - 0.75 * s.extra * w) * (s.y1 - s.y0);
      break;
    }
  }
  return p;
}

__device__ Pt curve(const MeshSpecDev& s, double u0, double v0, double u1, double v1, double r) {
  const double t = 0.5 * (1.0 + r);
  return map_point(s, u0 + t * (u1 - u0), v0 + t * (v1 - v0));
}

__device__ double bathymetry(const MeshSpecDev& s, double x, double y) {
  const double* p = s.bathy;
  switch (s.bathy_kind) {
    case 1: return p[0];
    case 2: return p[0] * x + p[1] * y + p[2];
    case 3: return p[0] * (x * x + y * y);
    case 4: return 0.1 + 0.05 * sin(2.0 * M_PI * x) * sin(2.0 * M_PI * y);
    case 5: return x < p[0] ? p[1] : p[2];
    case 6: return p[0] + p[1] * sin(p[2] * x) * sin(p[2] * y);
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
  const Pt S = curve(s, u0, v0, u1, v0, xi), Nn = curve(s, u0, v1, u1, v1, xi);
  const Pt W = curve(s, u0, v0, u0, v1, eta), E = curve(s, u1, v0, u1, v1, eta);
  const Pt sw = curve(s, u0, v0, u1, v0, -1.0), se = curve(s, u0, v0, u1, v0, 1.0);
  const Pt nw = curve(s, u0, v1, u1, v1, -1.0), ne = curve(s, u0, v1, u1, v1, 1.0);
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
  o.b[n] = bathymetry(s, x[n], y[n]);
  o.len_xi[n] = 2.0 * jac / hypot(xeta, yeta);
  o.len_eta[n] = 2.0 * jac / hypot(xxi, yxi);
  if (!(jac > 0.0)) atomicExch(o.bad_jac, 1);
}

// compute_metrics face part (mesh.hpp:192-218), one thread per face node
__global__ void k_faces(int n1, long long nfn, MeshOut o) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= nfn) return;
  const int t = (int)(idx % n1), face = (int)((idx / n1) % 4);
  const long long e = idx / (4 * n1);
  const long long n = e * n1 * n1 + face_node(n1, face, t);
  double js, nx, ny;
  if (face == 1 || face == 3) {
    js = hypot(o.y_eta[n], o.x_eta[n]);
    const double sg = face == 1 ? 1.0 : -1.0;
    nx = sg * o.y_eta[n] / js;
    ny = -sg * o.x_eta[n] / js;
  } else {
    js = hypot(o.y_xi[n], o.x_xi[n]);
    const double sg = face == 0 ? 1.0 : -1.0;
    nx = sg * o.y_xi[n] / js;
    ny = -sg * o.x_xi[n] / js;
  }
  o.fjs[idx] = js;
  o.fnx[idx] = nx;
  o.fny[idx] = ny;
  o.fa[idx] = o.jac[n] / js;
}

}  // namespace

int launch_structured_mesh(const MeshSpecDev& s, const double* nodes, const double* D, int n1,
                           const MeshOut& o, cudaStream_t st) {
  const long long nn = s.n_elem * n1 * n1;
  const long long nfn = s.n_elem * 4 * n1;
  k_coords<<<(unsigned)((nn + 255) / 256), 256, 0, st>>>(s, nodes, n1, nn, o.x, o.y);
  k_metrics<<<(unsigned)((nn + 255) / 256), 256, 0, st>>>(s, D, n1, nn, o.x, o.y, o);
  k_faces<<<(unsigned)((nfn + 255) / 256), 256, 0, st>>>(n1, nfn, o);
  return 3;
}

}  // namespace swdg_dev
