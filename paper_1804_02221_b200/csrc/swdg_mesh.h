// swdg_mesh.h — device mesh generation interface (kernels_mesh.cu).
#pragma once

#include <cuda_runtime.h>

namespace swdg_dev {

struct MeshSpecDev {
  int kind, kx, ky, bathy_kind;
  double x0, x1, y0, y1, extra;
  double bathy[4];
  const int* gid;  // local -> global element id (partitions), nullptr = identity
  long long n_elem;  // elements generated
  // wavy map: the host's sin(2 pi u) of every u the edge curves sample
  // (mesh.hpp:370-379), so the coordinates are bitwise the reference's:
  // sin_u[ex * (n1 + 2) + k] at u = u0 + t_k (u1 - u0), k < n1 the LGL nodes,
  // k = n1, n1 + 1 the corners t = 0, 1; sin_ue[ex] at u = ex / kx.  Same for v.
  const double *sin_u, *sin_ue, *sin_v, *sin_ve;
};

// bathymetry kinds whose closure calls libm: sampled on the host (glibc), like the
// reference, from the device coordinates
__host__ __device__ inline bool bathy_needs_libm(int kind) { return kind == 4 || kind == 6; }

struct MeshOut {
  double *x, *y, *x_xi, *x_eta, *y_xi, *y_eta, *jac, *b, *len_xi, *len_eta;
  double *fnx, *fny, *fjs, *fa;
  int* bad_jac;
};

// coordinates, metrics, J and the polynomial bathymetries on the device (no
// FMA, no libm: bitwise the reference); the libm-dependent fields (CFL lengths
// and face arrays via hypot, sine bathymetries) are finished by the host
int launch_structured_mesh(const MeshSpecDev& s, const double* nodes, const double* D, int n1,
                           const MeshOut& o, cudaStream_t st);

}  // namespace swdg_dev
