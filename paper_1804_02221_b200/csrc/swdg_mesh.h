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
};

struct MeshOut {
  double *x, *y, *x_xi, *x_eta, *y_xi, *y_eta, *jac, *b, *len_xi, *len_eta;
  double *fnx, *fny, *fjs, *fa;
  int* bad_jac;
};

int launch_structured_mesh(const MeshSpecDev& s, const double* nodes, const double* D, int n1,
                           const MeshOut& o, cudaStream_t st);

}  // namespace swdg_dev
