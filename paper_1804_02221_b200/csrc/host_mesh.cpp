// host_mesh.cpp — host-side inputs for standalone use (bench, tests without the
// reference headers): the 1D LGL operators and the structured face lists.
//
// Operators follow operators.hpp:57-188 operation for operation (Newton on
// (1-x^2)L'_N with Chebyshev-Lobatto guesses, the closed-form LGL derivative,
// Dtilde = 2D + S, Dhat = -M^-1 D^T M, the Gauss-projection V^-1), so they
// are bitwise the reference's when compiled without FP contraction.  The face
// list is MeshTopology::faces in structured_topology's order (mesh.hpp:237-290).
#include <cmath>
#include <vector>

#include "../../include/swdg_gpu.h"
#include "swdg_host.h"

namespace {

// Legendre L_n and L_n' by the three-term recurrence (operators.hpp:10-28)
void legendre(int n, double x, double& l, double& dl) {
  double p0 = 1.0, d0 = 0.0;
  if (n == 0) {
    l = p0;
    dl = d0;
    return;
  }
  double p1 = x, d1 = 1.0;
  for (int k = 1; k < n; ++k) {
    const double p2 = ((2 * k + 1) * x * p1 - k * p0) / (k + 1);
    const double d2 = d0 + (2 * k + 1) * p1;
    p0 = p1;
    d0 = d1;
    p1 = p2;
    d1 = d2;
  }
  l = p1;
  dl = d1;
}

}  // namespace

extern "C" int swdg_operators(int degree, double* nodes, double* weights, double* deriv,
                              double* deriv_modified, double* deriv_weak, double* vand,
                              double* vand_inv) {
  if (degree < 1 || degree > 15) return SWDG_ERR_INPUT;
  const int n1 = degree + 1;
  const double nn1 = static_cast<double>(degree) * (degree + 1);
  // LGL nodes/weights
  nodes[0] = -1.0;
  nodes[degree] = 1.0;
  for (int j = 1; j < degree; ++j) {
    double x = -std::cos(M_PI * j / degree);
    for (int it = 0; it < 100; ++it) {
      double l, dl;
      legendre(degree, x, l, dl);
      const double dx = (1.0 - x * x) * dl / (nn1 * l);
      x += dx;
      if (std::abs(dx) < 1e-15) break;
    }
    nodes[j] = x;
  }
  std::vector<double> lN(n1);
  for (int j = 0; j < n1; ++j) {
    double l, dl;
    legendre(degree, nodes[j], l, dl);
    lN[j] = l;
    weights[j] = 2.0 / (nn1 * l * l);
  }
  // closed-form derivative matrix
  for (int i = 0; i < n1; ++i)
    for (int j = 0; j < n1; ++j)
      deriv[i * n1 + j] = i != j ? lN[i] / (lN[j] * (nodes[i] - nodes[j])) : 0.0;
  deriv[0] = -0.25 * degree * (degree + 1);
  deriv[n1 * n1 - 1] = 0.25 * degree * (degree + 1);
  for (int i = 0; i < n1; ++i)
    for (int j = 0; j < n1; ++j) {
      deriv_modified[i * n1 + j] = 2.0 * deriv[i * n1 + j];
      deriv_weak[i * n1 + j] = -deriv[j * n1 + i] * weights[j] / weights[i];
    }
  deriv_modified[0] += 1.0 / weights[0];
  deriv_modified[n1 * n1 - 1] -= 1.0 / weights[degree];
  // Gauss nodes/weights for the modal projection
  std::vector<double> gx(n1), gw(n1);
  for (int j = 0; j < n1; ++j) {
    double x = -std::cos(M_PI * (2 * j + 1) / (2.0 * n1));
    for (int it = 0; it < 100; ++it) {
      double l, dl;
      legendre(n1, x, l, dl);
      const double dx = -l / dl;
      x += dx;
      if (std::abs(dx) < 1e-15) break;
    }
    gx[j] = x;
    double l, dl;
    legendre(n1, x, l, dl);
    gw[j] = 2.0 / ((1.0 - x * x) * dl * dl);
  }
  for (int i = 0; i < n1; ++i)
    for (int j = 0; j < n1; ++j) {
      double l, dl;
      legendre(j, nodes[i], l, dl);
      vand[i * n1 + j] = l * std::sqrt(j + 0.5);
      vand_inv[i * n1 + j] = 0.0;
    }
  std::vector<double> lag(n1), wb(n1);
  for (int q = 0; q < n1; ++q) {
    // Lagrange basis at the Gauss node (barycentric, operators.hpp:126-146)
    const double x = gx[q];
    int hit = -1;
    for (int j = 0; j < n1; ++j)
      if (hit < 0 && std::abs(x - nodes[j]) < 1e-14) hit = j;
    if (hit >= 0) {
      for (int j = 0; j < n1; ++j) lag[j] = j == hit ? 1.0 : 0.0;
    } else {
      for (int i = 0; i < n1; ++i) {
        wb[i] = 1.0;
        for (int k = 0; k < n1; ++k)
          if (k != i) wb[i] *= nodes[i] - nodes[k];
      }
      double denom = 0.0;
      for (int j = 0; j < n1; ++j) {
        lag[j] = 1.0 / (wb[j] * (x - nodes[j]));
        denom += lag[j];
      }
      for (int j = 0; j < n1; ++j) lag[j] /= denom;
    }
    for (int i = 0; i < n1; ++i) {
      double li, dli;
      legendre(i, x, li, dli);
      for (int j = 0; j < n1; ++j) vand_inv[i * n1 + j] += std::sqrt(i + 0.5) * li * lag[j] * gw[q];
    }
  }
  return SWDG_OK;
}

namespace swdg_host {

// structured_topology (mesh.hpp:237-290): per element east face (+west wall on
// the first column), north face (+south wall on the first row).
std::vector<swdg_face> structured_faces(int kx, int ky, bool px, bool py) {
  std::vector<swdg_face> faces;
  faces.reserve(2 * (size_t)kx * ky + kx + ky);
  auto eid = [&](int ex, int ey) { return ey * kx + ex; };
  for (int ey = 0; ey < ky; ++ey)
    for (int ex = 0; ex < kx; ++ex) {
      swdg_face f{eid(ex, ey), 1, -1, -1, 0, SWDG_TAG_INTERIOR};
      if (ex + 1 < kx) {
        f.elem_plus = eid(ex + 1, ey);
        f.face_plus = 3;
      } else if (px) {
        f.elem_plus = eid(0, ey);
        f.face_plus = 3;
      } else {
        f.tag = SWDG_TAG_WALL;
      }
      faces.push_back(f);
      if (ex == 0 && !px) faces.push_back(swdg_face{eid(ex, ey), 3, -1, -1, 0, SWDG_TAG_WALL});
      swdg_face g{eid(ex, ey), 2, -1, -1, 0, SWDG_TAG_INTERIOR};
      if (ey + 1 < ky) {
        g.elem_plus = eid(ex, ey + 1);
        g.face_plus = 0;
      } else if (py) {
        g.elem_plus = eid(ex, 0);
        g.face_plus = 0;
      } else {
        g.tag = SWDG_TAG_WALL;
      }
      faces.push_back(g);
      if (ey == 0 && !py) faces.push_back(swdg_face{eid(ex, ey), 0, -1, -1, 0, SWDG_TAG_WALL});
    }
  return faces;
}

}  // namespace swdg_host

extern "C" int64_t swdg_structured_face_count(int kx, int ky, int px, int py) {
  return (int64_t)swdg_host::structured_faces(kx, ky, px != 0, py != 0).size();
}

extern "C" int swdg_structured_faces(int kx, int ky, int px, int py, swdg_face* out) {
  const auto f = swdg_host::structured_faces(kx, ky, px != 0, py != 0);
  for (size_t i = 0; i < f.size(); ++i) out[i] = f[i];
  return SWDG_OK;
}
