// swdg_device.cuh — device-side data layout and helpers shared by the stage kernels.
//
// Layout in HBM (one context = one GPU = one element partition):
//   nodal arrays      double[K*np], element-major e*np + i*n1 + j  (core.hpp:39-42)
//   face arrays       double[K*4*n1], (e*4+face)*n1 + t            (mesh.hpp:70-75)
//   element faces     int4[K*4]: {neighbour element, info bits, global face ordinal, 0}
//                     built once on the host from MeshTopology::faces (mesh.hpp:46-54)
// Elements [0, n_owned) are advanced; [n_owned, K) are halo copies (multi-GPU).
#pragma once

#include <cstdint>

namespace swdg_dev {

// ---- element-face connectivity (host builds it, kernels read it) ----
// info bits
constexpr int EF_NBR_FACE_MASK = 3;   // neighbour's local face id
constexpr int EF_REVERSED = 1 << 2;   // plus-side nodes run opposite (mesh.hpp:51)
constexpr int EF_WALL = 1 << 3;       // BoundaryTag::wall
constexpr int EF_MINUS = 1 << 4;      // this element is the face owner (minus side)
constexpr int EF_PRESENT = 1 << 5;    // the face is in MeshTopology::faces

struct Phys {
  double g, h_tol, h_des, h_ref;
  double epsilon0, sigma_min, sigma_max;
  int visc, limiter;
  int standard;  // SchemeMode::standard (exact kernels only)
};

struct Mesh {
  // the stage kernels advance elements [e_lo, n_owned): e_lo = 0 normally, a
  // sub-range when a partition runs its interior and halo-adjacent elements as
  // separate launches (overlap with the halo exchange)
  int K, n_owned, n1, np, degree, e_lo;
  double w0;
  // Operators1D (operators.hpp:35-52), device copies
  const double *w, *D, *Dt, *Dh, *Vinv;
  // MeshGeometry nodal arrays
  const double *ye, *xe, *yx, *xx, *jac, *b;
  // exact-mode extras: host-computed CFL lengths (std::hypot) and face arrays
  const double *len_xi, *len_eta;
  const double *fnx, *fny, *fjs, *fa;
  const int4* ef;  // [K*4]
  // fast mode: geometry-only part of the split source (dg_rhs.hpp:171-176),
  // S_x = y_eta D_xi b + D_xi(y_eta b) - y_xi D_eta b - D_eta(y_xi b) and S_y
  // likewise, so the stage adds (g h / 2) (S_x, S_y)
  const double *sx, *sy;
};

struct State {
  double *h, *hu, *hv;
};

struct CState {
  const double *h, *hu, *hv;
};

// Reductions / signals for one stage or one step.  Keys are order-preserving
// encodings of doubles so atomicMin works on them (min is order-independent).
struct Flags {
  unsigned long long min_h_key;   // min node height after limiting
  unsigned long long dt_key;      // CFL candidate min
  unsigned long long minlen_key;  // all-dry fallback length
  unsigned long long posdt_key;   // positivity bound min (diagnostic)
  unsigned long long max_eps_key; // max viscosity coefficient (ordered, max via ~key min)
  int reject;                     // some element mean < 0 (timeloop.hpp:205-209)
  int abort;                      // limiter off and a node < 0 (timeloop.hpp:211-218)
  int n_limited;                  // elements with theta < 1 (last stage)
  int stage_reject;               // stage index of the first reject (+1), device-resident runs
};

__host__ __device__ inline unsigned long long order_key(double x) {
  const unsigned long long b = *reinterpret_cast<const unsigned long long*>(&x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__host__ __device__ inline double key_value(unsigned long long k) {
  const unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return *reinterpret_cast<const double*>(&b);
}

#ifdef __CUDACC__
// warp-level min of order keys: one atomic per warp instead of one per thread
// (min is exact and order-independent)
__device__ __forceinline__ unsigned long long warp_min_key(unsigned long long k) {
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long other = __shfl_xor_sync(0xffffffffu, k, o);
    k = other < k ? other : k;
  }
  return k;
}

// block-level min of order keys (blockDim.x a multiple of 32, <= 1024): valid in
// thread 0; one atomic per block instead of per warp (per-warp atomics on one
// address serialise: 2M of them cost compute_dt 3.7 ms at 1M elements, N=7)
__device__ __forceinline__ unsigned long long block_min_key(unsigned long long k) {
  __shared__ unsigned long long s_min[32];
  k = warp_min_key(k);
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();  // s_min reuse across calls
  if ((threadIdx.x & 31) == 0) s_min[w] = k;
  __syncthreads();
  if (w == 0) {
    k = (int)threadIdx.x < nw ? s_min[threadIdx.x] : ~0ull;
    k = warp_min_key(k);
  }
  return k;
}
#endif

// node (i,j) of local face `face` at position t (core.hpp:53-61)
__host__ __device__ inline int face_node(int n1, int face, int t) {
  switch (face) {
    case 0: return t * n1;             // south (t, 0)
    case 1: return (n1 - 1) * n1 + t;  // east  (N, t)
    case 2: return t * n1 + (n1 - 1);  // north (t, N)
    default: return t;                 // west  (0, t)
  }
}

// Faces touching node (i,j): up to two (corners).  Writes local face ids and
// the position t along each face.
__host__ __device__ inline int node_faces(int n1, int i, int j, int* face, int* t) {
  int c = 0;
  if (j == 0) { face[c] = 0; t[c] = i; ++c; }
  if (i == n1 - 1) { face[c] = 1; t[c] = j; ++c; }
  if (j == n1 - 1) { face[c] = 2; t[c] = i; ++c; }
  if (i == 0) { face[c] = 3; t[c] = j; ++c; }
  return c;
}

}  // namespace swdg_dev
