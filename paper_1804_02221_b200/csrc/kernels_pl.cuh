// kernels_pl.cuh — instantiations of the P-part line stage kernel (stage_pl.cuh)
// for the degrees [PL_N1_LO, PL_N1_HI]; included by kernels_pl_{a,b,c}.cu so the
// three ranges compile in parallel.
#include <cstdlib>

#include "fast_common.cuh"

namespace swdg_dev {
namespace {

#include "stage_pl.cuh"

// parts per line, elements per group and register cap per degree; ALT > 0 are
// experimental alternatives selected at run time with SWDG_PL_ALT
template <int N1, int ALT = 0>
struct PLCfg {
  static constexpr int P = ALT == 1 && N1 == 16 ? 2 : N1 <= 4 ? 1 : N1 <= 8 ? 2 : N1 <= 12 ? 3 : 4;
  static constexpr int E0 = N1 == 2 ? 32 : N1 == 3 ? 16 : N1 == 4 ? 16 : N1 <= 7 ? 8 : N1 == 8 ? 4
                          : N1 <= 12 ? 4 : N1 <= 15 ? 2 : 1;
  static constexpr int E = ALT == 1 && N1 < 16 ? (E0 > 1 ? E0 / 2 : 1) : E0;
  static constexpr int REG = ALT == 2 ? 128 : 0;
  static constexpr int MINB = REG == 0 ? 1
                            : (65536 / REG) / PLP<N1, P, E>::THREADS > 0
                                  ? (65536 / REG) / PLP<N1, P, E>::THREADS : 1;
};

template <int N1, int ALT, bool FORCE>
void launch_pl(const Mesh& M, const Phys& P, const StageArgs& A, Flags* F, cudaStream_t st) {
  using C = PLCfg<N1, ALT>;
  using PL = PLP<N1, C::P, C::E>;
  static int cache = 0;
  auto kern = k_stage_pl<N1, C::P, C::E, C::MINB, FORCE>;
  const int grid = grid_for(kern, PL::THREADS, PL::bytes, (M.n_owned - M.e_lo + PL::E - 1) / PL::E, cache);
  kern<<<grid, PL::THREADS, PL::bytes, st>>>(M, P, A, F);
}

inline int pl_alt() {
  static int v = -1;
  if (v < 0) {
    const char* s = getenv("SWDG_PL_ALT");
    v = s ? atoi(s) : 0;
  }
  return v;
}

// experimental alternatives are instantiated for a few degrees only
template <int N1>
constexpr bool kPlAlts = N1 == 8 || N1 == 13 || N1 == 16;

template <int N1>
bool launch_pl_range(const Mesh& M, const Phys& P, const StageArgs& A, Flags* F,
                     cudaStream_t st) {
  if constexpr (N1 > PL_N1_HI) {
    return false;
  } else {
    if (M.n1 != N1) return launch_pl_range<N1 + 1>(M, P, A, F, st);
    const int alt = pl_alt();
    if constexpr (kPlAlts<N1>) {
      if (alt == 1) {
        if (A.fh) launch_pl<N1, 1, true>(M, P, A, F, st);
        else launch_pl<N1, 1, false>(M, P, A, F, st);
        return true;
      }
      if (alt == 2) {
        if (A.fh) launch_pl<N1, 2, true>(M, P, A, F, st);
        else launch_pl<N1, 2, false>(M, P, A, F, st);
        return true;
      }
    }
    if (A.fh) launch_pl<N1, 0, true>(M, P, A, F, st);
    else launch_pl<N1, 0, false>(M, P, A, F, st);
    return true;
  }
}

}  // namespace

int PL_UPLOAD(int base, const double* tab, int len) { return upload_ops_local(base, tab, len); }

int PL_LAUNCH(const Mesh& M, const Phys& P, const StageArgs& A, Flags* F, cudaStream_t st) {
  return launch_pl_range<PL_N1_LO>(M, P, A, F, st) ? 1 : 0;
}

}  // namespace swdg_dev
