/* oracle/swdg_port.h — TEST INFRASTRUCTURE ONLY (parity checker, never the product).
 *
 * Plain-C restatement of the reference's per-stage path (swdg, arXiv 1804.02221),
 * written from the reference's math, face-major scatter structure and
 * expression trees, compiled without FP contraction so it is bitwise equal to
 * the reference built at its own flags.  Every function cites the reference
 * lines it restates.  Pinned against oracle/_ref (the compiled reference) and
 * the golden fixtures in tests/golden.
 *
 * Mesh input is the product's C-ABI mesh view (include/swdg_gpu.h) so the
 * same borrowed arrays feed the checker and the device path.  Elements at or
 * beyond n_owned (halo copies in partitioned runs) are read but never
 * limited/updated by port_post_stage.
 */
#ifndef SWDG_PORT_H
#define SWDG_PORT_H

#include <stdint.h>

#include "../include/swdg_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

/* error text of the last failing call (thread-unsafe, test use only) */
const char* port_last_error(void);

/* assemble_rhs (dg_rhs.hpp:267-303), entropy-stable mode, optional viscous
 * momentum terms (NULL = inviscid) and nodal forcing (NULL = none). */
int port_assemble_rhs(const swdg_mesh_view* m, const swdg_params* p, const double* h,
                      const double* hu, const double* hv, const double* visc_hu,
                      const double* visc_hv, const double* f_h, const double* f_hu,
                      const double* f_hv, double* rh, double* rhu, double* rhv);

/* shock_indicator (viscosity.hpp:35-65) on one element field. */
double port_shock_indicator(int degree, const double* vinv, const double* field, int* err);
/* viscosity_coefficient (viscosity.hpp:69-78) */
double port_viscosity_coefficient(double sigma, const swdg_params* p, int* err);
/* compute_viscosity (viscosity.hpp:250-259) over elements [0, n_elem) */
int port_compute_viscosity(const swdg_mesh_view* m, const swdg_params* p, const double* h,
                           double* eps);
/* velocity loop of evaluate_rhs (timeloop.hpp:183-185) */
void port_velocities(const swdg_mesh_view* m, const swdg_params* p, const double* h,
                     const double* hu, const double* hv, double* u, double* v);
/* br1_gradients (viscosity.hpp:95-168) */
int port_br1_gradients(const swdg_mesh_view* m, const double* u, const double* v, double* u1,
                       double* u2, double* v1, double* v2);
/* viscous flux pairs of viscous_lhs (viscosity.hpp:187-194) */
int port_viscous_fluxes(const swdg_mesh_view* m, const double* h, const double* u1,
                        const double* u2, const double* v1, const double* v2, const double* eps,
                        double* fvu, double* fvv, double* gvu, double* gvv);
/* rest of viscous_lhs (viscosity.hpp:195-246) from the flux pairs */
int port_viscous_lhs(const swdg_mesh_view* m, const double* fvu, const double* fvv,
                     const double* gvu, const double* gvv, double* out_hu, double* out_hv);

/* TimeIntegrator::evaluate_rhs (timeloop.hpp:173-190).  eps (n_elem) is
 * written when viscosity is on; forcing arrays may be NULL. */
int port_evaluate_rhs(const swdg_mesh_view* m, const swdg_params* p, const double* h,
                      const double* hu, const double* hv, const double* f_h,
                      const double* f_hu, const double* f_hv, double* rh, double* rhu,
                      double* rhv, double* eps);

/* element_average (limiter.hpp:24-37) */
void port_element_average(const swdg_mesh_view* m, const double* h, const double* hu,
                          const double* hv, int e, double* avg3, double* area);
/* limit_element (limiter.hpp:43-84); returns theta, *err on a negative mean */
double port_limit_element(const swdg_mesh_view* m, const swdg_params* p, double* h, double* hu,
                          double* hv, int e, int zero_dry, int* err);

/* post_stage (timeloop.hpp:202-234) over owned elements.  Returns 1 accept,
 * 0 reject, -1 NumericalAbort (limiter off and a negative node). */
int port_post_stage(const swdg_mesh_view* m, const swdg_params* p, double* h, double* hu,
                    double* hv, int* n_limited, double* min_stage_h);

/* Forcing kinds for try_step: 0 none; 1 the traveling wave of
 * validate.hpp:543-556 with fparams = (h0, amp, u0, v0, k, g). */
int port_try_step(const swdg_mesh_view* m, const swdg_params* p, double* h, double* hu,
                  double* hv, double t, double dt, int forcing_kind, const double* fparams,
                  swdg_step_info* info);

/* compute_dt (timeloop.hpp:53-75) */
int port_compute_dt(const swdg_mesh_view* m, const swdg_params* p, const double* h,
                    const double* hu, const double* hv, double cfl, double* dt);
/* total_mass / total_entropy / min_height (field.hpp:39-68) and
 * min_positivity_dt (limiter.hpp:135-166) */
int port_diagnostics(const swdg_mesh_view* m, const swdg_params* p, const double* h,
                     const double* hu, const double* hv, swdg_diagnostics* out);

/* es_surface_flux_normal (fluxes.hpp:136-166) for flux-level goldens */
int port_es_flux(const double* wm, const double* wp, double bm, double bp, double nx,
                 double ny, double g, double h_des, double* out3);

#ifdef __cplusplus
}
#endif
#endif
