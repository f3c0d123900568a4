// Barreto-Cressman membrane + ion-concentration kinetics (ext).
//
// The reference registers "barreto-cressman" as an IonicModel slot but ships no
// kinetics (/root/reference/proj/src/ionics.cpp:52-57); the paper
// defers to Cressman et al. 2009 (J Comput Neurosci 26:159-170), whose published
// equations are restated here in the reference's IonicModel convention
// (ionics.hpp:18-31): current() is the outward membrane current density in
// uA/cm^2 and rates() returns m with dy/dt = -m. State y = (n, h, [K]o, [Na]i).
//
//   I    = g_Na m_inf^3 h (u - E_Na) + g_NaL (u - E_Na)          (I_Na)
//        + g_K n^4 (u - E_K) + g_KL (u - E_K)                    (I_K)
//        + g_ClL (u - E_Cl)
//   dn/dt = phi (a_n (1 - n) - b_n n),  dh/dt = phi (a_h (1 - h) - b_h h)
//   d[K]o/dt  = (gamma beta I_K - 2 beta I_pump - I_glia - I_diff) / tau
//   d[Na]i/dt = (-gamma I_Na - 3 I_pump) / tau
//   I_pump = rho / (1 + exp((25 - [Na]i)/3)) / (1 + exp(5.5 - [K]o))
//   I_glia = G_glia / (1 + exp((18 - [K]o)/2.5)),  I_diff = eps ([K]o - k_bath)
//   [K]i = K_i0 + (Na_i0 - [Na]i),  [Na]o = Na_o0 - beta ([Na]i - Na_i0)
//   E_X = RTF ln(out/in), E_Cl = RTF ln(Cl_i/Cl_o)
//
// One definition serves the device kernel (kernels.cu) and the host rest-state
// solve (problem.cpp); the oracle restates it independently
// (oracle/src/discretization.cpp).
#pragma once

#include <cmath>

#include "../../../include/polydg_b200.h"

#ifdef __CUDACC__
#define PDG_HD __host__ __device__ __forceinline__
#else
#define PDG_HD inline
#endif

namespace pdg::bc {

// x / (1 - exp(-x)), continuous through x = 0
PDG_HD double xexp(double x) { return x == 0.0 ? 1.0 : x / -expm1(-x); }

PDG_HD void gating_rates(double u, double& an, double& bn, double& ah, double& bh) {
  an = 0.1 * xexp(0.1 * (u + 34.0));
  bn = 0.125 * exp(-(u + 44.0) / 80.0);
  ah = 0.07 * exp(-(u + 44.0) / 20.0);
  bh = 1.0 / (1.0 + exp(-0.1 * (u + 14.0)));
}

// sodium and potassium membrane currents (outward positive); returns I_Na + I_K + I_Cl
PDG_HD double membrane(const double* P, double u, const double* y, double& ina, double& ik) {
  const double am = xexp(0.1 * (u + 30.0));
  const double bm = 4.0 * exp(-(u + 55.0) / 18.0);
  const double minf = am / (am + bm);
  const double ki = P[PDG_BC_K_I0] + (P[PDG_BC_NA_I0] - y[3]);
  const double nao = P[PDG_BC_NA_O0] - P[PDG_BC_BETA] * (y[3] - P[PDG_BC_NA_I0]);
  const double ena = P[PDG_BC_RTF] * log(nao / y[3]);
  const double ek = P[PDG_BC_RTF] * log(y[2] / ki);
  const double ecl = P[PDG_BC_RTF] * log(P[PDG_BC_CL_I] / P[PDG_BC_CL_O]);
  const double n2 = y[0] * y[0];
  ina = (P[PDG_BC_G_NA] * (minf * minf * minf) * y[1] + P[PDG_BC_G_NAL]) * (u - ena);
  ik = (P[PDG_BC_G_K] * (n2 * n2) + P[PDG_BC_G_KL]) * (u - ek);
  return ina + ik + P[PDG_BC_G_CLL] * (u - ecl);
}

PDG_HD double current(const double* P, double u, const double* y) {
  double ina, ik;
  return P[PDG_BC_AMP] * membrane(P, u, y, ina, ik);
}

PDG_HD void rates(const double* P, double u, const double* y, double* m) {
  double an, bn, ah, bh, ina, ik;
  gating_rates(u, an, bn, ah, bh);
  membrane(P, u, y, ina, ik);
  const double pump = P[PDG_BC_RHO] / (1.0 + exp((25.0 - y[3]) / 3.0)) / (1.0 + exp(5.5 - y[2]));
  const double glia = P[PDG_BC_G_GLIA] / (1.0 + exp((18.0 - y[2]) / 2.5));
  const double diff = P[PDG_BC_EPS] * (y[2] - P[PDG_BC_K_BATH]);
  const double beta = P[PDG_BC_BETA], tau = P[PDG_BC_TAU];
  m[0] = -P[PDG_BC_PHI] * (an * (1.0 - y[0]) - bn * y[0]);
  m[1] = -P[PDG_BC_PHI] * (ah * (1.0 - y[1]) - bh * y[1]);
  m[2] = -(P[PDG_BC_GAMMA] * beta * ik - 2.0 * beta * pump - glia - diff) / tau;
  m[3] = -(-P[PDG_BC_GAMMA] * ina - 3.0 * pump) / tau;
}

// admissible potential range for the out-of-range diagnostic (ionics.hpp:33-35)
constexpr double kUMin = -100.0, kUMax = 60.0;

}  // namespace pdg::bc
