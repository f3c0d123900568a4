// TEST INFRASTRUCTURE ONLY — CPU parity oracle and timed CPU baseline.
//
// An Eigen-free restatement of the reference's numeric path
// (/root/reference/proj/src/{dg_space,quadrature,assembly,ionics,krylov,
// schwarz,timestepper}.cpp). Pinned two ways: by the reference's own unit and
// acceptance assertions (tests/test_oracle_pins.py), and by the reference's
// numeric sources themselves, compiled in oracle/_ref against a small Eigen
// API stand-in (oracle/eigen_shim; Eigen3 is absent here): M/A/K/E agree
// bitwise, and acceptance criteria 2/3/7/8/9, config 1 and the default
// Simulation match the goldens that build produced (tests/golden/
// reference_numeric.json, tests/test_reference_numeric.py). The mesh half is
// pinned by the reference's compiled mesh sources (oracle/_ref). Only tests/,
// smoke() and bench.py's cpu_baseline / reference legs load it; the product
// never links it.
//
// Deliberately independent of the product code: its own quadrature, basis,
// assembly (triplets summed in insertion order like Eigen's setFromTriplets),
// exact local solvers (its own minimum-degree block Cholesky; the product
// packs supernodal factors for the GPU sweep), PCG loop and a QL tridiagonal
// eigensolver for the Lanczos estimate (the product uses bisection).
//
// Barreto-Cressman (ionic == 2): PARITY UNPINNED against the reference, which
// ships no kinetics (ionics.cpp:52-57). bc_current / bc_rates / model_rest
// restate Cressman et al. 2009 independently of the product's bc_model.hpp and
// are cross-checked against a numpy restatement (tests/test_barreto_cressman.py).
#pragma once

#include <cmath>
#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

namespace orc {

struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct SolverError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct P2 {
  double x = 0, y = 0;
};
inline P2 operator+(P2 a, P2 b) { return {a.x + b.x, a.y + b.y}; }
inline P2 operator-(P2 a, P2 b) { return {a.x - b.x, a.y - b.y}; }
inline P2 operator*(P2 a, double s) { return {a.x * s, a.y * s}; }
inline double cross(P2 a, P2 b) { return a.x * b.y - a.y * b.x; }

struct Box {
  double x0, y0, x1, y1;
  double w() const { return x1 - x0; }
  double h() const { return y1 - y0; }
};

using Vec = std::vector<double>;

// ---- threading: the reference's fork/join parallel_for (parallel.cpp:23-41) ----
int thread_count();
void parallel_for(std::size_t n, const std::function<void(std::size_t)>& fn);

// ---- operator threading and memory (large parity runs) ----
// set_parallel_ops(true): row-parallel Csr::apply (same bits; default off =
// single-threaded like Eigen's SpMV). set_lean(1): Discretization drops M and
// A after building K and K_rhs; set_lean(2): K only (one-solve workloads).
void set_parallel_ops(bool on);
void set_lean(int level);

// ---- scalar CSR matrix ----
struct Csr {
  int64_t rows = 0, cols = 0;
  std::vector<int64_t> ptr{0};
  std::vector<int64_t> idx;
  std::vector<double> val;
  void apply(const Vec& x, Vec& y) const;  // single-threaded like Eigen's SpMV
  double at(int64_t r, int64_t c) const;
};
struct Triplet {
  int64_t r, c;
  double v;
};
Csr from_triplets(int64_t rows, int64_t cols, std::vector<Triplet>& t);
Csr transpose(const Csr& A);
Csr multiply(const Csr& A, const Csr& B);
Csr combine(const Csr& A, double a, const Csr& B, double b);  // a*A + b*B

// ---- quadrature / basis (quadrature.cpp, dg_space.cpp) ----
struct Rule {
  std::vector<P2> pts;
  Vec w;
};
void gauss_legendre(int n, Vec& x, Vec& w);
Rule polygon_rule(const std::vector<P2>& poly, int order);
Rule segment_rule(P2 a, P2 b, int order);
int n_modes(int p);
// values/grads at points: n_pts x n_loc row-major
void eval_basis(const Box& box, int p, const std::vector<P2>& pts, Vec& val, Vec* gx, Vec* gy);

// ---- mesh view (topology restated from mesh.cpp:17-106) ----
struct Face {
  P2 a, b, n;
  int in = -1, out = -1;
  double len = 0;
};
struct MeshView {
  std::vector<P2> verts;
  std::vector<int> off, idx;
  std::vector<uint8_t> region;  // 0 grey, 1 white
  std::vector<Face> faces;      // interior only
  std::vector<double> diam;
  std::vector<Box> bbox;
  int n_cells() const { return static_cast<int>(region.size()); }
  double mesh_size() const;  // max cell diameter (mesh.cpp:40-47)
  std::vector<P2> cell(int c) const;
  void build();
};

struct Config {
  int degree = 1;
  double eta0 = 10, chi_m = 1000, C_m = 1, dt = 2.5e-3, T = 10;
  double sgl = 6.3, sgn = 6.3, swl = 6.9, swn = 25.71;
  P2 fiber_grey{0, 1}, fiber_white{0, 1};
  int fiber_random = 0;
  uint64_t fiber_seed = 42;
  int ionic = 1;  // 0 none, 1 fhn, 2 barreto-cressman (ext, unpinned)
  double fhn[8] = {0.13, 0.013, 0.26, 0.1, 1.0, -85.0, 20.0, 1.0};
  // g_Na g_K g_NaL g_KL g_ClL phi rho G_glia eps k_bath gamma beta tau RT/F Cl_i Cl_o Na_i0 K_i0 Na_o0 amp
  double bc[20] = {100, 40, 0.0175, 0.05, 0.05, 3, 1.25, 66, 1.2, 4, 0.0445, 7, 1000, 26.64, 6, 130, 18, 140, 144, 1};
  int init_kind = 0;
  double u_rest = -67, u_patch = -50;
  P2 omega0{0.5, 1.0};
  double omega0_r2 = 0.016;
  double init_params[4] = {0, 0, 0, 0};
  int stim_kind = 0;
  double stim_params[4] = {0, 0, 0, 0};
  double tol = 1e-9;
  int maxit = 0;
  int warm_start = 1;
  int precond = 2;  // 0 none, 1 block-jacobi, 2 two-level
  int q = 0;
};

// ---- assembly (assembly.cpp) ----
struct Discretization {
  const MeshView* mesh;
  int p, nloc;
  Csr M, A, K, Krhs;
  std::vector<Vec> Mchol;  // per-cell dense Cholesky factor (row-major lower)
  void build(const MeshView& m, const Config& c);
  Vec mass_solve(const Vec& rhs) const;
  Vec l2_project(const std::function<double(P2)>& g) const;
};

// ---- snapshot.cpp:13-28 ----
Vec cell_means(const Discretization& D, const Vec& U);
// ---- dg_space.cpp:94-115 ----
double l2_error(const Discretization& D, const Vec& U, const std::function<double(P2)>& g);

// ---- ionics (ionics.cpp:20-113) ----
double fhn_current(const double* prm, double u, double w);
double fhn_rate(const double* prm, double u, double w);
struct IonicTerms {
  Vec I;
  std::vector<Vec> G;
};
// Barreto-Cressman (ext): Cressman et al. 2009 kinetics in the IonicModel
// convention (dy/dt = -m), state (n, h, [K]o, [Na]i); parity unpinned (the
// reference ships no kinetics, ionics.cpp:52-57)
double bc_current(const double* prm, double u, const double* y);
void bc_rates(const double* prm, double u, const double* y, double* m);
// resting_potential / resting_state (ionics.hpp:29-30); returns state_dim
int model_rest(const Config& c, double* u, double* y);
IonicTerms ionic_terms(const Discretization& D, const Vec& U, const std::vector<Vec>& Y,
                       const Config& cfg, bool* out_of_box);

// ---- linear algebra: operators, PCG, Lanczos (krylov.cpp) ----
struct Operator {
  int64_t n;
  std::function<void(const Vec&, Vec&)> apply;
};
struct PcgReport {
  int iterations = 0;
  bool converged = false;
  Vec resid, alpha, beta;
  bool has_cond = false;
  double cond = 0;
};
int default_max_iterations(int64_t n);
Vec pcg(const Operator& K, const Vec& b, const Operator* P, double tol, int maxit, const Vec& x0,
        PcgReport& rep);
bool condition_estimate(const Vec& alpha, const Vec& beta, double* kappa);

// ---- exact local / coarse solver: minimum-degree block Cholesky (blockchol.cpp) ----
struct BlockChol {
  int nb = 0, b = 1;
  std::vector<int> perm;         // new -> old block
  std::vector<int64_t> colptr;   // block column j: rows rowidx[colptr[j]..colptr[j+1]), first = j
  std::vector<int> rowidx;
  Vec L;                         // b x b row-major blocks, aligned with rowidx
  void factor(const Csr& A, int block);  // throws SolverError
  void solve(Vec& x) const;              // in place, original numbering
  int64_t blocks() const { return colptr.empty() ? 0 : colptr.back(); }
};

// ---- Schwarz (schwarz.cpp) ----
struct Schwarz {
  int64_t n = 0;
  std::vector<std::vector<int64_t>> dofs;
  std::vector<BlockChol> local;
  bool two_level = false;
  Csr E, Et, K0;
  BlockChol coarse;
  void build(const Csr& K, const Discretization& D, const std::vector<int>& sub_owner, int n_sub,
             const std::vector<int>& coarse_owner, int n_coarse, int q);
  void apply(const Vec& r, Vec& z) const;
};
Csr coarse_embedding(const Discretization& D, const std::vector<int>& owner, int count, int q);

// ---- time stepper (timestepper.cpp) ----
struct StepStats {
  int iterations = 0;
  double final_residual = 0;
  bool converged = false;
  bool has_cond = false;
  double cond = 0;
};
struct Simulation {
  Config cfg;
  MeshView mesh;
  Discretization D;
  Schwarz S;
  bool has_precond = false;
  int k = 0;
  double t = 0;
  Vec U, Up;
  std::vector<Vec> Y, Yp;
  void build(const Config& c, MeshView m, const std::vector<int>& sub_owner, int n_sub,
             const std::vector<int>& coarse_owner, int n_coarse);
  StepStats step();
  Vec external_term(double t_mid) const;
  double initial(P2 x) const;
};

}  // namespace orc
