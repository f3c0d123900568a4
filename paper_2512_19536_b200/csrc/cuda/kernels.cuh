// Launch wrappers for the sm_100a kernels (kernels.cu). All FP64; the whole
// per-step path is HBM-bound, so the kernels are organised around one
// coalesced pass over each operand.
#pragma once

#include "common.cuh"

namespace pdg {

struct PcgHist {
  double* resid;
  double* alpha;
  double* beta;
};

// What the last CTA does with a grid-wide deterministic sum.
enum Finish : int {
  kFinNone = 0,
  kFinPq = 1,      // S->pq = sum
  kFinDenom = 2,   // S->denom = sqrt(sum); zero -> converged with 0 iterations
  kFinRr = 3,      // residual history, iteration count, convergence
  kFinRzInit = 4,  // first rho with breakdown checks
  kFinRz = 5,      // rho_next, beta, maxit
  kFinStore = 6,   // *out = sum
  kFinAccum = 7,   // *out += sum (a second partial added in a fixed order)
};

struct ReduceCtx {
  Reducer red;
  PcgScalars* S;
  PcgHist H;
  double* out;  // kFinStore target
  int finish;
};

// y = K x (+ grid dot with `dotw`), BSR rows [0, rows), or the `rows` block
// rows listed in `rowlist` (multi-rank: interior rows while the halo is in
// flight, then the rows that read it). Early-exits when S->stop.
void launch_spmv(int b, int rows, const int* ptr, const int* col, const double* val,
                 const double* x, double* y, const double* dotw, ReduceCtx rc, bool honor_stop,
                 cudaStream_t st, const int* rowlist = nullptr);
// r = bvec - K x ; x untouched ; sum r.r -> kFinDenom
void launch_residual(int b, int rows, const int* ptr, const int* col, const double* val,
                     const double* x, const double* bvec, double* r, ReduceCtx rc, cudaStream_t st);
// CN right-hand side and the warm-started residual in one pass over K:
//   KU = K U ; rhs = 2 a M U - KU + ion ; x = warm ? U : 0 ; r = rhs - (warm ? KU : 0)
void launch_rhs(int b, int rows, const int* ptr, const int* col, const double* val,
                const double* M, double two_a, const double* U, const double* ion, int warm,
                double* rhs, double* x, double* r, ReduceCtx rc, cudaStream_t st);
// alpha = rho/pq ; x += alpha p ; r -= alpha q ; sum r.r -> kFinRr
void launch_update(long long n, double* x, double* r, const double* p, const double* q,
                   ReduceCtx rc, cudaStream_t st);
// p = z + beta p  (beta from S) ; or p = z when first
void launch_pupdate(long long n, double* p, const double* z, PcgScalars* S, bool first,
                    cudaStream_t st);
// z += E y0 (coarse prolongation, optional) ; sum r.z -> kFinRzInit / kFinRz
void launch_prolong_dot(int b, int bq, int ncells, const double* E, const int* cell_agg,
                        const double* y0, const double* r, double* z, ReduceCtx rc,
                        cudaStream_t st);
// r0 = E^T r per coarse node
void launch_restrict(int b, int bq, int n_agg, const int* agg_ptr, const int* agg_cells,
                     const double* E, const double* r, double* r0, const PcgScalars* S,
                     cudaStream_t st);

// update_kernel fused with the restriction: per chunk of <= 64 cells of one
// agglomerate, x += alpha p, r -= alpha q, r0part[chunk] = E^T r (chunk cells)
void launch_update_restrict(int b, int bq, int n_chunks, const int* chunk_ptr, const int* cells, const double* E,
                            double* x, double* r, const double* p, const double* q, double* r0part, ReduceCtx rc,
                            cudaStream_t st);

// the same two coarse-space steps when every chunk is a run of consecutive
// cells: the chunk's E blocks are brought into shared memory by one bulk copy
void launch_update_restrict_tma(int b, int bq, int n_chunks, int max_chunk_cells, const int* chunk_ptr,
                                const int* cells, const double* E, double* x, double* r, const double* p,
                                const double* q, double* r0part, ReduceCtx rc, cudaStream_t st);
void launch_prolong_dot_tma(int b, int bq, int n_chunks, int max_chunk_cells, const int* chunk_ptr, const int* cells,
                            const int* cell_agg, const double* E, const double* y0, const double* r, double* z,
                            ReduceCtx rc, cudaStream_t st);

// r0 chunk partials -> r0 (one CTA-sized chunk of an agglomerate per restrict CTA)
void launch_restrict_combine(int bq, int n_agg, const int* node_chunk_ptr, const double* part, double* r0,
                             const PcgScalars* S, cudaStream_t st);

// One launch runs the forward units (tickets [0, n_units_f)) then the
// backward units; counters: flags[task] forward, flags[n_tasks + task] backward.
struct SweepArgs {
  const DevTask* tasks;
  const DevUnit* units;   // ticket order (topological): forward units, then backward units
  int n_units_f, n_units;
  int n_tasks;
  unsigned int* ticket;
  int* flags;             // tiles completed: [fwd n_tasks | bwd n_tasks]
  int* tile_ctr;          // chunks completed per split tile
  double* part;           // 32 partial sums per column chunk
  const int* task_child;
  const double* fmat;
  const double* hmat;
  const DevTile* ftiles;
  const DevTile* htiles;
  const long long* row_dof;
  const int* in_ptr;
  const long long* in_idx;
  double* ubuf;
  const double* r;
  double* z;
  const double* r0;
  double* y0;
  double* yf;             // forward results y_S (fine / coarse), read by the backward units
  double* yc;
  const double* r0part;   // non-null: the coarse forward sums r0 from the restriction chunks
  const int* node_chunk_ptr;
  // level chunks of the bottom supernodes (host/problem.hpp LevelChunk): records, forward publish list
  // {root task, its forward tiles}, backward wait list {counter, count}
  const int* bmeta;
  const int2* broots;
  const int2* bdeps;
  const PcgScalars* S;
  int* epoch;        // [0] sweep number (counters wait for (epoch+1) * count), [1] CTAs finished
  int xcap;          // doubles per unit input buffer
  unsigned long long* live;  // [0] start of this launch (CTA 0), [1] summed launch ns, [2] launches
  long long* trace;  // optional: 4 globaltimer stamps per unit (start, deps met, gathered, done)
  int prefetch;      // 1: L2 bulk prefetch of each unit's panel when it starts (PDG_SWEEP_PREFETCH)
  int threads;       // CTA size: 128, or 64 for large problems with small blocks (sim.cu)
};
void launch_sweep(const SweepArgs& a, int smem_bytes, cudaStream_t st);

// Device assembly (assemble.cu): volume terms, faces, K, M^-1, U0/Y0, E, K0.
struct AsmArgs {
  int ncells, cell0, b, p, q, bq, n_comp, ngl, ngs, init_kind, two_level;
  const double* bbox;     // 4 per cell (internal order; world 1: all cells)
  const int* tri_ptr;
  const double* tri;      // fan triangles, 6 doubles each
  const double *glx, *glw, *gsx, *gsw;  // triangle-rule / segment-rule Gauss nodes
  const double* sigma;    // 4 per cell (t00 t01 t10 t11)
  const int* fptr;        // per local cell: its faces in face order
  const int* fent;        // 2 f + side
  const int* fcell;       // (K, L) per face, internal cell ids
  const double* fgeo;     // mid.x mid.y dir.x dir.y half n.x n.y eta per face
  const int *kptr, *kcol;
  double* kval;
  double *M, *Minv, *U0, *Y0;
  double am, hb;          // K = am M + hb A
  double u_rest, u_patch, omega0[2], omega0_r2, ip[4], y_rest[4];
  const double* abox;     // coarse label -> bbox
  const int* cell_label;  // local cell -> coarse label
  const int* cell_agg;    // local cell -> coarse internal node
  const int *agg_ptr, *agg_cells;
  double* E;
  const int *k0ptr, *k0col;
  double* k0val;
  int* err;               // bit 0: mass block not SPD, bit 1: E mass not SPD
};
void launch_assembly(const AsmArgs& a, cudaStream_t st);
void launch_k0(const AsmArgs& a, int n_agg, cudaStream_t st);

// Ionic model + stimulus at quadrature nodes (one warp per cell).
struct IonicArgs {
  int b, p, ncells, n_comp, ngl, has_prev, model, stim;
  const double* bbox;
  const int* tri_ptr;
  const double* tri;
  const double* U;
  const double* Up;
  const double* Y;    // n_comp fields of n (current)
  const double* Yp;   // previous
  double* Ynext;      // Y - dt M^-1 G
  const double* Minv;
  double* ion;        // -chi dt I* + dt F
  long long n;
  double chi, dt, t_mid;
  double fhn[8];
  double bc[PDG_BC_NPARAM];  // Barreto-Cressman parameters (bc_model.hpp)
  double ubounds[2];         // admissible potential range of the model (diagnostic only)
  double stim_p[4];
  int* flags;         // bit0 out-of-range warning, bit1 non-finite state
};
void set_gauss_nodes(const double* x, const double* w, int n);
void launch_ionic(const IonicArgs& a, cudaStream_t st);
// per-cell means of U over the order-2p+2 rule (snapshot.cpp:13-28)
void launch_cell_means(int p, int ncells, int ngl, const double* bbox, const int* tri_ptr, const double* tri,
                       const double* U, const double* area, double* out, cudaStream_t st);

// multi-rank helpers: apply a finish to an all-reduced sum; pack halo cells
void launch_finish(ReduceCtx rc, const double* sum, bool honor, cudaStream_t st);
void launch_pack(const double* v, const int* cells, int ncells, int b, double* out, cudaStream_t st);

// dst_int[i*b + r] = src_ref[perm[i]*b + r] and the inverse
void launch_gather_perm(const double* src, double* dst, const int* perm, int ncells, int b, int nfields,
                        long long stride_src, long long stride_dst, cudaStream_t st);
void launch_scatter_perm(const double* src, double* dst, const int* perm, int ncells, int b, int nfields,
                         long long stride_src, long long stride_dst, cudaStream_t st);

}  // namespace pdg
