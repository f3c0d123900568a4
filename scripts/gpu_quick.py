"""Ad-hoc GPU bring-up check (numerics vs scipy on exported operators)."""
import sys, time, numpy as np, scipy.sparse as sp, scipy.sparse.linalg as spl
sys.path.insert(0, '.')
from paper_2512_19536_b200.simulation import SimulationConfig, Simulation

def precond_ref(P, K, r):
    own = P.owner("subdomain"); b = P.n_local
    z = np.zeros_like(r)
    for s in range(own.max() + 1):
        cells = np.nonzero(own == s)[0]
        dofs = (cells[:, None] * b + np.arange(b)).ravel()
        Ki = K[dofs][:, dofs].tocsc()
        z[dofs] = spl.spsolve(Ki, r[dofs])
    if P.coarse_dim:
        E = P.export("E"); K0 = (E.T @ K @ E).tocsc()
        z += E @ spl.spsolve(K0, E.T @ r)
    return z

rng = np.random.default_rng(0)
for kw in [dict(cells=64, degree=1), dict(cells=256, degree=2, subdomains=8, coarse=-1),
           dict(cells=1024, degree=1, lloyd=5, subdomains=16, coarse=-1),
           dict(cells=2048, degree=3, lloyd=5, subdomains=16, coarse=-1, fiber_random=True),
           dict(cells=512, degree=1, precond="none"), dict(cells=512, degree=2, precond="block-jacobi")]:
    t = time.time(); sim = Simulation(SimulationConfig(**kw)); t1 = time.time() - t
    P = sim.problem; K = P.export("K"); n = sim.dimension
    x = rng.uniform(-1, 1, n)
    y = sim.apply_K(x); e1 = abs(y - K @ x).max() / abs(K @ x).max()
    r = rng.uniform(-1, 1, n)
    z = sim.apply_precond(r); zr = precond_ref(P, K, r) if kw.get("precond", "two-level") != "none" else r
    e2 = abs(z - zr).max() / abs(zr).max()
    xs, rep = sim.pcg_solve(r, 1e-10)
    xr = spl.spsolve(K.tocsc(), r); e3 = abs(xs - xr).max() / abs(xr).max()
    print(kw, f"create {t1:.2f}s spmv {e1:.1e} precond {e2:.1e} pcg it={rep.iterations} conv={rep.converged} err {e3:.1e} kappa={rep.condition_estimate}")
    st = [sim.step() for _ in range(3)]
    print("   steps", [(s.iterations, s.converged, round(s.step_ms, 3)) for s in st])
