"""Synthetic SPD operators shaped like the paper's workloads (BASELINE.json configs).

The paper measures on Antarctica first-order-Stokes matrices from Albany
(§5); those matrices are not available,
so these seeded generators stand in for them, taking their *shape*: thin
extruded domains, 2 DOF per node, strong vertical vs weak horizontal coupling
(the model problem of P:68) and near-singular basal regions.
The recipes are stated in DESIGN.md ("Input recipe") and SURVEY.md §8(d).

Every generator returns a `Problem`: CSR with BOTH triangles stored
(int64 rowptr, int32 colind, float64 vals, sorted columns per row),
coordinates (n x d float64), an optional extruded `column_id` (int32) and the
right-hand side b ~ N(0,1) drawn with numpy PCG64 seed 0 in the ORIGINAL
ordering.  Nothing here implements any step of the hierarchical method.
"""
from __future__ import annotations

import dataclasses
import numpy as np

RHS_SEED = 0          # b = default_rng(0).standard_normal(N)
FIELD_SEED = 1        # g (C2, C3)
MU_SEED = 2           # g_mu (C4, C5)
BETA_SEED = 3         # g_beta (C4, C5)


@dataclasses.dataclass
class Problem:
    name: str
    n: int
    rowptr: np.ndarray          # int64 [n+1]
    colind: np.ndarray          # int32 [nnz]
    vals: np.ndarray            # float64 [nnz]
    coords: np.ndarray          # float64 [n, d]
    column_id: np.ndarray | None  # int32 [n] or None
    b: np.ndarray               # float64 [n]
    # solver parameters the config names (BASELINE.json configs[*])
    leaf_size: int = 0          # DOFs per leaf when column_id is None
    leaf_columns: int = 0       # columns per leaf when column_id is given
    eps: float = 1e-2
    tol: float = 1e-8
    meta: dict = dataclasses.field(default_factory=dict)

    @property
    def nnz(self) -> int:
        return int(self.colind.shape[0])

    def to_scipy(self):
        import scipy.sparse as sp
        return sp.csr_matrix((self.vals, self.colind, self.rowptr), shape=(self.n, self.n))


def rhs(n: int, seed: int = RHS_SEED) -> np.ndarray:
    return np.random.default_rng(seed).standard_normal(n)


# ----------------------------------------------------------------------------
# Gaussian random field (SURVEY.md §8(d) "GRF recipe")
# ----------------------------------------------------------------------------
def grf(shape, ell: float, sigma: float, seed: int) -> np.ndarray:
    """White noise on a grid padded 2x per axis, circularly convolved with
    exp(-|x|^2/ell^2), cropped, normalised to mean 0 / std 1, times sigma."""
    shape = tuple(int(s) for s in shape)
    pad = tuple(2 * s for s in shape)
    rng = np.random.default_rng(seed)
    xi = rng.standard_normal(pad)
    d2 = np.zeros(pad)
    for ax, p in enumerate(pad):
        x = np.arange(p, dtype=np.float64)
        x = np.minimum(x, p - x)                 # circular distance
        sh = [1] * len(pad)
        sh[ax] = p
        d2 = d2 + (x * x).reshape(sh)
    ker = np.exp(-d2 / (ell * ell))
    axes = list(range(len(pad)))
    f = np.fft.irfftn(np.fft.rfftn(xi, axes=axes) * np.fft.rfftn(ker, axes=axes), s=pad, axes=axes)
    f = f[tuple(slice(0, s) for s in shape)]
    f = (f - f.mean()) / f.std()
    return sigma * f


# ----------------------------------------------------------------------------
# structured-stencil CSR assembly helper
# ----------------------------------------------------------------------------
def _stencil_csr(dims, entries):
    """dims = (nx, ny, nz) nodes (x fastest: idx = i + nx*(j + ny*k)).
    entries: list of ((dx,dy,dz), values[nz,ny,nx]) — A[idx, idx+delta] = values[idx].
    Entries outside the grid are dropped.  Returns rowptr, colind, vals with
    columns sorted ascending in every row (stencil sorted by linear offset)."""
    nx, ny, nz = dims
    n = nx * ny * nz
    k, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    lin = lambda d: d[0] + nx * (d[1] + ny * d[2])
    entries = sorted(entries, key=lambda e: lin(e[0]))
    S = len(entries)
    cols = np.empty((n, S), dtype=np.int64)
    vals = np.empty((n, S), dtype=np.float64)
    mask = np.empty((n, S), dtype=bool)
    base = (i + nx * (j + ny * k)).reshape(-1)
    for t, (d, v) in enumerate(entries):
        ok = ((i + d[0] >= 0) & (i + d[0] < nx) & (j + d[1] >= 0) & (j + d[1] < ny)
              & (k + d[2] >= 0) & (k + d[2] < nz))
        mask[:, t] = ok.reshape(-1)
        cols[:, t] = base + lin(d)
        vals[:, t] = np.broadcast_to(v, (nz, ny, nx)).reshape(-1)
    counts = mask.sum(axis=1)
    rowptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=rowptr[1:])
    return rowptr, cols[mask].astype(np.int32), vals[mask]


def _harm(a, b):
    return 2.0 * a * b / (a + b)


# ----------------------------------------------------------------------------
# C1: 2-D Poisson 5-point, Dirichlet eliminated (BASELINE configs[0])
# ----------------------------------------------------------------------------
def gen_poisson2d(nx: int = 32, ny: int | None = None, aniso: float = 1.0,
                  leaf_size: int = 16, eps: float = 1e-2, tol: float = 1e-10) -> Problem:
    """eps_a*u_xx + u_yy model of P:68 (aniso = eps_a; C1 uses 1): diagonal
    2*aniso + 2, off-diagonals -aniso (x) and -1 (y); h^2 dropped.
    Coordinates (i, j), index i + nx*j."""
    ny = nx if ny is None else ny
    one = np.ones((1, ny, nx))
    ent = [((0, 0, 0), (2.0 * aniso + 2.0) * one),
           ((-1, 0, 0), -aniso * one), ((1, 0, 0), -aniso * one),
           ((0, -1, 0), -1.0 * one), ((0, 1, 0), -1.0 * one)]
    rowptr, colind, vals = _stencil_csr((nx, ny, 1), ent)
    n = nx * ny
    j, i = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
    coords = np.stack([i.reshape(-1), j.reshape(-1)], axis=1).astype(np.float64)
    return Problem(f"poisson2d_{nx}x{ny}", n, rowptr, colind, vals, coords, None, rhs(n),
                   leaf_size=leaf_size, eps=eps, tol=tol, meta={"nx": nx, "ny": ny, "aniso": aniso})


# ----------------------------------------------------------------------------
# C2: 3-D cell-centred 7-point FV, k = exp(g), Dirichlet on all faces
# ----------------------------------------------------------------------------
def gen_laplace3d(nc: int = 64, sigma: float = 1.0, ell: float = 8.0, leaf_size: int = 64,
                  eps: float = 1e-2, tol: float = 1e-8, field_seed: int = FIELD_SEED) -> Problem:
    """k = exp(g), g a GRF (sigma, ell); face transmissibility = harmonic mean;
    Dirichlet boundary term 2*k_c on every boundary face.  sigma=0 gives k=1."""
    if sigma > 0:
        g = grf((nc, nc, nc), ell, 1.0, field_seed) * sigma   # axes (z, y, x)
        kf = np.exp(g)
    else:
        kf = np.ones((nc, nc, nc))
    diag = np.zeros_like(kf)
    ent = []
    for ax, (dx, dy, dz) in enumerate([(1, 0, 0), (0, 1, 0), (0, 0, 1)]):
        axis = 2 - ax                             # numpy axis for x/y/z
        sl_lo = [slice(None)] * 3
        sl_hi = [slice(None)] * 3
        sl_lo[axis] = slice(0, nc - 1)
        sl_hi[axis] = slice(1, nc)
        T = _harm(kf[tuple(sl_lo)], kf[tuple(sl_hi)])
        up = np.zeros_like(kf)
        dn = np.zeros_like(kf)
        up[tuple(sl_lo)] = -T                      # A[c, c+e]
        dn[tuple(sl_hi)] = -T                      # A[c+e, c]
        diag[tuple(sl_lo)] += T
        diag[tuple(sl_hi)] += T
        # Dirichlet faces: 2 k_c on the two boundary layers of this axis
        b0 = [slice(None)] * 3
        b1 = [slice(None)] * 3
        b0[axis] = 0
        b1[axis] = nc - 1
        diag[tuple(b0)] += 2.0 * kf[tuple(b0)]
        diag[tuple(b1)] += 2.0 * kf[tuple(b1)]
        ent.append(((dx, dy, dz), up))
        ent.append(((-dx, -dy, -dz), dn))
    ent.append(((0, 0, 0), diag))
    rowptr, colind, vals = _stencil_csr((nc, nc, nc), ent)
    n = nc ** 3
    k, j, i = np.meshgrid(np.arange(nc), np.arange(nc), np.arange(nc), indexing="ij")
    coords = np.stack([i.reshape(-1), j.reshape(-1), k.reshape(-1)], axis=1).astype(np.float64)
    return Problem(f"laplace3d_{nc}", n, rowptr, colind, vals, coords, None, rhs(n),
                   leaf_size=leaf_size, eps=eps, tol=tol,
                   meta={"nc": nc, "sigma": sigma, "ell": ell})


# ----------------------------------------------------------------------------
# C3: thin anisotropic slab, whole vertical columns
# ----------------------------------------------------------------------------
def gen_slab(nh: int = 256, nl: int = 10, ratio: float = 1e4, sigma: float = 2.0,
             ell: float = 8.0, leaf_columns: int = 8, eps: float = 1e-2, tol: float = 1e-8,
             field_seed: int = FIELD_SEED) -> Problem:
    """7-point FV on nh x nh x nl cells; T_h = harmonic-mean k, T_v = k*ratio
    ((1 km / 10 m)^2 = 1e4); k(x,y) = exp(sigma*g2D) constant per column;
    Dirichlet on the bottom face (2 T_v), Neumann elsewhere.  Coordinates in
    metres (x = 1000 i, y = 1000 j, z = 10 k); column_id = i + nh*j."""
    if sigma > 0:
        g = grf((nh, nh), ell, 1.0, field_seed) * sigma    # axes (y, x)
        k2 = np.exp(g)
    else:
        k2 = np.ones((nh, nh))
    kf = np.broadcast_to(k2, (nl, nh, nh)).copy()
    diag = np.zeros_like(kf)
    ent = []
    for (dx, dy, dz), axis, scale in [((1, 0, 0), 2, 1.0), ((0, 1, 0), 1, 1.0), ((0, 0, 1), 0, ratio)]:
        n_ax = kf.shape[axis]
        sl_lo = [slice(None)] * 3
        sl_hi = [slice(None)] * 3
        sl_lo[axis] = slice(0, n_ax - 1)
        sl_hi[axis] = slice(1, n_ax)
        T = scale * _harm(kf[tuple(sl_lo)], kf[tuple(sl_hi)])
        up = np.zeros_like(kf)
        dn = np.zeros_like(kf)
        up[tuple(sl_lo)] = -T
        dn[tuple(sl_hi)] = -T
        diag[tuple(sl_lo)] += T
        diag[tuple(sl_hi)] += T
        ent.append(((dx, dy, dz), up))
        ent.append(((-dx, -dy, -dz), dn))
    diag[0] += 2.0 * ratio * kf[0]                 # Dirichlet bottom face
    ent.append(((0, 0, 0), diag))
    rowptr, colind, vals = _stencil_csr((nh, nh, nl), ent)
    n = nh * nh * nl
    k, j, i = np.meshgrid(np.arange(nl), np.arange(nh), np.arange(nh), indexing="ij")
    coords = np.stack([1000.0 * i.reshape(-1), 1000.0 * j.reshape(-1), 10.0 * k.reshape(-1)], axis=1)
    column_id = (i + nh * j).reshape(-1).astype(np.int32)
    return Problem(f"slab_{nh}x{nh}x{nl}", n, rowptr, colind, vals, coords, column_id, rhs(n),
                   leaf_columns=leaf_columns, eps=eps, tol=tol,
                   meta={"nh": nh, "nl": nl, "ratio": ratio, "sigma": sigma})


# ----------------------------------------------------------------------------
# C4/C5: Q1 hexahedral FE of the frozen-viscosity first-order-Stokes form
# ----------------------------------------------------------------------------
def _q1_reference(hx, hy, hz):
    """16x16 element matrix of the first-order-Stokes form (mu = 1) and the
    4x4 basal-face mass matrix (beta = 1).  Form (strain-rate typo
    fixed per SURVEY Q15):  a(u,v) = int 2mu[(2u1x+u2y)v1x + exy v1y + 1/2 u1z v1z
    + exy v2x + (u1x+2u2y)v2y + 1/2 u2z v2z],  exy = 1/2(u1y+u2x).
    Local node a = (ax, ay, az) -> a = ax + 2ay + 4az; local DOF = 2a + c."""
    gp = np.array([-1.0, 1.0]) / np.sqrt(3.0)
    K = np.zeros((16, 16))
    nodes = [(ax, ay, az) for az in (0, 1) for ay in (0, 1) for ax in (0, 1)]
    w = (hx * hy * hz) / 8.0          # Gauss weights 1 on [-1,1]^3 times detJ
    for gx in gp:
        for gy in gp:
            for gz in gp:
                xi = [(1 + gx) / 2, (1 + gy) / 2, (1 + gz) / 2]   # in [0,1]
                N = np.zeros(8)
                dN = np.zeros((8, 3))
                for a, (ax, ay, az) in enumerate(nodes):
                    fx = xi[0] if ax else 1 - xi[0]
                    fy = xi[1] if ay else 1 - xi[1]
                    fz = xi[2] if az else 1 - xi[2]
                    sx = 1.0 if ax else -1.0
                    sy = 1.0 if ay else -1.0
                    sz = 1.0 if az else -1.0
                    N[a] = fx * fy * fz
                    dN[a] = [sx * fy * fz / hx, fx * sy * fz / hy, fx * fy * sz / hz]
                for a in range(8):
                    ax_, ay_, az_ = dN[a]
                    for b in range(8):
                        bx, by, bz = dN[b]
                        K[2 * a, 2 * b] += w * 2 * (2 * bx * ax_ + 0.5 * by * ay_ + 0.5 * bz * az_)
                        K[2 * a, 2 * b + 1] += w * 2 * (by * ax_ + 0.5 * bx * ay_)
                        K[2 * a + 1, 2 * b] += w * 2 * (0.5 * by * ax_ + bx * ay_)
                        K[2 * a + 1, 2 * b + 1] += w * 2 * (0.5 * bx * ax_ + 2 * by * ay_ + 0.5 * bz * az_)
    M = np.zeros((4, 4))
    wf = (hx * hy) / 4.0
    fn = [(ax, ay) for ay in (0, 1) for ax in (0, 1)]
    for gx in gp:
        for gy in gp:
            xi = [(1 + gx) / 2, (1 + gy) / 2]
            N = np.array([(xi[0] if ax else 1 - xi[0]) * (xi[1] if ay else 1 - xi[1]) for ax, ay in fn])
            M += wf * np.outer(N, N)
    return K, M


def gen_stokes_q1(nx: int = 512, ny: int | None = None, nz: int = 20, aspect: float = 1e3,
                  sigma_mu: float = 2.0, sigma_beta: float = 3.0, ell: float = 8.0,
                  leaf_columns: int = 2, eps: float = 1e-2, tol: float = 1e-8) -> Problem:
    """Q1 hex FE, nx x ny x nz NODES, 2 velocity DOF per node (DOF = 2*node + c,
    node = i + nx*(j + ny*k)).  hx = hy = 1, H = (nx-1)/aspect, hz = H/(nz-1).
    mu = exp(sigma_mu*g_mu) per element column; beta = beta0*exp(sigma_beta*g_beta)
    per basal face with beta0 = median(mu)/H (Robin condition P:767-773; lateral
    and top boundaries natural).  column_id = i + nx*j for both DOFs of a node."""
    ny = nx if ny is None else ny
    ex, ey, ez = nx - 1, ny - 1, nz - 1
    hx = hy = 1.0
    H = (nx - 1) / aspect
    hz = H / ez
    Kref, Mref = _q1_reference(hx, hy, hz)
    mu2 = np.exp(grf((ey, ex), ell, 1.0, MU_SEED) * sigma_mu) if sigma_mu > 0 else np.ones((ey, ex))
    bt2 = np.exp(grf((ey, ex), ell, 1.0, BETA_SEED) * sigma_beta) if sigma_beta > 0 else np.ones((ey, ex))
    beta = (np.median(mu2) / H) * bt2
    # values V[(delta, c, c')] on the node grid (nz, ny, nx)
    loc = [(ax, ay, az) for az in (0, 1) for ay in (0, 1) for ax in (0, 1)]
    V = {}
    for a, (ax, ay, az) in enumerate(loc):
        for b, (bx, by, bz) in enumerate(loc):
            d = (bx - ax, by - ay, bz - az)
            for c in (0, 1):
                for c2 in (0, 1):
                    key = (d, c, c2)
                    if key not in V:
                        V[key] = np.zeros((nz, ny, nx))
                    kv = Kref[2 * a + c, 2 * b + c2]
                    if kv != 0.0:
                        V[key][az:az + ez, ay:ay + ey, ax:ax + ex] += kv * mu2[None, :, :]
    floc = [(ax, ay) for ay in (0, 1) for ax in (0, 1)]
    for a, (ax, ay) in enumerate(floc):
        for b, (bx, by) in enumerate(floc):
            d = (bx - ax, by - ay, 0)
            for c in (0, 1):
                V[(d, c, c)][0, ay:ay + ey, ax:ax + ex] += Mref[a, b] * beta
    # CSR over DOFs: row (node, c); columns (node+d, c') sorted by (lin(d), c')
    deltas = sorted({k[0] for k in V}, key=lambda d: d[0] + nx * (d[1] + ny * d[2]))
    nn = nx * ny * nz
    n = 2 * nn
    k, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    base = (i + nx * (j + ny * k)).reshape(-1)
    S = 2 * len(deltas)
    rowptr = np.zeros(n + 1, dtype=np.int64)
    okm = np.empty((nn, len(deltas)), dtype=bool)
    for t, d in enumerate(deltas):
        okm[:, t] = ((i + d[0] >= 0) & (i + d[0] < nx) & (j + d[1] >= 0) & (j + d[1] < ny)
                     & (k + d[2] >= 0) & (k + d[2] < nz)).reshape(-1)
    cnt_node = okm.sum(axis=1) * 2                    # entries per DOF row
    counts = np.repeat(cnt_node, 2)
    np.cumsum(counts, out=rowptr[1:])
    nnz = int(rowptr[-1])
    colind = np.empty(nnz, dtype=np.int32)
    vals = np.empty(nnz, dtype=np.float64)
    # fill row by row component: position of entry (t, c2) within its row
    pos_in_row = np.cumsum(np.repeat(okm, 2, axis=1), axis=1) - 1   # [nn, S]
    for c in (0, 1):
        rstart = rowptr[2 * np.arange(nn) + c]
        for t, d in enumerate(deltas):
            ok = okm[:, t]
            lin = d[0] + nx * (d[1] + ny * d[2])
            for c2 in (0, 1):
                col = t * 2 + c2
                dst = rstart[ok] + pos_in_row[ok, col]
                colind[dst] = (2 * (base[ok] + lin) + c2).astype(np.int32)
                vals[dst] = V[(d, c, c2)].reshape(-1)[ok]
    coords_n = np.stack([hx * i.reshape(-1), hy * j.reshape(-1), hz * k.reshape(-1)], axis=1)
    coords = np.repeat(coords_n, 2, axis=0)
    column_id = np.repeat((i + nx * j).reshape(-1), 2).astype(np.int32)
    return Problem(f"stokes_q1_{nx}x{ny}x{nz}", n, rowptr, colind, vals, coords, column_id, rhs(n),
                   leaf_columns=leaf_columns, eps=eps, tol=tol,
                   meta={"nx": nx, "ny": ny, "nz": nz, "aspect": aspect, "H": H})


# ----------------------------------------------------------------------------
# the BASELINE.json configs
# ----------------------------------------------------------------------------
CONFIGS = {
    # configs[0]: 2D Poisson 32x32, leaf 16, eps 1e-2, PCG 1e-10
    "C1": lambda **kw: gen_poisson2d(32, **kw),
    # configs[1]: 3D 64^3, k=exp(g) sigma=1 ell=8, leaf 64, eps 1e-2 (and 1e-4), PCG 1e-8
    "C2": lambda **kw: gen_laplace3d(64, **kw),
    # configs[2]: 256x256x10 slab, ratio 1e4, lognormal sigma 2, column leaves (8 columns)
    "C3": lambda **kw: gen_slab(256, 10, **kw),
    # configs[3]: Q1 first-order-Stokes 512x512x20 nodes x 2 DOF
    "C4": lambda **kw: gen_stokes_q1(512, 512, 20, aspect=1e3, **{"leaf_columns": 2, **kw}),
    # configs[4]: 1024x1024x16 nodes x 2 DOF, aspect 1e4
    "C5": lambda **kw: gen_stokes_q1(1024, 1024, 16, aspect=1e4, **{"leaf_columns": 4, **kw}),
}


def gen_config(name: str, **kw) -> Problem:
    return CONFIGS[name](**kw)


def gen_config_scaled(name: str, scale: int) -> Problem:
    """The config's operator on a horizontally reduced grid (1/scale per horizontal axis);
    used for proxies of C4/C5 that fit quick runs (same layers, leaf, eps, tol, fields)."""
    if name == "C4":
        return gen_stokes_q1(512 // scale, 512 // scale, 20, aspect=1e3, leaf_columns=2)
    if name == "C5":
        return gen_stokes_q1(1024 // scale, 1024 // scale, 16, aspect=1e4, leaf_columns=4)
    if name == "C3":
        return gen_slab(256 // scale, 10)
    if name == "C2":
        return gen_laplace3d(64 // scale)
    raise KeyError(name)


def gen_family(layers: int, level: int, base: int = 32) -> Problem:
    """NEXT f2: weak-scaling family of the config-4 operator at a fixed number of element
    layers (the paper's 6- and 11-layer Antarctica families, Tables `ilu` / `10layers`,
    P:920-1007): (base 2^level)^2 horizontal nodes x (layers + 1) node layers x 2 DOF;
    each level has 4x the DOFs of the previous one.  Same fields, leaf (2 columns), eps,
    tol and domain aspect ratio as C4."""
    n = base << level
    return gen_stokes_q1(n, n, layers + 1, aspect=1e3, leaf_columns=2)

