"""Distance-curve helpers (SPEC.md module ``curve``).

The hot-path estimator (power law on the measured prefix, segment radii) runs
on the device in K2 (csrc/sampler.cu); these host functions hold the O(n)
pieces that are fixed before launch -- the prefix length, the i**e table, the
segment positions and sampler boundaries -- and the user-facing full-curve
operations of the SPEC (``estimate_power``, ``segment_thresholds``,
``fit_power_exponent``), which share the exact definitions K2 evaluates:

* k0 = ceil(p * n)
* a  = (sum_{i=1}^{k0-1} v_i * i**e, summed in order) / (k0 - 1)
* est[i] = v[i] for i < k0; min(est[i-1], a / i**e) for i >= k0
                                                      
* d_s = min(floor(n s / nseg), n - 1), R_s = running min of est[d_s]
                                                      
* sampler boundaries = (d_1 .. d_{nseg-1}, n)
* R <= 0 -> 5e-324 and r2 = max(R*R, 5e-324)
"""

from __future__ import annotations

import math

import numpy as np

TINY = 5e-324


def prefix_len(n: int, p: float) -> int:
    if not (0.0 < p < 1.0):
        raise ValueError(f"p must be in (0, 1), got {p}")
    return int(math.ceil(p * n))


class FpsState:
    """Live FPS state after a prefix: float64 min-distances
    and the taken mask, reusable to continue the run (fps_loop k_start)."""

    def __init__(self, md, taken):
        self.md = md
        self.taken = taken


def extract_prefix(cloud, n: int, p: float = 0.1, seed_index: int = 0):
    """SPEC.md:238-246 on the device (K1 with k_stop = ceil(p n)) ->
    (prefix curve float64[k0] with [0] = +inf, FpsState, SampleResult of the
    k0 prefix indices)."""
    from . import core, engine

    pc = cloud if isinstance(cloud, core.PointCloud) else core.PointCloud(cloud)
    k0 = prefix_len(n, p)
    if k0 < 2:
        raise ValueError("ceil(p*n) must be >= 2 (SPEC.md:240)")
    if not (1 <= n <= pc.n):
        raise ValueError(f"n must be in [1, {pc.n}], got {n}")
    k0 = min(k0, n)
    xyz4 = engine.as_xyz4(pc.coords)
    idx, cv, md, taken = engine.fps(xyz4, n, seed_index, k_stop=k0)
    core.add_pair_evals(pc.n * (k0 - 1))
    res = core.SampleResult(idx[0, :k0].cpu().numpy(), "fps", {"fps_prefix_iters": k0})
    return cv[0, :k0].cpu().numpy(), FpsState(md[0].cpu().numpy(), taken[0].cpu().numpy()), res


def power_table(n: int, exponent: float) -> np.ndarray:
    """i**e as float64 for i in [0, n) (entry 0 unused)."""
    return np.power(np.arange(n, dtype=np.float64), np.float64(exponent))


def threshold_positions(n: int, nseg: int) -> np.ndarray:
    if nseg < 1:
        raise ValueError("nseg must be >= 1")
    if n < nseg + 1:
        raise ValueError(f"curve length n={n} must be >= nseg + 1 = {nseg + 1}")
    return np.array([min(n * s // nseg, n - 1) for s in range(1, nseg + 1)], np.int64)


def sampler_boundaries(n: int, nseg: int) -> np.ndarray:
    return np.array([n * s // nseg for s in range(1, nseg)] + [n], np.int64)


def clamp_radius(R: float) -> float:
    return R if R > 0 else TINY


def radius_sq(R: float) -> float:
    r2 = R * R
    return r2 if r2 > TINY else TINY


def fit_power_exponent(curves) -> float:
    """pooled least squares of log(v_i) on log(i), i >= 1."""
    xs, ys = [], []
    for c in curves:
        c = np.asarray(c, np.float64)
        if c.shape[0] < 9:
            raise ValueError("each curve needs >= 8 finite positions")
        v = c[1:]
        if np.any(~(v > 0)):
            raise ValueError("non-positive curve value")
        xs.append(np.log(np.arange(1, c.shape[0], dtype=np.float64)))
        ys.append(np.log(v))
    X = np.concatenate(xs)
    Y = np.concatenate(ys)
    X0 = X - X.mean()
    slope = float(np.dot(X0, Y - Y.mean()) / np.dot(X0, X0))
    return -slope


def estimate_power(prefix, n: int, exponent: float) -> np.ndarray:
    """Full estimated curve.  The sampling pipeline only
    needs est[d_s] and evaluates those on the device (K2); this host version
    returns the whole curve for users and reports."""
    v = np.asarray(prefix, np.float64)
    k0 = v.shape[0]
    if k0 < 2:
        raise ValueError("prefix needs >= 2 values")
    pw = power_table(max(n, k0), exponent)
    acc = 0.0
    for i in range(1, k0):
        acc = acc + float(v[i]) * float(pw[i])
    amp = acc / float(k0 - 1)
    out = np.empty(n, np.float64)
    out[:min(n, k0)] = v[:min(n, k0)]
    if n > k0:
        tail = amp / pw[k0:n]
        out[k0:n] = np.minimum.accumulate(np.concatenate([[v[k0 - 1]], tail]))[1:]
    return out


def segment_thresholds(curve, nseg: int):
    """SPEC.md:318-326 -> (d int64[nseg], R float64[nseg])."""
    c = np.asarray(curve, np.float64)
    d = threshold_positions(c.shape[0], nseg)
    R = np.minimum.accumulate(c[d])
    return d, R


def resample_curve(values, target_len: int) -> np.ndarray:
    """linear interpolation over normalised abscissa,
    endpoints exact.  Pinned formula (identical in K2 and the oracle):
    u = (t (S-1)) / (T-1), i0 = floor(u), out = v[i0] + (u - i0)(v[i0+1] - v[i0])."""
    v = np.asarray(values, np.float64)
    S = v.shape[0]
    if S < 2:
        raise ValueError("need >= 2 values")
    T = int(target_len)
    if T < 1:
        raise ValueError("target length must be >= 1")
    if T == 1:
        return v[:1].copy()
    t = np.arange(T, dtype=np.float64)
    u = (t * float(S - 1)) / float(T - 1)
    i0 = np.minimum(np.floor(u).astype(np.int64), S - 1)
    i1 = np.minimum(i0 + 1, S - 1)
    frac = u - i0
    out = v[i0] + frac * (v[i1] - v[i0])
    out[i0 >= S - 1] = v[S - 1]
    return out


# ---------------------------------------------------------------------------
# MLP estimator: 32 -> 128 -> 128 -> 64, relu, float64.
# Offline training on the host (SGD, batch 1, MSE; SPEC non-goal: no GPU
# training); inference runs on the device inside K2 (csrc/sampler.cu) with a
# fixed dot-product order, restated by oracle.estimate_mlp.

MLP_SIZES = (32, 128, 128, 64)


class MlpModel:
    """Weights W1 [128,32], b1, W2 [128,128], b2, W3 [64,128], b3 (float64)."""

    def __init__(self, W1, b1, W2, b2, W3, b3):
        self.W = [np.ascontiguousarray(W, np.float64) for W in (W1, W2, W3)]
        self.b = [np.ascontiguousarray(b, np.float64) for b in (b1, b2, b3)]
        for k, (W, b) in enumerate(zip(self.W, self.b)):
            if W.shape != (MLP_SIZES[k + 1], MLP_SIZES[k]) or b.shape != (MLP_SIZES[k + 1],):
                raise ValueError(f"layer {k + 1}: expected W {(MLP_SIZES[k + 1], MLP_SIZES[k])}")

    @staticmethod
    def init(rng: np.random.Generator) -> "MlpModel":
        """Uniform +-sqrt(6 / (fan_in + fan_out)) weights, zero biases."""
        mats = []
        for k in range(3):
            fi, fo = MLP_SIZES[k], MLP_SIZES[k + 1]
            lim = math.sqrt(6.0 / (fi + fo))
            mats += [rng.uniform(-lim, lim, size=(fo, fi)), np.zeros(fo)]
        return MlpModel(*mats)

    def copy(self) -> "MlpModel":
        return MlpModel(self.W[0], self.b[0], self.W[1], self.b[1], self.W[2], self.b[2])

    def forward(self, x):
        """Batch forward (numpy; training and reports)."""
        h = np.asarray(x, np.float64)
        for k in range(3):
            h = h @ self.W[k].T + self.b[k]
            if k < 2:
                h = np.maximum(h, 0.0)
        return h

    def packed(self) -> np.ndarray:
        """Device layout: W1 row-major, b1, W2, b2, W3, b3 (float64)."""
        return np.concatenate([a.ravel() for k in range(3) for a in (self.W[k], self.b[k])])

    def save(self, path):
        """SPEC.md:357 text format."""
        with open(path, "w") as f:
            f.write("MLP 32 128 128 64\n")
            for W, b in zip(self.W, self.b):
                f.write(f"W {W.shape[0]} {W.shape[1]}\n")
                f.write(" ".join(repr(float(x)) for x in W.ravel()) + "\n")
                f.write(f"B {b.shape[0]}\n")
                f.write(" ".join(repr(float(x)) for x in b) + "\n")

    @staticmethod
    def load(path) -> "MlpModel":
        tok = open(path).read().split()
        if tok[:5] != ["MLP", "32", "128", "128", "64"]:
            raise ValueError("not an `MLP 32 128 128 64` weight file")
        pos, mats = 5, []
        for _ in range(3):
            if tok[pos] != "W":
                raise ValueError("expected a `W r c` header")
            r, c = int(tok[pos + 1]), int(tok[pos + 2])
            W = np.array(tok[pos + 3:pos + 3 + r * c], np.float64).reshape(r, c)
            pos += 3 + r * c
            if tok[pos] != "B" or int(tok[pos + 1]) != r:
                raise ValueError("expected a `B c` header")
            mats += [W, np.array(tok[pos + 2:pos + 2 + r], np.float64)]
            pos += 2 + r
        return MlpModel(*mats)


def mlp_pair(curve, p: float = 0.1):
    """Training pair of one exact curve: finite prefix 1..k0-1
    resampled to 32 and the tail k0..n-1 to 64, both divided by v[k0-1]."""
    c = np.asarray(curve, np.float64)
    n = c.shape[0]
    k0 = prefix_len(n, p)
    scale = c[k0 - 1]
    if not scale > 0:
        raise ValueError("last prefix value must be > 0")
    return resample_curve(c[1:k0], 32) / scale, resample_curve(c[k0:], 64) / scale


def mlp_train(pairs, epochs: int, lr: float = 0.01, rng=None, model: MlpModel | None = None):
    """plain SGD on MSE, batch size 1, order shuffled per epoch
    by ``rng``.  Returns (model, per-epoch mean loss)."""
    rng = np.random.default_rng(0) if rng is None else rng
    m = MlpModel.init(rng) if model is None else model.copy()
    X = np.asarray([p[0] for p in pairs], np.float64)
    Y = np.asarray([p[1] for p in pairs], np.float64)
    losses = []
    for ep in range(int(epochs)):
        order = rng.permutation(X.shape[0])
        tot = 0.0
        for i in order:
            loss, grads = mlp_loss_grad(m, X[i], Y[i])
            if not math.isfinite(loss):
                raise FloatingPointError(f"training diverged at epoch {ep + 1}")
            tot += loss
            for k in range(3):
                m.W[k] -= lr * grads[2 * k]
                m.b[k] -= lr * grads[2 * k + 1]
        losses.append(tot / X.shape[0])
    return m, losses


def mlp_loss_grad(m: MlpModel, x, y):
    """MSE loss of one pair and its gradients [dW1, db1, dW2, db2, dW3, db3]."""
    a0 = np.asarray(x, np.float64)
    z1 = m.W[0] @ a0 + m.b[0]
    a1 = np.maximum(z1, 0.0)
    z2 = m.W[1] @ a1 + m.b[1]
    a2 = np.maximum(z2, 0.0)
    out = m.W[2] @ a2 + m.b[2]
    diff = out - np.asarray(y, np.float64)
    loss = float(np.mean(diff * diff))
    g3 = 2.0 * diff / diff.shape[0]
    dW3, db3 = np.outer(g3, a2), g3
    g2 = (m.W[2].T @ g3) * (z2 > 0)
    dW2, db2 = np.outer(g2, a1), g2
    g1 = (m.W[1].T @ g2) * (z1 > 0)
    dW1, db1 = np.outer(g1, a0), g1
    return loss, [dW1, db1, dW2, db2, dW3, db3]


def mlp_forward_exact(m: MlpModel, x) -> np.ndarray:
    """Inference with K2's order: each dot product summed in input order from
    0.0, bias added last, relu(a) = a if a > 0 else 0."""
    h = [float(v) for v in x]
    for k in range(3):
        W, b = m.W[k], m.b[k]
        nxt = []
        for j in range(W.shape[0]):
            acc = 0.0
            row = W[j]
            for i in range(W.shape[1]):
                acc = acc + float(row[i]) * h[i]
            acc = acc + float(b[j])
            nxt.append((acc if acc > 0.0 else 0.0) if k < 2 else acc)
        h = nxt
    return np.array(h, np.float64)


def estimate_mlp(prefix, n: int, model: MlpModel) -> np.ndarray:
    """SPEC.md:298-306 full estimated curve (the device evaluates only the
    segment radii, bit-identically)."""
    v = np.asarray(prefix, np.float64)
    k0 = v.shape[0]
    if k0 < 3:
        raise ValueError("the MLP estimator needs >= 2 finite prefix values")
    scale = float(v[k0 - 1])
    if not scale > 0:
        raise ValueError("last measured prefix value must be > 0")
    x = resample_curve(v[1:k0], 32) / scale
    y = mlp_forward_exact(model, x) * scale
    out = np.empty(n, np.float64)
    out[:k0] = v
    if n > k0:
        tail = resample_curve(y, n - k0)
        out[k0:] = np.minimum.accumulate(np.concatenate([[scale], tail]))[1:]
    return out


def estimator_mape(estimated, truth, p: float) -> float:
    """mean |est - truth| / truth over positions > ceil(p n)."""
    e = np.asarray(estimated, np.float64)
    t = np.asarray(truth, np.float64)
    k0 = prefix_len(t.shape[0], p)
    tail_t = t[k0 + 1:] if k0 + 1 < t.shape[0] else t[k0:]
    tail_e = e[k0 + 1:] if k0 + 1 < t.shape[0] else e[k0:]
    if np.any(tail_t == 0):
        raise ValueError("zero truth value in the tail")
    return float(np.mean(np.abs(tail_e - tail_t) / tail_t) * 100.0)
