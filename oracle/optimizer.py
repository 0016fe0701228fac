"""FP64 CPU oracle of the iteration driver.  TEST INFRASTRUCTURE ONLY.

Restates reference ``paball/optimizer.py`` on plain arrays:

* Adam with global step t, betas (0.9, 0.999), eps 1e-8     optimizer.py:48-50, 203-209
* zero-gradient filter (p0 := 0 probe, coarse backward)      optimizer.py:230-258
* one step: backward, finite guard, Adam on p0 / a0 (floor
  1e-9) / positions (fine only)                              optimizer.py:266-306
* density control: destroy, split, duplicate, moments        optimizer.py:314-406
* hierarchical driver with density cadence and plateau       optimizer.py:453-500

State is a dict: pos (n,3), p0, a0, a0_free, generation, m/v dicts keyed
"p0", "a0", "position", t (global step), last_gpos (or None), seed.
"""

from __future__ import annotations

import math

import numpy as np

from . import radiator as R
from .rng import CounterRng

BETA1, BETA2, EPS = 0.9, 0.999, 1e-8
A0_FLOOR = 1e-9
COARSE_DENSITY_EVERY = 100
PLATEAU_REL, PLATEAU_WINDOW = 1e-5, 50


class Problem:
    """Detectors + acquisition grid + directivity (the ForwardContext)."""

    def __init__(self, sensors, normals, v, t0, dt, n_samples, cutoff=6.0, kind=("none",), threads=1):
        self.sensors = np.asarray(sensors, dtype=np.float64)
        self.normals = normals
        self.v, self.t0, self.dt, self.n_samples = v, t0, dt, n_samples
        self.cutoff, self.kind, self.threads = cutoff, kind, threads

    def n_out(self, f):
        return -(-self.n_samples // f) if f > 1 else self.n_samples

    def backward(self, pos, p0, a0, real_k, f, stage):
        _, L, g, _ = R.run_model(pos, p0, a0, self.sensors, self.normals, self.v, self.t0,
                                 self.dt, self.n_samples, f, self.cutoff, real=real_k,
                                 stage=stage, kind=self.kind, threads=self.threads)
        return L, g

    def simulate(self, pos, p0, a0, f=1):
        rows, _, _, _ = R.run_model(pos, p0, a0, self.sensors, self.normals, self.v, self.t0,
                                    self.dt, self.n_samples, f, self.cutoff, kind=self.kind,
                                    threads=self.threads)
        return rows


def new_state(pos, p0, a0, seed=0, generation=0):
    n = len(p0)
    return {
        "pos": np.array(pos, dtype=np.float64).reshape(n, 3), "p0": np.array(p0, dtype=np.float64),
        "a0": np.array(a0, dtype=np.float64), "a0_free": np.full(n, math.nan),
        "generation": generation, "t": 0, "seed": int(seed), "last_gpos": None,
        "m": {"p0": np.zeros(n), "a0": np.zeros(n), "position": np.zeros((n, 3))},
        "v": {"p0": np.zeros(n), "a0": np.zeros(n), "position": np.zeros((n, 3))},
    }


def adam(state, key, values, grad, lr):
    t = state["t"]
    m = state["m"][key] = BETA1 * state["m"][key] + (1.0 - BETA1) * grad
    v = state["v"][key] = BETA2 * state["v"][key] + (1.0 - BETA2) * grad * grad
    return values - lr * (m / (1.0 - BETA1 ** t)) / (np.sqrt(v / (1.0 - BETA2 ** t)) + EPS)


def zero_gradient_filter(prob, pos, p0, a0, real, f, strict=True):
    """Returns (keep mask, g)."""
    if len(p0) == 0:
        raise ValueError("cannot filter an empty cloud")
    real_k = R.downsample(real, f) if f > 1 else real
    _, (g, _, _) = prob.backward(pos, np.zeros(len(p0)), a0, real_k, f, "coarse")
    keep = (g < 0.0) if strict else (g <= 0.0)
    return keep, g


def step(prob, state, real_k, f, stage, lr):
    """lr = (p0, a0, position).  Returns the pre-update loss."""
    L, (gp0, ga0, gpos) = prob.backward(state["pos"], state["p0"], state["a0"], real_k, f, stage)
    if not (math.isfinite(L) and np.isfinite(gp0).all() and np.isfinite(ga0).all()
            and np.isfinite(gpos).all()):
        raise FloatingPointError(f"non-finite loss or gradient at step {state['t']}")
    state["t"] += 1
    state["p0"] = adam(state, "p0", state["p0"], gp0, lr[0])
    state["a0"] = np.maximum(adam(state, "a0", state["a0"], ga0, lr[1]), A0_FLOOR)
    if stage == "fine":
        state["pos"] = adam(state, "position", state["pos"], gpos, lr[2])
    state["last_gpos"] = gpos
    return L


def density_control(state, th, stage):
    """th = dict(destroy_p0_frac, split_a0, duplicate_grad_quantile, a0_min, a0_max)."""
    n = len(state["p0"])
    if n == 0:
        state["generation"] += 1
        return state
    rng = CounterRng(state["seed"]).spawn(state["generation"])
    p0, a0 = state["p0"], state["a0"]
    weak = p0 < th["destroy_p0_frac"] * float(np.median(p0))
    bad = (a0 < th["a0_min"]) | (a0 > th["a0_max"])
    idx = np.flatnonzero(~(weak | bad))
    pos, p0, a0, free = state["pos"][idx], p0[idx], a0[idx], state["a0_free"][idx]
    m = {k: v[idx] for k, v in state["m"].items()}
    v = {k: x[idx] for k, x in state["v"].items()}
    gn = None
    if state["last_gpos"] is not None:
        gn = np.linalg.norm(state["last_gpos"], axis=1)[idx]
    big = a0 > th["split_a0"]
    bi = np.flatnonzero(big)
    new_pos, new_p0, new_a0, new_free = [pos[~big]], [p0[~big]], [a0[~big]], [free[~big]]
    if bi.size:
        off = 0.5 * a0[bi, None] * rng.unit_vectors(bi.size)
        new_pos.append(np.concatenate([pos[bi] + off, pos[bi] - off]))
        new_p0.append(np.concatenate([0.5 * p0[bi]] * 2))
        new_a0.append(np.concatenate([a0[bi] / math.sqrt(2.0)] * 2))
        new_free.append(np.concatenate([free[bi]] * 2))
    m = {k: x[~big] for k, x in m.items()}
    v = {k: x[~big] for k, x in v.items()}
    kept_pos, kept_p0, kept_a0, kept_free = new_pos[0], new_p0[0], new_a0[0], new_free[0]
    if stage == "fine" and gn is not None:
        gn = gn[~big]
        if gn.size:
            k = min(math.ceil((1.0 - th["duplicate_grad_quantile"]) * gn.size), gn.size)
            if k > 0:
                sel = np.sort(np.argsort(-gn, kind="stable")[:k])
                jit = (kept_a0[sel, None] / 4.0) * rng.unit_vectors(sel.size)
                new_pos.append(kept_pos[sel] + jit)
                new_p0.append(kept_p0[sel])
                new_a0.append(kept_a0[sel])
                new_free.append(kept_free[sel])
    n_keep = kept_pos.shape[0]
    state["pos"] = np.concatenate(new_pos)
    state["p0"] = np.concatenate(new_p0)
    state["a0"] = np.concatenate(new_a0)
    state["a0_free"] = np.concatenate(new_free)
    n_new = state["pos"].shape[0]
    for key in m:
        z = np.zeros((n_new - n_keep,) + m[key].shape[1:])
        state["m"][key] = np.concatenate([m[key], z])
        state["v"][key] = np.concatenate([v[key], z])
    state["generation"] += 1
    state["last_gpos"] = None
    return state


def run_hierarchical(prob, state, real, levels, th, lr, duplication_period=200,
                     plateau=True):
    """levels: list of (f, max_iters, stage).  Returns (state, losses, counts)."""
    losses_all, counts = [], []
    for f, iters, stage in levels:
        if len(state["p0"]) == 0:
            raise FloatingPointError("all points destroyed")
        real_k = R.downsample(real, f) if f > 1 else real
        period = COARSE_DENSITY_EVERY if stage == "coarse" else duplication_period
        losses = []
        for it in range(iters):
            L = step(prob, state, real_k, f, stage, lr)
            losses.append(L)
            losses_all.append(L)
            counts.append(len(state["p0"]))
            if (it + 1) % period == 0:
                density_control(state, th, stage)
                if len(state["p0"]) == 0:
                    raise FloatingPointError("all points destroyed")
            if plateau and len(losses) > PLATEAU_WINDOW:
                past = losses[-1 - PLATEAU_WINDOW]
                if abs(past - L) < PLATEAU_REL * max(abs(past), 1e-300):
                    break
    return state, losses_all, counts


# ---------------------------------------------------------------------------
# Positivity-constrained refinement (optimizer.py:507-573)
# ---------------------------------------------------------------------------


def softplus(x):
    """log(1 + e^x), overflow-safe split form (optimizer.py:507-510)."""
    x = np.asarray(x, dtype=np.float64)
    return np.log1p(np.exp(-np.abs(x))) + np.maximum(x, 0.0)


def inv_softplus(y):
    """Preimage of softplus for y > 0 (optimizer.py:513-523)."""
    y = np.asarray(y, dtype=np.float64)
    if np.any(y <= 0.0):
        raise ValueError("inv_softplus requires strictly positive input")
    small = y < 0.7
    out = np.empty_like(y)
    out[small] = np.log(np.expm1(y[small]))
    out[~small] = y[~small] + np.log1p(-np.exp(-y[~small]))
    return out


def sigmoid(x):
    """Logistic function, split by sign (optimizer.py:526-533)."""
    x = np.asarray(x, dtype=np.float64)
    pos = x >= 0.0
    out = np.empty_like(x)
    out[pos] = 1.0 / (1.0 + np.exp(-x[pos]))
    ex = np.exp(x[~pos])
    out[~pos] = ex / (1.0 + ex)
    return out


def positivity_refine(prob, state, real, iters, lr):
    """a0 = softplus(a0_free), fresh moments, fine backward at f = 1, Adam on
    p0, a0_free (chain rule through sigmoid) and positions; no a0 floor
    (optimizer.py:536-573).  Returns (pos, p0, a0, a0_free)."""
    pos, p0, a0 = state["pos"].copy(), state["p0"].copy(), state["a0"].copy()
    if len(p0) and np.any(a0 <= 0.0):
        raise ValueError("positivity refinement requires a0 > 0 at entry")
    free = inv_softplus(a0) if len(p0) else np.empty(0)
    ref = new_state(pos, p0, a0, seed=state["seed"])
    for _ in range(int(iters)):
        a0 = softplus(free)
        L, (gp0, ga0, gpos) = prob.backward(pos, p0, a0, real, 1, "fine")
        if not math.isfinite(L):
            raise FloatingPointError(f"non-finite loss during refinement: {L}")
        ref["t"] += 1
        p0 = adam(ref, "p0", p0, gp0, lr[0])
        free = adam(ref, "a0", free, ga0 * sigmoid(free), lr[1])
        pos = adam(ref, "position", pos, gpos, lr[2])
    return pos, p0, softplus(free), free.copy()
