"""FP64 CPU oracle of the Gaussian-ball forward model and its adjoint.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates reference ``paball/radiator.py`` (paths relative to
/root/reference/pkg/src/paball):

* per-pair window rule, absolute-index u, support mask   radiator.py:194-245
* u- / u+ terms and the near-field skip                  radiator.py:197-208
* scatter into sensor rows                               radiator.py:251-255
* residual, loss, per-ball sums and gradients            radiator.py:263-286
* sensor blocks of 8, fixed-order merge, 2/N scaling     radiator.py:290-359
* decimation and factor inference                        radiator.py:382-416

Differences from the reference, all deliberate:

1. The gradient-mode scratch-key collision (radiator.py:235 vs :240/:273,
   SURVEY.md §0.2) does not exist here: every cached quantity is a fresh array.
2. Ragged evaluation: instead of padded (chunk, sensor, width) slabs, only the
   (pair, sample) entries of each window are materialised.  Padded entries of
   the reference contribute exact zeros, so the forward rows are bit-identical
   (same u, G, weight per entry, same bincount order per 512-ball chunk).
3. Detector directivity multiplies each pair's amplitude
   by D_ij; ``("none",)`` is the reference semantics (D = 1).
"""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor

import numpy as np

CHUNK = 512          # balls per slab (radiator.py:50); fixes the rows' summation grouping
SENSOR_BLOCK = 8     # sensors per block / worker task (radiator.py:51)


class OracleSimulationError(Exception):
    """Ball coincident with a sensor (reference SimulationError)."""


# ---------------------------------------------------------------------------
# Directivity (not in the reference)
# ---------------------------------------------------------------------------

def element_axes(facing: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """In-plane unit axes (e1, e2) of each detector face: the global x axis
    projected on the face plane (y if the face is normal to x), e2 = n x e1."""
    ref = np.zeros_like(facing)
    ref[:, 0] = 1.0
    near_x = np.abs(facing[:, 0]) > 0.9
    ref[near_x] = [0.0, 1.0, 0.0]
    e1 = ref - np.sum(ref * facing, axis=1, keepdims=True) * facing
    e1 /= np.linalg.norm(e1, axis=1, keepdims=True)
    e2 = np.cross(facing, e1)
    return e1, e2


def _sinc_and_slope(x):
    """sinc(x) = sin x / x and d sinc/dx, with series near 0."""
    small = np.abs(x) < 1e-4
    xs = np.where(small, 1.0, x)
    s = np.where(small, 1.0 - x * x / 6.0, np.sin(xs) / xs)
    ds = np.where(small, -x / 3.0, (np.cos(xs) - np.sin(xs) / xs) / xs)
    return s, ds


def directivity(kind, diff, d, facing, a0, e1=None, e2=None):
    """Per-pair weight D and its gradients.

    diff (nc, sb, 3) = r_ball - r_sensor, d (nc, sb), facing (sb, 3) the unit
    receive direction, a0 (nc,).  Returns (D, dD_dr (nc, sb, 3), dD_da0).
    """
    name = kind[0]
    if name == "none":
        return None, None, None
    rhat = diff / d[..., None]
    if name == "cos_power":
        p = float(kind[1])
        c = np.einsum("bsx,sx->bs", rhat, facing)
        cp = np.maximum(c, 0.0)
        D = cp ** p
        dDdc = np.where(c > 0.0, p * cp ** (p - 1.0), 0.0)
        # d cos / d r_ball = (facing - cos * rhat) / d
        dc_dr = (facing[None, :, :] - c[..., None] * rhat) / d[..., None]
        return D, dDdc[..., None] * dc_dr, np.zeros_like(D)
    if name == "element":
        w = float(kind[1])
        s1 = np.einsum("bsx,sx->bs", rhat, e1)
        s2 = np.einsum("bsx,sx->bs", rhat, e2)
        scale = (w / (2.0 * a0))[:, None]
        f1, g1 = _sinc_and_slope(scale * s1)
        f2, g2 = _sinc_and_slope(scale * s2)
        D = f1 * f2
        # d s_k / d r_ball = (e_k - s_k rhat) / d
        ds1 = (e1[None] - s1[..., None] * rhat) / d[..., None]
        ds2 = (e2[None] - s2[..., None] * rhat) / d[..., None]
        dD_dr = (g1 * f2 * scale)[..., None] * ds1 + (f1 * g2 * scale)[..., None] * ds2
        # d(scale)/d a0 = -scale / a0
        dD_da0 = -(g1 * f2 * scale * s1 + f1 * g2 * scale * s2) / a0[:, None]
        return D, dD_dr, dD_da0
    raise ValueError(f"unknown directivity {kind!r}")


# ---------------------------------------------------------------------------
# One sensor block: all balls against up to 8 sensors
# ---------------------------------------------------------------------------

def _windows(lo_vt, hi_vt, vt0, vdt, f, n_out):
    """Decimated sample range [j_lo, j_hi] covering |u| <= hw with one sample
    of padding each side (radiator.py:209-212)."""
    k_lo = np.floor((lo_vt - vt0) / vdt).astype(np.int64) - 1
    k_hi = np.ceil((hi_vt - vt0) / vdt).astype(np.int64) + 1
    j_lo = np.maximum(-((-k_lo) // f), 0)
    j_hi = np.minimum(k_hi // f, n_out - 1)
    return j_lo, j_hi


def _ragged(j_lo, j_hi):
    """Flatten windows into (pair id, sample index) entries, pair-major."""
    length = np.maximum(j_hi - j_lo + 1, 0).ravel()
    total = int(length.sum())
    pair = np.repeat(np.arange(length.size), length)
    start = np.cumsum(length) - length
    J = j_lo.ravel()[pair] + (np.arange(total) - start[pair])
    return pair, J


def block_pass(positions, p0, a0, sensors, facing, kind, e1, e2, v, t0, dt, f,
               n_out, cutoff, real_blk, stage):
    """Forward rows for one sensor block, and (real_blk given) the loss part
    and unnormalised per-ball gradient sums.  Returns
    (rows, loss_part, g_p0, g_a0, g_pos, ops)."""
    sb = sensors.shape[0]
    n = positions.shape[0]
    grad = real_blk is not None
    fine = stage == "fine"
    vt0 = v * t0
    vdt = v * dt
    rows = np.zeros(sb * n_out)
    inv_a2 = 1.0 / (a0 * a0)
    nh = -0.5 * inv_a2
    inv_a3 = inv_a2 / a0
    row_off = np.arange(sb, dtype=np.int64) * n_out
    ops = 0
    cache = []
    for c0 in range(0, n, CHUNK):
        c1 = min(c0 + CHUNK, n)
        nc = c1 - c0
        diff = positions[c0:c1, None, :] - sensors[None, :, :]
        d = np.sqrt(np.einsum("bsx,bsx->bs", diff, diff))
        if np.any(d < 1e-12):
            raise OracleSimulationError(
                "ball coincident with a sensor (zero source-sensor distance)")
        hw = cutoff * a0[c0:c1]
        hw2 = hw * hw
        D, dD_dr, dD_da0 = directivity(kind, diff, d, facing, a0[c0:c1], e1, e2)
        base = p0[c0:c1, None] / (2.0 * d)
        amp = base if D is None else base * D
        for main in (True, False):
            if main:
                lo_vt, hi_vt = d - hw[:, None], d + hw[:, None]
            else:
                hi_vt = hw[:, None] - d
                if np.all(hi_vt < vt0):
                    continue
                lo_vt = -(d + hw[:, None])
            j_lo, j_hi = _windows(lo_vt, hi_vt, vt0, vdt, f, n_out)
            pair, J = _ragged(j_lo, j_hi)
            if pair.size == 0:
                continue
            ball = pair // sb
            sens = pair % sb
            kv = (J * f).astype(np.float64) * vdt
            dflat = d.ravel()[pair]
            u = (dflat - vt0) - kv if main else (dflat + vt0) + kv
            u2 = u * u
            keep = u2 <= hw2[ball]
            ops += int(np.count_nonzero(keep))
            pair, ball, sens, J, u, u2 = (a[keep] for a in (pair, ball, sens, J, u, u2))
            G = np.exp(u2 * nh[c0 + ball])
            w = u * G
            w *= amp.ravel()[pair]
            flat = row_off[sens] + J
            rows += np.bincount(flat, weights=w, minlength=sb * n_out)
            if grad:
                cache.append((pair, flat, u, u2, G))
        if grad:
            cache_chunk = (c0, c1, d, diff, amp, base, D, dD_dr, dD_da0)
            cache.append(cache_chunk)
    rows = rows.reshape(sb, n_out)
    if not grad:
        return rows, 0.0, None, None, None, ops

    res = rows - real_blk
    loss_part = float(np.vdot(res, res))
    res_flat = res.ravel()
    g_p0 = np.zeros(n)
    g_a0 = np.zeros(n)
    g_pos = np.zeros((n, 3)) if fine else None
    pending = []
    for item in cache:
        if len(item) == 5:
            pending.append(item)
            continue
        c0, c1, d, diff, amp, base, D, dD_dr, dD_da0 = item
        npair = (c1 - c0) * sb
        s_uG = np.zeros(npair)
        s_u3G = np.zeros(npair)
        s_G = np.zeros(npair)
        s_Gu2 = np.zeros(npair)
        for pair, flat, u, u2, G in pending:
            RG = res_flat[flat] * G
            t = RG * u
            s_uG += np.bincount(pair, weights=t, minlength=npair)
            s_u3G += np.bincount(pair, weights=t * u2, minlength=npair)
            if fine:
                s_G += np.bincount(pair, weights=RG, minlength=npair)
                s_Gu2 += np.bincount(pair, weights=RG * u2, minlength=npair)
        pending = []
        shape = (c1 - c0, sb)
        s_uG, s_u3G, s_G, s_Gu2 = (s.reshape(shape) for s in (s_uG, s_u3G, s_G, s_Gu2))
        # dL/dp0: amp = p0 * D / (2d)
        dp0 = s_uG * (0.5 / d)
        if D is not None:
            dp0 = dp0 * D
        g_p0[c0:c1] += dp0.sum(axis=1)
        ga0 = (amp * s_u3G) * inv_a3[c0:c1, None]
        if D is not None and kind[0] == "element":
            ga0 = ga0 + base * dD_da0 * s_uG
        g_a0[c0:c1] += ga0.sum(axis=1)
        if fine:
            g_dist = amp * (s_G - s_Gu2 * inv_a2[c0:c1, None]) - (amp / d) * s_uG
            gp = np.einsum("bs,bsx->bx", g_dist / d, diff)
            if D is not None:
                gp = gp + np.einsum("bs,bsx->bx", base * s_uG, dD_dr)
            g_pos[c0:c1] += gp
    return rows, loss_part, g_p0, g_a0, g_pos, ops


# ---------------------------------------------------------------------------
# Whole model: sensor blocks (threaded), fixed-order merge, MSE scaling
# ---------------------------------------------------------------------------

def facing_directions(normals, n_sensors):
    """Receive direction = -outward normal (reference convention,
    model.py:298, geometry.py:391)."""
    if normals is None:
        return np.zeros((n_sensors, 3))
    nrm = np.asarray(normals, dtype=np.float64)
    return -nrm / np.linalg.norm(nrm, axis=1, keepdims=True)


def run_model(positions, p0, a0, sensors, normals, v, t0, dt, n_samples, f,
              cutoff=6.0, real=None, stage="fine", kind=("none",), threads=1):
    """Reference ``_run_model`` (radiator.py:290-359) on plain arrays.

    Returns (rows (J, n_out), loss or None, (g_p0, g_a0, g_pos) or None, ops).
    """
    positions = np.asarray(positions, dtype=np.float64).reshape(-1, 3)
    p0 = np.asarray(p0, dtype=np.float64).reshape(-1)
    a0 = np.asarray(a0, dtype=np.float64).reshape(-1)
    sensors = np.asarray(sensors, dtype=np.float64).reshape(-1, 3)
    if np.any(a0 <= 0.0):
        raise ValueError("all a0 must be > 0 for forward simulation")
    n_out = -(-n_samples // f) if f > 1 else n_samples
    grad = real is not None
    if grad and real.shape[1] != n_out:
        raise ValueError(f"supervision has {real.shape[1]} samples, expected {n_out}")
    nsens = sensors.shape[0]
    n = positions.shape[0]
    rows = np.zeros((nsens, n_out))
    if n == 0:
        if grad:
            return rows, float(np.sum(real * real) / real.size), (
                np.zeros(0), np.zeros(0), np.zeros((0, 3))), 0
        return rows, None, None, 0
    facing = facing_directions(normals, nsens)
    e1 = e2 = None
    if kind[0] == "element":
        e1, e2 = element_axes(facing)

    def one(lo):
        hi = min(lo + SENSOR_BLOCK, nsens)
        out = block_pass(positions, p0, a0, sensors[lo:hi], facing[lo:hi], kind,
                         None if e1 is None else e1[lo:hi],
                         None if e2 is None else e2[lo:hi],
                         v, t0, dt, f, n_out, cutoff,
                         real[lo:hi] if grad else None, stage)
        return (lo,) + out

    starts = list(range(0, nsens, SENSOR_BLOCK))
    workers = min(max(1, int(threads)), len(starts))
    if workers <= 1:
        results = [one(lo) for lo in starts]
    else:
        with ThreadPoolExecutor(max_workers=workers) as pool:
            results = list(pool.map(one, starts))
    loss_sum = 0.0
    ops = 0
    g_p0, g_a0, g_pos = np.zeros(n), np.zeros(n), np.zeros((n, 3))
    for lo, brows, bloss, bp0, ba0, bpos, bops in sorted(results, key=lambda r: r[0]):
        rows[lo:lo + brows.shape[0]] = brows
        ops += bops
        if grad:
            loss_sum += bloss
            g_p0 += bp0
            g_a0 += ba0
            if bpos is not None:
                g_pos += bpos
    if not grad:
        return rows, None, None, ops
    total = nsens * n_out
    scale = 2.0 / total
    return rows, loss_sum / total, (scale * g_p0, scale * g_a0, scale * g_pos), ops


def infer_factor(dt_ctx, t0_ctx, n_ctx, dt_real, t0_real, n_real):
    """radiator.py:405-416."""
    ratio = dt_real / dt_ctx
    f = int(round(ratio))
    if f < 1 or abs(ratio - f) > 1e-9 * f or t0_real != t0_ctx:
        raise ValueError("supervision grid is not an integer decimation of the context grid")
    if -(-n_ctx // f) != n_real:
        raise ValueError("supervision grid is not an integer decimation of the context grid")
    return f


def downsample(data, f):
    """radiator.py:382-390: keep samples 0, f, 2f, ..."""
    f = int(f)
    if f < 1:
        raise ValueError(f"decimation factor must be >= 1, got {f}")
    return np.array(data[:, ::f], copy=True)


def mse(a, b):
    """radiator.py:393-402."""
    diff = a - b
    return float(np.sum(diff * diff) / diff.size)


def single_ball_kernel(d, p0, a0, times, v, cutoff=6.0):
    """Direct closed form for one pair (reference test_radiator.py:70-81)."""
    um, up = d - v * times, d + v * times
    cut = cutoff * a0
    return (p0 / (2.0 * d)) * (
        um * np.exp(-um ** 2 / (2.0 * a0 ** 2)) * (np.abs(um) <= cut)
        + up * np.exp(-up ** 2 / (2.0 * a0 ** 2)) * (np.abs(up) <= cut))

