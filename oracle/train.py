"""CPU oracle of the C5 training step -- TEST INFRASTRUCTURE, fp64 NumPy.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s oracle legs may import this.

P:210-213: "we use the loss formulation of 3DGS, consisting of L1 and SSIM terms.  The gradients
are then optimized using ADAM [kingma_adam_2017] and backpropagated through the entire rendering
pipeline".  P:1169-1185 (Table "learning rates"): colour 2.5e-3, SH coefficients 1.25e-4, opacity
2.5e-2, rotation 1e-3, distance 2.6^-1 x 1e-4 scaled by the camera extent (dagger); the position
rate "consistent with 3DGS" is 1.6e-4 x extent (3DGS's initial position rate).

What this module computes, each step written out in the paper's order:
  * ``adam_step``: Adam as Kingma & Ba (Algorithm 1) state it -- m <- b1 m + (1 - b1) g,
    v <- b2 v + (1 - b2) g^2, m_hat = m / (1 - b1^t), v_hat = v / (1 - b2^t),
    p <- p - lr m_hat / (sqrt(v_hat) + eps) -- per parameter group, fp64; elements outside every
    group are untouched.
  * ``lr_table``: the paper's per-feature learning rates as groups of the flat feature buffer
    [pos 3N | rot 4N | dist KN | opacity N | sh (deg+1)^2 3N] (SH DC = "colour", the rest = "SH").
  * ``c5_step``: one training iteration over a batch of views: render every view (oracle.forward),
    the 3DGS loss of the batch (oracle.loss.batch_loss_and_grad: mean over views), the backward of
    every view with its dL/dimage (oracle.render + oracle.preprocess_bwd), the sum of the per-view
    feature gradients, and one Adam step.  The oracle never sees the CUDA path's values.
"""
from __future__ import annotations

import numpy as np

import oracle
from oracle import loss as oloss

SECTIONS = ("pos", "rot", "dist", "opacity", "sh")


def sizes(kind, n, sh_degree):
    K = 3 if kind == oracle.OCTA else 4
    return {"pos": 3 * n, "rot": 4 * n, "dist": K * n, "opacity": n, "sh": (sh_degree + 1) ** 2 * 3 * n}


def offsets(kind, n, sh_degree):
    out, o = {}, 0
    for name in SECTIONS:
        sz = sizes(kind, n, sh_degree)[name]
        out[name] = (o, o + sz)
        o += sz
    return out


def lr_table(kind, n, sh_degree, extent):
    """(begin, end, lr) groups of the flat buffer: P:1169-1185 (+ position per 3DGS)."""
    off = offsets(kind, n, sh_degree)
    sh0 = off["sh"][0]
    return [(off["pos"][0], off["pos"][1], 1.6e-4 * extent),
            (off["rot"][0], off["rot"][1], 1e-3),
            (off["dist"][0], off["dist"][1], 1e-4 / 2.6 * extent),
            (off["opacity"][0], off["opacity"][1], 2.5e-2),
            (sh0, sh0 + 3 * n, 2.5e-3),                       # SH DC coefficients = "colour"
            (sh0 + 3 * n, off["sh"][1], 1.25e-4)]


def adam_step(p, g, m, v, groups, t, b1=0.9, b2=0.999, eps=1e-15):
    """Kingma & Ba, Algorithm 1, one step t >= 1 per group (fp64).  Returns new (p, m, v)."""
    p = np.array(p, np.float64)
    g = np.asarray(g, np.float64)
    m = np.array(m, np.float64)
    v = np.array(v, np.float64)
    for b, e, lr in groups:
        gs = g[b:e]
        m[b:e] = b1 * m[b:e] + (1.0 - b1) * gs
        v[b:e] = b2 * v[b:e] + (1.0 - b2) * gs * gs
        m_hat = m[b:e] / (1.0 - b1 ** t)
        v_hat = v[b:e] / (1.0 - b2 ** t)
        p[b:e] = p[b:e] - lr * m_hat / (np.sqrt(v_hat) + eps)
    return p, m, v


def adam_update_sensitivity(g, m, v, groups, t, b1=0.9, b2=0.999, eps=1e-15):
    """|d p_new / d g| per element (fp64): how far an error in the gradient moves the updated
    parameter -- the derivative of lr m_hat / (sqrt(v_hat) + eps) with m, v as in adam_step."""
    g = np.asarray(g, np.float64)
    out = np.zeros_like(g)
    for b, e, lr in groups:
        gs = g[b:e]
        mn = b1 * m[b:e] + (1.0 - b1) * gs
        vn = b2 * v[b:e] + (1.0 - b2) * gs * gs
        c1, c2 = 1.0 - b1 ** t, 1.0 - b2 ** t
        s = np.sqrt(vn / c2)
        den = s + eps
        dm = (1.0 - b1) / c1
        dv = 2.0 * (1.0 - b2) * gs / c2
        ds = np.where(s > 0, dv / (2.0 * np.where(s > 0, s, 1.0)), 0.0)
        out[b:e] = np.abs(lr * (dm / den - (mn / c1) * ds / (den * den)))
    return out


def flat(grads: "oracle.Grads"):
    """Feature gradients in the flat [pos | rot | dist | opacity | sh] layout (fp64)."""
    return np.concatenate([np.asarray(getattr(grads, k), np.float64).reshape(-1) for k in SECTIONS])


def c5_step(scene: "oracle.Scene", cams, targets, groups, m, v, t, lam=oloss.LAMBDA, kappa=0.1, t_stop=1e-3,
            bg=(0.0, 0.0, 0.0), b1=0.9, b2=0.999, eps=1e-15, bounds=False, face_margin=2e-5, clamp_margin=1e-6,
            mode=0):
    """One training iteration over the views `cams`.  Returns a dict with the loss, the
    images [V,3,H,W], dL/dimage [V,3,H,W], the summed flat gradient, the new flat parameters, m, v
    and the per-view forward results.  bounds=True adds (test tolerances only) the summed flat
    conditioning bound of the gradient, the primitives any view flags for an entry / exit face within
    `face_margin` of switching, and the (primitive, channel) colour clamps within `clamp_margin`.
    mode: geometry precision of oracle.preprocess (0 canonical fp32, 1 fp64 for finite differences)."""
    fwd = [oracle.forward(scene, c, kappa=kappa, t_stop=t_stop, bg=bg, mode=mode) for c in cams]
    X = np.stack([f.out.image for f in fwd])
    L, dL = oloss.batch_loss_and_grad(X, np.asarray(targets, np.float64), lam)
    gsum = bsum = None
    flagged = clamp = None
    for f, c, d in zip(fwd, cams, dL):
        rb = oracle.render(scene, c, f.pre, f.vals, f.ranges, bg=bg, t_stop=t_stop,
                           dL_dimage=d.astype(np.float32), bounds=bounds)
        gv = flat(oracle.preprocess_bwd(scene, c, f.pre, rb))
        gsum = gv if gsum is None else gsum + gv
        if bounds:
            bv = flat(oracle.feature_bounds(scene, c, f.pre, rb))
            bsum = bv if bsum is None else bsum + bv
            fl = rb.face_margin < face_margin
            cl = (np.abs(f.pre.rgb_raw) < clamp_margin) & (f.pre.flag == 0)[:, None]
            flagged = fl if flagged is None else flagged | fl
            clamp = cl if clamp is None else clamp | cl
    p0 = np.concatenate([np.asarray(getattr(scene, k), np.float64).reshape(-1) for k in SECTIONS])
    p1, m1, v1 = adam_step(p0, gsum, m, v, groups, t, b1, b2, eps)
    return {"loss": L, "images": X, "dL": dL, "grad": gsum, "p0": p0, "p": p1, "m": m1, "v": v1, "fwd": fwd,
            "bound": bsum, "flagged": flagged, "clamp": clamp}
