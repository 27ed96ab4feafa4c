"""Shared test helpers (marshalling only)."""
import numpy as np

import oracle
from paper_2501_16312_b200 import scenegen


def oscene(scene, filter3d=None):
    return oracle.Scene(scene["kind"], scene["pos"], scene["rot"], scene["dist"], scene["opacity"],
                        scene["sh"], scene["sh_degree"], filter3d=filter3d)


def one_prim(kind, pos, rot, dist, logit=0.0, sh_degree=0, rgb_dc=(1.0, 1.0, 1.0)):
    """A single-primitive scene dict."""
    K = 3 if kind == oracle.OCTA else 4
    sh = np.zeros(((sh_degree + 1) ** 2, 3, 1), np.float32)
    sh[0, :, 0] = rgb_dc
    return {"kind": kind, "sh_degree": sh_degree,
            "pos": np.asarray(pos, np.float32).reshape(3, 1),
            "rot": np.asarray(rot, np.float32).reshape(4, 1),
            "dist": np.asarray(dist, np.float32).reshape(K, 1),
            "opacity": np.asarray([logit], np.float32),
            "sh": sh}


def concat(scenes):
    out = dict(scenes[0])
    for k in ("pos", "rot", "dist", "sh"):
        out[k] = np.concatenate([s[k] for s in scenes], axis=-1)
    out["opacity"] = np.concatenate([s["opacity"] for s in scenes])
    return out


def cam(width=64, height=48, **kw):
    return scenegen.pinhole(width, height, **kw)
