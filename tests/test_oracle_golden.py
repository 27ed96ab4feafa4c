"""Golden values (tests/golden/paper_values.json): paper-printed constants and SPEC worked examples."""
import json
import math
import os

import numpy as np
import pytest

import oracle
from tests.helpers import cam, one_prim, oscene

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


@pytest.mark.parametrize("case", GOLD["density"])
def test_density_golden(case):
    s = one_prim(oracle.OCTA, (0, 0, 5), (1, 0, 0, 0), (case["min_d"], 2.0, 3.0), logit=case["alpha_logit"])
    pre = oracle.preprocess(oscene(s), cam(), mode=1)
    assert math.isclose(pre.sigma[0], case["sigma"], abs_tol=5e-7), case["cite"]


@pytest.mark.parametrize("case", GOLD["opacity"])
def test_opacity_golden(case):
    # on-axis octahedron with d_z = min d, optical axis through a pixel centre: chord = 2 d_z
    dz = case["chord"] / 2.0
    logit = math.log(case["alpha"] / (1 - case["alpha"]))
    c = dict(cam(64, 48), cx=np.float32(32.5), cy=np.float32(24.5))
    s = one_prim(oracle.OCTA, (0, 0, 5.0), (1, 0, 0, 0), (3.0, 3.0, dz), logit=logit)
    den = np.array([2.0 * case["min_d"]])            # frozen Eq. 1 denominator with the quoted min d
    f = oracle.forward(oscene(s), c, kappa=0.0, mode=1, t_stop=0.0, den_override=den)
    assert math.isclose(1.0 - f.out.T_final[24, 32], case["o"], abs_tol=5e-7), case["cite"]


@pytest.mark.parametrize("case", GOLD["mtia"])
def test_mtia_golden(case):
    hit, u, v, d, depth = oracle.mtia(case["v0"], case["v1"], case["v2"], case["r"])
    assert hit
    assert math.isclose(u, case["u"], abs_tol=1e-15) and math.isclose(v, case["v"], abs_tol=1e-15)
    assert math.isclose(depth, case["depth"], abs_tol=1e-15), case["cite"]


def test_mtia_grad_golden_third_row():
    case = GOLD["mtia_grad_third_row"][0]
    m = GOLD["mtia"][0]
    hit, u, v, d, depth = oracle.mtia(m["v0"], m["v1"], m["v2"], case["r"])
    di = oracle.mtia_grad(m["v0"], m["v1"], m["v2"], case["r"], u, v, d)
    assert np.allclose(di[:, 2], case["dz"], atol=1e-15), case["cite"]


def test_mtia_grad_finite_differences():
    """App. E corner derivatives against central differences of the hit depth."""
    rng = np.random.default_rng(0)
    n_ok = 0
    while n_ok < 30:
        V = rng.normal(0, 1, (3, 3))
        r = V[:, :2].mean(0) + rng.normal(0, 0.2, 2)
        hit, u, v, d, depth = oracle.mtia(V[0], V[1], V[2], r)
        if not hit or min(u, v, 1 - u - v) < 0.02:
            continue
        di = oracle.mtia_grad(V[0], V[1], V[2], r, u, v, d)
        h = 1e-6
        for k in range(3):
            for a in range(3):
                Vp, Vm = V.copy(), V.copy()
                Vp[k, a] += h
                Vm[k, a] -= h
                fd = (oracle.mtia(*Vp, r)[4] - oracle.mtia(*Vm, r)[4]) / (2 * h)
                assert abs(fd - di[k, a]) < 1e-7 * (1 + abs(fd))
        n_ok += 1


def test_ray_space_map_golden():
    case = GOLD["ray_space_map"][0]
    c = dict(cam(), fx=np.float32(case["fx"]), fy=np.float32(case["fy"]), cx=np.float32(case["cx"]),
             cy=np.float32(case["cy"]))
    pre = oracle.preprocess(oscene(one_prim(oracle.OCTA, case["p"], (1, 0, 0, 0), (0.01, 0.01, 0.01))), c, mode=1)
    assert np.allclose(pre.geom[0, :3], case["phi"], atol=1e-12), case["cite"]


def test_constants_are_the_paper_defaults():
    """The library defaults quoted in DESIGN.md equal the paper's printed constants."""
    k = GOLD["constants"]
    assert k["eq1_opacity_scale"]["value"] == 0.99 and k["stop_cumulative"]["value"] == 0.999
    assert k["aa_kernel"]["value"] == 0.1 and k["tile_size"]["value"] == oracle.TILE
