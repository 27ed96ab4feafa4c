"""Third, vectorised implementation of DESIGN.md's canonical fp32 contract in NumPy float32.

Test-only arbiter: NumPy performs every element-wise float32 operation as one correctly
rounded IEEE binary32 op with no fusion, so this reproduces the contract bit for bit.
It is compared bitwise against BOTH the oracle (mode 0) and the CUDA kernel's debug
output; it imports neither.
"""
import numpy as np

f32 = np.float32
K_TETRA = f32(0.57735026918962576451)


def canonical(scene, cam, kappa=0.1, filter3d=None, exact=False):
    """exact: the no-ray-space variant's canonical geometry (DESIGN.md §3 "exact mode")."""
    kind = scene["kind"]
    K = 3 if kind == 0 else 4
    n = scene["pos"].shape[1]
    pos = scene["pos"].astype(f32)
    rot = scene["rot"].astype(f32)
    dist = scene["dist"].astype(f32)
    op = scene["opacity"].astype(f32)
    Wm = np.asarray(cam["W"], f32).reshape(3, 3)
    t = np.asarray(cam["t"], f32)
    fx, fy, cx, cy, zn = (f32(cam[k]) for k in ("fx", "fy", "cx", "cy", "znear"))
    Wd, Hd = int(cam["width"]), int(cam["height"])
    with np.errstate(all="ignore"):
        fin = np.isfinite(pos).all(0) & np.isfinite(rot).all(0) & np.isfinite(dist).all(0) & np.isfinite(op)
        if filter3d is not None:
            fin &= np.isfinite(filter3d)
        valid = fin & (dist > 0).all(0)
        if filter3d is not None:
            fl = filter3d.astype(f32)
            dh = np.sqrt(dist * dist + fl * fl)
        else:
            dh = dist
        qw, qx, qy, qz = rot
        n2 = ((qw * qw + qx * qx) + qy * qy) + qz * qz
        valid &= n2 != 0
        nq = np.sqrt(n2)
        w, x, y, z = qw / nq, qx / nq, qy / nq, qz / nq
        xx, yy, zz = x * x, y * y, z * z
        xy, xz, yz, wx, wy, wz = x * y, x * z, y * z, w * x, w * y, w * z
        one, two = f32(1), f32(2)
        R = [[one - two * (yy + zz), two * (xy - wz), two * (xz + wy)],
             [two * (xy + wz), one - two * (xx + zz), two * (yz - wx)],
             [two * (xz - wy), two * (yz + wx), one - two * (xx + yy)]]
        p = [((Wm[r, 0] * pos[0] + Wm[r, 1] * pos[1]) + Wm[r, 2] * pos[2]) + t[r] for r in range(3)]
        culled = valid & ~(p[2] > zn)
        ok = valid & ~culled
        l = np.sqrt((p[0] * p[0] + p[1] * p[1]) + p[2] * p[2])
        crx = fx * (p[0] / p[2]) + cx
        cry = fy * (p[1] / p[2]) + cy
        pz2 = p[2] * p[2]
        J00 = fx / p[2]
        J02 = -((fx * p[0]) / pz2)
        J11 = fy / p[2]
        J12 = -((fy * p[1]) / pz2)
        J20, J21, J22 = p[0] / l, p[1] / l, p[2] / l
        if kind == 0:
            ow = [[dh[j] * R[r][j] for r in range(3)] for j in range(3)]
        else:
            k = K_TETRA
            B = [(k, k, k), (k, -k, -k), (-k, k, -k), (-k, -k, k)]
            ow = [[dh[j] * ((R[r][0] * B[j][0] + R[r][1] * B[j][1]) + R[r][2] * B[j][2]) for r in range(3)]
                  for j in range(4)]
        off = np.zeros((K, 3, n), f32)
        for j in range(K):
            oc = [(Wm[r, 0] * ow[j][0] + Wm[r, 1] * ow[j][1]) + Wm[r, 2] * ow[j][2] for r in range(3)]
            if exact:
                off[j, 0], off[j, 1], off[j, 2] = oc
            else:
                off[j, 0] = J00 * oc[0] + J02 * oc[2]
                off[j, 1] = J11 * oc[1] + J12 * oc[2]
                off[j, 2] = (J20 * oc[0] + J21 * oc[1]) + J22 * oc[2]
        if exact:
            verts = []
            for j in range(K):
                verts.append([p[r] + off[j, r] for r in range(3)])
                if kind == 0:
                    verts.append([p[r] - off[j, r] for r in range(3)])
            behind = np.zeros(n, bool)
            us, ws = [], []
            for v in verts:
                behind |= ~(v[2] > 0)
                us.append(fx * (v[0] / v[2]) + cx)
                ws.append(fy * (v[1] / v[2]) + cy)
            us, ws = np.stack(us), np.stack(ws)
            lo = [np.where(behind, f32(-2), us.min(0)), np.where(behind, f32(-2), ws.min(0))]
            hi = [np.where(behind, f32(Wd + 2), us.max(0)), np.where(behind, f32(Hd + 2), ws.max(0))]
            crx, cry = p[0], p[1]
        h = f32(0.5) * f32(kappa)
        ar = np.arange(n)
        for ax in range(2 if not exact else 0):
            if kind == 0:
                a = np.abs(off[:, ax])
                jm = np.argmax(a, axis=0)           # first max
                v = off[jm, ax, ar]
                off[jm, ax, ar] = v + np.where(v >= 0, h, -h)
            else:
                kmin = np.argmin(off[:, ax], axis=0)     # both chosen before any shift
                kmax = np.argmax(off[:, ax], axis=0)
                off[kmin, ax, ar] = off[kmin, ax, ar] - h
                off[kmax, ax, ar] = off[kmax, ax, ar] + h
        if not exact:
            lo, hi = [], []
        for ax, c in (((0, crx), (1, cry)) if not exact else ()):
            if kind == 0:
                m = np.abs(off[:, ax]).max(0)
                lo.append(c - m)
                hi.append(c + m)
            else:
                lo.append(c + off[:, ax].min(0))
                hi.append(c + off[:, ax].max(0))
        rect = np.zeros((n, 4), np.int32)
        tt = np.zeros(n, np.uint32)
        pmin, pmax = [], []
        for ax, dim in ((0, Wd), (1, Hd)):
            a = np.clip(lo[ax] - f32(0.5), f32(-2), f32(dim + 2))
            b = np.clip(hi[ax] - f32(0.5), f32(-2), f32(dim + 2))
            a = np.where(np.isfinite(a), a, 0).astype(f32)
            b = np.where(np.isfinite(b), b, 0).astype(f32)
            pmin.append(np.maximum(0, np.ceil(a).astype(np.int64)))
            pmax.append(np.minimum(dim - 1, np.floor(b).astype(np.int64)))
        vis = ok & (pmin[0] <= pmax[0]) & (pmin[1] <= pmax[1])
        rect[:, 0] = np.where(vis, pmin[0] >> 4, 0)
        rect[:, 1] = np.where(vis, pmin[1] >> 4, 0)
        rect[:, 2] = np.where(vis, pmax[0] >> 4, 0)
        rect[:, 3] = np.where(vis, pmax[1] >> 4, 0)
        tt[vis] = ((rect[vis, 2] - rect[vis, 0] + 1) * (rect[vis, 3] - rect[vis, 1] + 1)).astype(np.uint32)
        key = np.where(ok, l.astype(f32).view(np.uint32), 0).astype(np.uint32)
        flag = np.where(~valid, 1, np.where(culled, 2, 0)).astype(np.int32)
        canon = np.zeros((n, 2 + 3 * K), f32)
        canon[:, 0] = np.where(ok, crx, 0)
        canon[:, 1] = np.where(ok, cry, 0)
        for j in range(K):
            for a in range(3):
                canon[:, 2 + 3 * j + a] = np.where(ok, off[j, a], 0)
    return {"flag": flag, "tiles_touched": tt, "rect": rect, "depth_key": key, "canon": canon}
