"""3DGS PLY scene IO (SPEC S:545-553 `load_ply`): binary little-endian PLY with
the standard 3DGS vertex properties

    x, y, z, [nx, ny, nz], f_dc_0..2, f_rest_0..(3*((deg+1)^2-1)-1), opacity, scale_0..2, rot_0..3
    [, vtrain]

and the 3DGS activations: scale = exp(stored), opacity = sigmoid(stored), rotation normalised
(rot_0 = w). f_rest is channel-major (all coefficients of R, then G, then B); the renderer's SH
layout is coefficient-major, channel-minor (N x (deg+1)^2 x 3). An optional `vtrain` property
carries v_hat_train (Eq. 6); without it v_train is +inf (the filter is purely render-adaptive,
S:192) until `Renderer.compute_vtrain(cams, store=True)` sets it from training cameras.

Host-side plumbing only: the arrays go to `Renderer.load`, which validates them.
"""
from __future__ import annotations

import dataclasses

import numpy as np

_TYPES = {"float": "<f4", "float32": "<f4", "double": "<f8", "float64": "<f8", "uchar": "u1", "uint8": "u1",
          "char": "i1", "int8": "i1", "short": "<i2", "int16": "<i2", "ushort": "<u2", "uint16": "<u2",
          "int": "<i4", "int32": "<i4", "uint": "<u4", "uint32": "<u4"}


class PlyError(ValueError):
    pass


@dataclasses.dataclass
class PlyScene:
    means: np.ndarray      # (N, 3) float32
    scales: np.ndarray     # (N, 3) float32, activated (exp)
    quats: np.ndarray      # (N, 4) float32, (w, x, y, z), normalised
    opacities: np.ndarray  # (N,) float32, activated (sigmoid)
    sh: np.ndarray         # (N, (deg+1)^2, 3) float32
    v_train: np.ndarray    # (N,) float32, +inf when absent
    sh_degree: int

    @property
    def n(self) -> int:
        return int(self.means.shape[0])


def _parse_header(buf: bytes):
    end = buf.find(b"end_header\n")
    if end < 0:
        raise PlyError("byte 0: no 'end_header' line")
    lines = buf[:end].decode("ascii", errors="replace").split("\n")
    if not lines or lines[0].strip() != "ply":
        raise PlyError("line 1: not a PLY file (missing 'ply' magic)")
    fmt, n, props, in_vertex = None, None, [], False
    for i, raw in enumerate(lines[1:], start=2):
        tok = raw.split()
        if not tok or tok[0] in ("comment", "obj_info"):
            continue
        if tok[0] == "format":
            if len(tok) < 2 or tok[1] != "binary_little_endian":
                raise PlyError(f"line {i}: unsupported format {' '.join(tok[1:])!r} (need binary_little_endian)")
            fmt = tok[1]
        elif tok[0] == "element":
            if len(tok) != 3:
                raise PlyError(f"line {i}: malformed element line {raw!r}")
            in_vertex = tok[1] == "vertex"
            if in_vertex:
                try:
                    n = int(tok[2])
                except ValueError:
                    raise PlyError(f"line {i}: bad vertex count {tok[2]!r}") from None
                if n < 0:
                    raise PlyError(f"line {i}: negative vertex count")
            elif n is not None and int(tok[2]) > 0:
                raise PlyError(f"line {i}: element {tok[1]!r} after vertex is not supported")
        elif tok[0] == "property":
            if not in_vertex:
                continue
            if len(tok) != 3 or tok[1] == "list":
                raise PlyError(f"line {i}: unsupported vertex property {raw!r}")
            if tok[1] not in _TYPES:
                raise PlyError(f"line {i}: unknown property type {tok[1]!r}")
            props.append((tok[2], _TYPES[tok[1]]))
        else:
            raise PlyError(f"line {i}: unexpected header keyword {tok[0]!r}")
    if fmt is None:
        raise PlyError("header: missing 'format' line")
    if n is None:
        raise PlyError("header: missing 'element vertex'")
    return n, props, end + len(b"end_header\n")


def read_ply(path) -> PlyScene:
    buf = open(path, "rb").read()
    n, props, off = _parse_header(buf)
    dt = np.dtype(props)
    need = n * dt.itemsize
    if len(buf) - off < need:
        raise PlyError(f"byte {off}: vertex data truncated ({len(buf) - off} of {need} bytes)")
    v = np.frombuffer(buf, dtype=dt, count=n, offset=off)
    names = set(dt.names)
    for req in ("x", "y", "z", "f_dc_0", "f_dc_1", "f_dc_2", "opacity", "scale_0", "scale_1", "scale_2",
                "rot_0", "rot_1", "rot_2", "rot_3"):
        if req not in names:
            raise PlyError(f"header: missing vertex property {req!r}")
    n_rest = sum(1 for nm in names if nm.startswith("f_rest_"))
    if n_rest % 3:
        raise PlyError(f"header: {n_rest} f_rest properties (not a multiple of 3)")
    K = n_rest // 3 + 1
    deg = int(round(np.sqrt(K))) - 1
    if (deg + 1) ** 2 != K or deg > 3:
        raise PlyError(f"header: {n_rest} f_rest properties do not form SH degree <= 3")
    f = lambda nm: np.asarray(v[nm], dtype=np.float64)
    means = np.stack([f("x"), f("y"), f("z")], 1).astype(np.float32)
    scales = np.exp(np.stack([f(f"scale_{i}") for i in range(3)], 1)).astype(np.float32)
    q = np.stack([f(f"rot_{i}") for i in range(4)], 1)
    qn = np.linalg.norm(q, axis=1, keepdims=True)
    quats = np.where(qn > 0, q / np.where(qn > 0, qn, 1), q).astype(np.float32)  # q = 0 stays 0: load rejects it
    opac = (1.0 / (1.0 + np.exp(-f("opacity")))).astype(np.float32)
    sh = np.zeros((n, K, 3), dtype=np.float32)
    for c in range(3):
        sh[:, 0, c] = f(f"f_dc_{c}")
        for k in range(1, K):
            sh[:, k, c] = f(f"f_rest_{c * (K - 1) + k - 1}")
    vt = f("vtrain").astype(np.float32) if "vtrain" in names else np.full(n, np.inf, np.float32)
    return PlyScene(means, scales, quats, opac, sh, vt, deg)


def write_ply(path, scene, with_vtrain: bool = True) -> None:
    """Inverse of read_ply (log scales, logit opacities): for round trips and exports."""
    n = int(scene.means.shape[0])
    K = (scene.sh_degree + 1) ** 2
    cols = [("x", scene.means[:, 0]), ("y", scene.means[:, 1]), ("z", scene.means[:, 2]),
            ("nx", np.zeros(n)), ("ny", np.zeros(n)), ("nz", np.zeros(n))]
    sh = np.asarray(scene.sh, dtype=np.float64).reshape(n, K, 3)
    cols += [(f"f_dc_{c}", sh[:, 0, c]) for c in range(3)]
    cols += [(f"f_rest_{c * (K - 1) + k - 1}", sh[:, k, c]) for c in range(3) for k in range(1, K)]
    o = np.asarray(scene.opacities, dtype=np.float64)
    cols.append(("opacity", np.log(o) - np.log1p(-o)))
    cols += [(f"scale_{i}", np.log(np.asarray(scene.scales, dtype=np.float64)[:, i])) for i in range(3)]
    cols += [(f"rot_{i}", np.asarray(scene.quats, dtype=np.float64)[:, i]) for i in range(4)]
    if with_vtrain:
        cols.append(("vtrain", np.asarray(scene.v_train, dtype=np.float64)))
    dt = np.dtype([(nm, "<f4") for nm, _ in cols])
    rec = np.empty(n, dtype=dt)
    for nm, a in cols:
        rec[nm] = a
    hdr = ["ply", "format binary_little_endian 1.0", f"element vertex {n}"]
    hdr += [f"property float {nm}" for nm, _ in cols] + ["end_header"]
    with open(path, "wb") as fh:
        fh.write(("\n".join(hdr) + "\n").encode("ascii"))
        fh.write(rec.tobytes())
