"""Binary sidecar formats for the two bulk inputs of the fit.

The reference exchanges grain maps and parameter matrices as CSV text
(fileio.py:36-44, 101-111 ``x1,x2,label`` rows; fileio.py:114-179 the theta
table with its ``# basis=...`` line).  At c5 that is 4.2 M text rows parsed
field by field before the first evaluation.  The sidecars hold the same
information as flat little-endian arrays that load with one read (or a memory
map) into exactly the dtypes ``pgx_problem_create`` / ``pgx_eval`` take:

``.pgxg`` grain map   64-byte header | labels (uint16 when N < 65536, else int32;
                      1-based as in the CSV) | float64 points (point lists only:
                      a regular grid stores its resolution, fileio.py:89-98)
``.pgxt`` theta       64-byte header | float64 K x N row-major (basis.py:287-327)

Both carry a CRC-32 of the payload; a truncated or corrupted file raises
``InputFormatError`` like the reference's CSV readers do for malformed text.
The CSV readers / writers here follow the reference's text formats, so a
sidecar can be produced from (and turned back into) the reference's own files.
"""

from __future__ import annotations

import struct
import zlib
from pathlib import Path

import numpy as np

from .basis import BASIS_KINDS, GAUGE_FREE, GAUGE_LAST_ZERO, ORDERING_CONVENTION, DesignBasis, ParamMatrix
from .errors import InputFormatError
from .geometry import GrainMap, PixelGrid, make_grid

MAGIC_MAP = b"PGXG"
MAGIC_THETA = b"PGXT"
VERSION = 1
# magic, version, dim, resolution (0 = point list), n_points, n_grains, label dtype code,
# payload crc32, padding to 64 bytes
_HDR_MAP = struct.Struct("<4sIIIQIII28x")
# magic, version, dim, degree, K, N, kind code, gauge code, payload crc32, padding to 64 bytes
_HDR_THETA = struct.Struct("<4sIIIIIIII28x")
assert _HDR_MAP.size == 64 and _HDR_THETA.size == 64
_LABEL_DTYPES = {2: np.dtype("<u2"), 4: np.dtype("<i4")}
_GAUGES = (GAUGE_FREE, GAUGE_LAST_ZERO)


# ---------------------------------------------------------------- grain maps
def write_grain_map_bin(path, grain_map) -> None:
    """Write a grain map (labels 1..N over a regular grid or a point list)."""
    grid = grain_map.grid
    labels = np.asarray(grain_map.labels)
    n = int(grain_map.n_grains)
    code = 2 if n < 65536 else 4
    lab = np.ascontiguousarray(labels, dtype=_LABEL_DTYPES[code])
    res = getattr(grid, "resolution", None)
    dim = int(getattr(grid, "dim", 2))
    payload = [lab.tobytes()]
    if res is None:
        payload.append(np.ascontiguousarray(grid.points, dtype="<f8").tobytes())
    crc = 0
    for part in payload:
        crc = zlib.crc32(part, crc)
    with open(path, "wb") as fh:
        fh.write(_HDR_MAP.pack(MAGIC_MAP, VERSION, dim, int(res or 0), lab.size, n, code, crc))
        for part in payload:
            fh.write(part)


def read_grain_map_bin(path, *, verify: bool = True) -> GrainMap:
    """Read a ``.pgxg`` sidecar; labels come back as one contiguous int64 array
    (the package's GrainMap dtype) converted from the stored narrow type in one pass."""
    raw = np.memmap(path, dtype=np.uint8, mode="r")
    if raw.size < 64:
        raise InputFormatError(f"{path}: shorter than the 64-byte header")
    magic, version, dim, res, n_points, n_grains, code, crc = _HDR_MAP.unpack(bytes(raw[:64]))
    if magic != MAGIC_MAP:
        raise InputFormatError(f"{path}: not a grain-map sidecar (magic {magic!r})")
    if version != VERSION:
        raise InputFormatError(f"{path}: unsupported version {version}")
    if code not in _LABEL_DTYPES or dim not in (2, 3) or n_points < 2 or n_grains < 2:
        raise InputFormatError(f"{path}: malformed header")
    lab_bytes = n_points * code
    pts_bytes = 0 if res else n_points * dim * 8
    if raw.size != 64 + lab_bytes + pts_bytes:
        raise InputFormatError(
            f"{path}: expected {64 + lab_bytes + pts_bytes} bytes for {n_points} pixels, got {raw.size}")
    if verify and zlib.crc32(raw[64:]) != crc:
        raise InputFormatError(f"{path}: payload checksum mismatch")
    labels = np.frombuffer(raw, dtype=_LABEL_DTYPES[code], count=n_points, offset=64).astype(np.int64)
    if labels.min() < 1 or labels.max() > n_grains:
        raise InputFormatError(f"{path}: labels must lie in 1..{n_grains}")
    if res:
        if (2 * res) ** dim != n_points:
            raise InputFormatError(f"{path}: resolution {res} does not match {n_points} pixels")
        grid = make_grid(res, dim)
    else:
        pts = np.frombuffer(raw, dtype="<f8", count=n_points * dim, offset=64 + lab_bytes)
        try:
            grid = PixelGrid(points=pts.reshape(n_points, dim).copy())
        except ValueError as exc:
            raise InputFormatError(f"{path}: {exc}") from None
    return GrainMap(grid=grid, labels=labels, n_grains=n_grains)


def _infer_resolution(points: np.ndarray):
    """M when the points are exactly the canonical regular 2-D grid (fileio.py:89-98)."""
    n = points.shape[0]
    side = int(round(n ** 0.5))
    if side * side != n or side % 2 != 0 or points.shape[1] != 2:
        return None
    m = side // 2
    return m if np.array_equal(points, make_grid(m).points) else None


def read_grain_map_csv(path) -> GrainMap:
    """The reference's ``x1,x2,label`` text format (fileio.py:101-111), parsed in bulk."""
    with open(path, newline="") as fh:
        header = fh.readline()
        if not header:
            raise InputFormatError(f"{path}: empty file")
        if [h.strip() for h in header.strip().split(",")] != ["x1", "x2", "label"]:
            raise InputFormatError(f"{path}: expected header 'x1,x2,label', got {header.strip()!r}")
        rows = [ln for ln in fh.read().splitlines() if ln.strip()]
    if len(rows) < 2:
        raise InputFormatError(f"{path}: need at least two pixels")
    pts = np.empty((len(rows), 2))
    labels = np.empty(len(rows), dtype=np.int64)
    for i, ln in enumerate(rows):
        f = ln.split(",")
        if len(f) != 3:
            raise InputFormatError(f"{path}: row {i + 2}: expected 3 fields, got {len(f)}")
        try:
            pts[i, 0], pts[i, 1] = float(f[0]), float(f[1])
        except ValueError:
            raise InputFormatError(f"row {i + 2}: not a number: {ln!r}") from None
        try:
            labels[i] = int(f[2])
        except ValueError:
            raise InputFormatError(f"row {i + 2}, column 'label': not an integer: {f[2]!r}") from None
        if labels[i] < 1:
            raise InputFormatError(f"row {i + 2}, column 'label': labels are 1-based, got {labels[i]}")
    try:
        grid = PixelGrid(points=pts, resolution=_infer_resolution(pts))
    except ValueError as exc:
        raise InputFormatError(f"{path}: {exc}") from None
    return GrainMap(grid=grid, labels=labels, n_grains=int(labels.max()))


def write_grain_map_csv(path, grain_map) -> None:
    """fileio.py:36-44 (repr-exact floats, one row per pixel)."""
    pts = grain_map.grid.points
    lines = ["x1,x2,label"]
    lines += [f"{float(x1)!r},{float(x2)!r},{int(lab)}" for (x1, x2), lab in zip(pts, grain_map.labels)]
    Path(path).write_text("\n".join(lines) + "\n")


# ---------------------------------------------------------------- theta
def write_theta_bin(path, theta: ParamMatrix) -> None:
    vals = np.ascontiguousarray(theta.values, dtype="<f8")
    basis = theta.basis
    payload = vals.tobytes()
    with open(path, "wb") as fh:
        fh.write(_HDR_THETA.pack(MAGIC_THETA, VERSION, int(getattr(basis, "dim", 2)), int(basis.degree),
                                 vals.shape[0], vals.shape[1], BASIS_KINDS.index(basis.kind),
                                 _GAUGES.index(theta.gauge), zlib.crc32(payload)))
        fh.write(payload)


def read_theta_bin(path, *, verify: bool = True) -> ParamMatrix:
    raw = np.memmap(path, dtype=np.uint8, mode="r")
    if raw.size < 64:
        raise InputFormatError(f"{path}: shorter than the 64-byte header")
    magic, version, dim, degree, k, n, kind, gauge, crc = _HDR_THETA.unpack(bytes(raw[:64]))
    if magic != MAGIC_THETA:
        raise InputFormatError(f"{path}: not a theta sidecar (magic {magic!r})")
    if version != VERSION:
        raise InputFormatError(f"{path}: unsupported version {version}")
    if kind >= len(BASIS_KINDS) or gauge >= len(_GAUGES) or dim not in (2, 3) or n < 2:
        raise InputFormatError(f"{path}: malformed header")
    basis = DesignBasis.make(BASIS_KINDS[kind], degree, dim)
    if k != basis.dimension:
        raise InputFormatError(f"{path}: {k} rows, but degree {degree} in {dim}-D has {basis.dimension}")
    if raw.size != 64 + k * n * 8:
        raise InputFormatError(f"{path}: expected {64 + k * n * 8} bytes for a {k} x {n} matrix, got {raw.size}")
    if verify and zlib.crc32(raw[64:]) != crc:
        raise InputFormatError(f"{path}: payload checksum mismatch")
    vals = np.frombuffer(raw, dtype="<f8", count=k * n, offset=64).reshape(k, n).copy()
    try:
        return ParamMatrix(values=vals, basis=basis, gauge=_GAUGES[gauge])
    except ValueError as exc:
        raise InputFormatError(f"{path}: {exc}") from None


def write_theta_csv(path, theta: ParamMatrix) -> None:
    """The reference's theta table (fileio.py:114-124): a ``# basis=...`` line,
    ``alpha1,alpha2,theta_1..theta_N`` and one repr-exact row per multi-index (2-D)."""
    idx = theta.basis.index_set.indices
    if len(idx[0]) != 2:
        raise ValueError("the CSV theta format is two-dimensional; use the binary sidecar")
    n = theta.n_grains
    lines = [f"# basis={theta.basis.kind},degree={theta.degree},ordering={ORDERING_CONVENTION},"
             f"gauge={theta.gauge}",
             "alpha1,alpha2," + ",".join(f"theta_{i}" for i in range(1, n + 1))]
    for row, (a1, a2) in enumerate(idx):
        lines.append(f"{a1},{a2}," + ",".join(repr(float(v)) for v in theta.values[row]))
    Path(path).write_text("\n".join(lines) + "\n")


def read_theta_csv(path) -> ParamMatrix:
    """fileio.py:127-179."""
    text = Path(path).read_text().splitlines()
    if not text or not text[0].startswith("#"):
        raise InputFormatError(f"{path}: missing '# basis=...' metadata line")
    meta = {}
    for item in text[0][1:].strip().split(","):
        if "=" not in item:
            raise InputFormatError(f"{path}: malformed metadata item {item!r}")
        key, value = item.split("=", 1)
        meta[key.strip()] = value.strip()
    if meta.get("basis") not in BASIS_KINDS:
        raise InputFormatError(f"{path}: unknown basis kind {meta.get('basis')!r}")
    try:
        degree = int(meta.get("degree", ""))
    except ValueError:
        raise InputFormatError(f"{path}: bad degree {meta.get('degree')!r}") from None
    if meta.get("ordering") != ORDERING_CONVENTION:
        raise InputFormatError(f"{path}: ordering {meta.get('ordering')!r} not supported "
                               f"(expected {ORDERING_CONVENTION!r})")
    gauge = meta.get("gauge", GAUGE_FREE)
    if gauge not in _GAUGES:
        raise InputFormatError(f"{path}: unknown gauge {gauge!r}")
    basis = DesignBasis.make(meta["basis"], degree)
    if len(text) < 2 or [h.strip() for h in text[1].split(",")][:2] != ["alpha1", "alpha2"]:
        raise InputFormatError(f"{path}: expected header starting with alpha1,alpha2")
    n = len(text[1].split(",")) - 2
    if n < 2:
        raise InputFormatError(f"{path}: need at least two coefficient columns")
    values = np.zeros((basis.dimension, n))
    seen = 0
    for i, ln in enumerate(text[2:], start=3):
        if not ln.strip():
            continue
        f = ln.split(",")
        if len(f) != n + 2:
            raise InputFormatError(f"{path}: row {i}: expected {n + 2} fields, got {len(f)}")
        try:
            pos = basis.index_set.position((int(f[0]), int(f[1])))
            values[pos] = [float(v) for v in f[2:]]
        except ValueError as exc:
            raise InputFormatError(f"{path}: row {i}: {exc}") from None
        seen += 1
    if seen != basis.dimension:
        raise InputFormatError(
            f"{path}: expected {basis.dimension} coefficient rows for degree {degree}, got {seen}")
    try:
        return ParamMatrix(values=values, basis=basis, gauge=gauge)
    except ValueError as exc:
        raise InputFormatError(f"{path}: {exc}") from None


# ---------------------------------------------------------------- conversions
def grain_map_csv_to_bin(csv_path, bin_path) -> GrainMap:
    gm = read_grain_map_csv(csv_path)
    write_grain_map_bin(bin_path, gm)
    return gm


def theta_csv_to_bin(csv_path, bin_path) -> ParamMatrix:
    th = read_theta_csv(csv_path)
    write_theta_bin(bin_path, th)
    return th
