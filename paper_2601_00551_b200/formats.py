"""On-disk interchange with the reference CLI (reference ``paball/formats.py``).

Little-endian binaries, 4-byte magic + u32 version 1 (formats.py:1-14):

  PASG  signals: u32 n_sensors, u32 n_samples, f64 t0, f64 dt, f32 rows
        (sensor-major)                                   formats.py:97-113
  PCBG  cloud:   u32 count, f32 (x, y, z, p0, a0) per ball  formats.py:121-140
  PAVX  volume:  u32 dx, dy, dz, f64 spacing, f64 origin[3], f32 values with x
        fastest                                          formats.py:148-166

plus the sensor CSV (``x,y,z[,nx,ny,nz]``, formats.py:174-216) and the 16-bit
PGM / raw float32 image pair (formats.py:224-242).  Files written here are
byte-identical to the reference writer's; readers reject foreign magics and
versions and name the byte offset of a truncation or trailing garbage
(``FormatError``).

Headers are numpy structured dtypes; payloads are decoded from the file image
in one vectorised pass, for PASG optionally straight into page-locked host
memory (``read_signals(path, pinned=True)``) so the FP64 rows are ready for the
device upload without a further staging copy.
"""

from __future__ import annotations

from pathlib import Path

import numpy as np

from .model import FormatError, PointCloud, SensorArray, SignalSet, TimeGrid, VoxelGrid

__all__ = ["write_signals", "read_signals", "write_cloud", "read_cloud", "write_volume", "read_volume",
           "write_sensors_csv", "read_sensors_csv", "write_pgm", "write_float_sidecar"]

VERSION = 1
_PREAMBLE = np.dtype([("magic", "S4"), ("version", "<u4")])
_HEAD = {
    b"PASG": ("signals", np.dtype([("n_sensors", "<u4"), ("n_samples", "<u4"), ("t0", "<f8"), ("dt", "<f8")])),
    b"PCBG": ("cloud", np.dtype([("count", "<u4")])),
    b"PAVX": ("volume", np.dtype([("dims", "<u4", (3,)), ("spacing", "<f8"), ("origin", "<f8", (3,))])),
}
# the reference reads the PAVX origin as its own record (formats.py:159-160)
_PAVX_PARTS = ((20, "volume header"), (24, "volume origin"))


class _Blob:
    """A whole file in memory with a read cursor; every failure names its byte."""

    def __init__(self, path):
        self.path = Path(path)
        try:
            self.buf = memoryview(self.path.read_bytes())
        except OSError as exc:
            raise FormatError(f"cannot read {path}: {exc}") from exc
        self.at = 0

    def need(self, n: int, what: str) -> int:
        left = len(self.buf) - self.at
        if n > left:
            raise FormatError(f"{self.path}: truncated {what} at byte {self.at} "
                              f"(wanted {n} bytes, file has {left} left)")
        start, self.at = self.at, self.at + n
        return start

    def record(self, dtype: np.dtype, what: str):
        start = self.need(dtype.itemsize, what)
        return np.frombuffer(self.buf, dtype=dtype, count=1, offset=start)[0]

    def payload(self, dtype: str, count: int, what: str, out: np.ndarray | None = None) -> np.ndarray:
        dt = np.dtype(dtype)
        start = self.need(dt.itemsize * count, what)
        src = np.frombuffer(self.buf, dtype=dt, count=count, offset=start)
        if out is None:
            return src
        out.reshape(-1)[...] = src
        return out

    def done(self) -> None:
        extra = len(self.buf) - self.at
        if extra:
            raise FormatError(f"{self.path}: {extra} unexpected trailing bytes at byte {self.at}")


def _open(path, magic: bytes) -> tuple[_Blob, str]:
    name, _ = _HEAD[magic]
    b = _Blob(path)
    start = b.need(4, f"{name} magic")
    got = bytes(b.buf[start:start + 4])
    if got != magic:
        raise FormatError(f"{b.path}: bad magic at byte 0: expected {magic!r}, got {got!r}")
    start = b.need(4, f"{name} version")
    version = int(np.frombuffer(b.buf, "<u4", 1, start)[0])
    if version != VERSION:
        raise FormatError(f"{b.path}: unsupported {name} version {version} at byte 4 (reader supports {VERSION})")
    return b, name


def _write(path, magic: bytes, head: np.ndarray, body: np.ndarray) -> None:
    pre = np.array([(magic, VERSION)], dtype=_PREAMBLE)
    with open(path, "wb") as fh:
        fh.write(pre.tobytes())
        fh.write(head.tobytes())
        fh.write(np.ascontiguousarray(body).tobytes())


# ---- signals --------------------------------------------------------------

def write_signals(path, signals: SignalSet) -> None:
    """PASG v1 (formats.py:97-104); samples rounded to f32."""
    head = np.zeros(1, _HEAD[b"PASG"][1])
    head["n_sensors"], head["n_samples"] = signals.n_sensors, signals.grid.n_samples
    head["t0"], head["dt"] = signals.grid.t0, signals.grid.dt
    _write(path, b"PASG", head, np.asarray(signals.data).astype("<f4"))


def read_signals(path, pinned: bool = False) -> SignalSet:
    """PASG v1 (formats.py:107-113) -> FP64 SignalSet.  ``pinned`` widens the
    samples straight into page-locked host memory (device-upload ready)."""
    b, _ = _open(path, b"PASG")
    h = b.record(_HEAD[b"PASG"][1], "signals header")
    j, n = int(h["n_sensors"]), int(h["n_samples"])
    out = None
    if pinned:
        import torch
        out = torch.empty((j, n), dtype=torch.float64, pin_memory=True).numpy()
    rows = b.payload("<f4", j * n, "signal samples", out)
    b.done()
    data = rows.reshape(j, n) if out is not None else rows.astype(np.float64).reshape(j, n)
    return SignalSet(TimeGrid(float(h["t0"]), float(h["dt"]), n), data)


# ---- point clouds ---------------------------------------------------------

def write_cloud(path, cloud: PointCloud) -> None:
    """PCBG v1 (formats.py:121-130): f32 (x, y, z, p0, a0) per ball."""
    rec = np.column_stack([np.asarray(cloud.positions).reshape(-1, 3), cloud.p0, cloud.a0]).astype("<f4")
    _write(path, b"PCBG", np.array([len(cloud)], "<u4"), rec)


def read_cloud(path) -> PointCloud:
    """PCBG v1 (formats.py:133-140) -> FP64 PointCloud."""
    b, _ = _open(path, b"PCBG")
    n = int(b.record(_HEAD[b"PCBG"][1], "ball count")["count"])
    rec = b.payload("<f4", 5 * n, "ball records").astype(np.float64).reshape(n, 5)
    b.done()
    return PointCloud(rec[:, 0:3], rec[:, 3], rec[:, 4])


# ---- volumes --------------------------------------------------------------

def write_volume(path, grid: VoxelGrid) -> None:
    """PAVX v1 (formats.py:148-155): x fastest on disk."""
    head = np.zeros(1, _HEAD[b"PAVX"][1])
    head["dims"], head["spacing"], head["origin"] = grid.dims, grid.spacing, grid.origin
    _write(path, b"PAVX", head, np.asarray(grid.values, dtype="<f4").transpose(2, 1, 0))


def read_volume(path) -> VoxelGrid:
    """PAVX v1 (formats.py:158-166)."""
    b, _ = _open(path, b"PAVX")
    (n_dims, w_dims), (n_org, w_org) = _PAVX_PARTS
    s = b.need(n_dims, w_dims)
    dims = tuple(int(d) for d in np.frombuffer(b.buf, "<u4", 3, s))
    spacing = float(np.frombuffer(b.buf, "<f8", 1, s + 12)[0])
    s = b.need(n_org, w_org)
    origin = np.frombuffer(b.buf, "<f8", 3, s).copy()
    flat = b.payload("<f4", dims[0] * dims[1] * dims[2], "voxel values")
    b.done()
    values = flat.astype(np.float64).reshape(dims[::-1]).transpose(2, 1, 0)
    return VoxelGrid(dims, spacing, origin, np.ascontiguousarray(values))


# ---- sensor CSV -----------------------------------------------------------

_CSV_WIDTH = {"x,y,z": 3, "x,y,z,nx,ny,nz": 6}


def write_sensors_csv(path, array: SensorArray) -> None:
    """Header ``x,y,z`` or ``x,y,z,nx,ny,nz``, %.17g fields (formats.py:174-185)."""
    cols = array.positions if array.normals is None else np.hstack([array.positions, array.normals])
    head = "x,y,z" if array.normals is None else "x,y,z,nx,ny,nz"
    body = "".join(",".join(f"{v:.17g}" for v in row) + "\n" for row in cols)
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        fh.write(head + "\n" + body)


def read_sensors_csv(path, sound_speed: float = 1500.0) -> SensorArray:
    """Inverse of ``write_sensors_csv`` (formats.py:188-216); blank lines ignored."""
    path = Path(path)
    try:
        text = path.read_text(encoding="utf-8")
    except OSError as exc:
        raise FormatError(f"cannot read {path}: {exc}") from exc
    lines = [ln.strip() for ln in text.splitlines()]
    lines = [ln for ln in lines if ln]
    if not lines:
        raise FormatError(f"{path}: empty sensor file at byte 0")
    width = _CSV_WIDTH.get(lines[0].replace(" ", ""))
    if width is None:
        raise FormatError(f"{path}: bad header at byte 0: expected 'x,y,z[,nx,ny,nz]', got {lines[0]!r}")
    data = np.empty((len(lines) - 1, width))
    for row, ln in enumerate(lines[1:]):
        fields = ln.split(",")
        if len(fields) != width:
            raise FormatError(f"{path}: line {row + 2} has {len(fields)} fields, expected {width}")
        try:
            data[row] = [float(x) for x in fields]
        except ValueError as exc:
            raise FormatError(f"{path}: line {row + 2} is not numeric: {ln!r}") from exc
    return SensorArray(data[:, :3], sound_speed=sound_speed, normals=data[:, 3:] if width == 6 else None)


# ---- images ---------------------------------------------------------------

def write_pgm(path, image: np.ndarray) -> None:
    """Binary 16-bit PGM (P5, big-endian samples), max-normalised (formats.py:224-236)."""
    img = np.asarray(image, dtype=np.float64)
    if img.ndim != 2:
        raise ValueError("PGM image must be 2D")
    top = img.max()
    scaled = img / top if top > 0.0 else np.zeros_like(img)
    level = np.clip(np.rint(scaled * 65535.0), 0, 65535).astype(">u2")
    with open(path, "wb") as fh:
        fh.write(b"P5\n%d %d\n65535\n" % (img.shape[1], img.shape[0]))
        fh.write(level.tobytes())


def write_float_sidecar(path, image: np.ndarray) -> None:
    """Raw little-endian float32, row-major (formats.py:239-243)."""
    with open(path, "wb") as fh:
        fh.write(np.ascontiguousarray(image, dtype="<f4").tobytes())
