"""Interchange formats (reference pkg/src/paball/formats.py): byte-identical
writers and value-identical readers against files the reference wrote
(tests/golden/make_golden_formats.py), round trips, and every rejection the
reference reader makes (bad magic, version, truncation, trailing bytes, CSV
header / width / non-numeric)."""

import os
import shutil
import struct

import numpy as np
import pytest

from paper_2601_00551_b200 import formats as F
from paper_2601_00551_b200.model import (FormatError, PointCloud, SensorArray, SignalSet, TimeGrid,
                                         VoxelGrid)

GD = os.path.join(os.path.dirname(__file__), "golden", "formats")
VALS = np.load(os.path.join(GD, "values.npz"))


def raw(name):
    with open(os.path.join(GD, name), "rb") as fh:
        return fh.read()


def rewrite(tmp_path, name, writer, obj):
    out = tmp_path / name
    writer(out, obj)
    return out.read_bytes()


class TestReferenceFiles:
    def test_signals(self, tmp_path):
        s = F.read_signals(os.path.join(GD, "sig.pasg"))
        assert s.data.shape == (3, 5) and s.grid.t0 == -1.25e-6 and s.grid.dt == 2.5e-8
        assert s.data.dtype == np.float64
        assert rewrite(tmp_path, "s.pasg", F.write_signals, s) == raw("sig.pasg")

    @pytest.mark.gpu
    def test_signals_pinned_same_values(self):
        a = F.read_signals(os.path.join(GD, "sig.pasg"))
        b = F.read_signals(os.path.join(GD, "sig.pasg"), pinned=True)
        np.testing.assert_array_equal(a.data, b.data)

    def test_cloud(self, tmp_path):
        c = F.read_cloud(os.path.join(GD, "cloud.pcbg"))
        assert len(c) == 4
        assert rewrite(tmp_path, "c.pcbg", F.write_cloud, c) == raw("cloud.pcbg")

    def test_volume(self, tmp_path):
        v = F.read_volume(os.path.join(GD, "vol.pavx"))
        assert v.dims == (3, 4, 2) and v.spacing == 2.5e-4
        np.testing.assert_array_equal(v.origin, [-1e-3, 2e-3, 0.5e-3])
        # x fastest on disk
        flat = np.frombuffer(raw("vol.pavx")[52:], "<f4")
        assert flat[1] == np.float32(v.values[1, 0, 0]) and flat[3] == np.float32(v.values[0, 1, 0])
        assert rewrite(tmp_path, "v.pavx", F.write_volume, v) == raw("vol.pavx")

    @pytest.mark.parametrize("name,width", [("sensors3.csv", 3), ("sensors6.csv", 6)])
    def test_sensor_csv(self, tmp_path, name, width):
        a = F.read_sensors_csv(os.path.join(GD, name), sound_speed=1480.0)
        np.testing.assert_array_equal(a.positions, VALS["pos"])
        assert a.sound_speed == 1480.0
        if width == 6:
            np.testing.assert_array_equal(a.normals, VALS["nrm"])
        else:
            assert a.normals is None
        assert rewrite(tmp_path, name, F.write_sensors_csv, a) == raw(name)

    def test_images(self, tmp_path):
        F.write_pgm(tmp_path / "i.pgm", VALS["img"])
        F.write_float_sidecar(tmp_path / "i.f32", VALS["img"])
        assert (tmp_path / "i.pgm").read_bytes() == raw("img.pgm")
        assert (tmp_path / "i.f32").read_bytes() == raw("img.f32")


class TestRoundTrips:
    def test_signals_f32_rounding(self, tmp_path):
        data = np.random.default_rng(0).standard_normal((4, 7))
        F.write_signals(tmp_path / "a.pasg", SignalSet(TimeGrid(0.0, 1e-8, 7), data))
        back = F.read_signals(tmp_path / "a.pasg")
        np.testing.assert_array_equal(back.data, data.astype(np.float32).astype(np.float64))

    def test_empty_cloud(self, tmp_path):
        F.write_cloud(tmp_path / "e.pcbg", PointCloud.empty())
        assert len(F.read_cloud(tmp_path / "e.pcbg")) == 0
        assert (tmp_path / "e.pcbg").stat().st_size == 12

    def test_volume_ragged(self, tmp_path):
        vals = np.arange(5 * 2 * 3, dtype=np.float64).reshape(5, 2, 3)
        F.write_volume(tmp_path / "r.pavx", VoxelGrid((5, 2, 3), 1e-3, np.zeros(3), vals))
        np.testing.assert_array_equal(F.read_volume(tmp_path / "r.pavx").values, vals)

    def test_pgm_all_zero_and_header(self, tmp_path):
        F.write_pgm(tmp_path / "z.pgm", np.zeros((2, 3)))
        b = (tmp_path / "z.pgm").read_bytes()
        assert b.startswith(b"P5\n3 2\n65535\n") and b.endswith(b"\x00" * 12)
        with pytest.raises(ValueError):
            F.write_pgm(tmp_path / "bad.pgm", np.zeros(4))


class TestRejections:
    def corrupt(self, tmp_path, name, data):
        p = tmp_path / name
        p.write_bytes(data)
        return p

    def test_bad_magic(self, tmp_path):
        p = self.corrupt(tmp_path, "m.pasg", b"PCBG" + raw("sig.pasg")[4:])
        with pytest.raises(FormatError, match="bad magic at byte 0"):
            F.read_signals(p)

    def test_bad_version(self, tmp_path):
        p = self.corrupt(tmp_path, "v.pcbg", raw("cloud.pcbg")[:4] + struct.pack("<I", 2) + raw("cloud.pcbg")[8:])
        with pytest.raises(FormatError, match="version 2 at byte 4"):
            F.read_cloud(p)

    @pytest.mark.parametrize("cut,what", [(2, "magic at byte 0"), (6, "version at byte 4"),
                                          (20, "signals header at byte 8"), (40, "signal samples at byte 32")])
    def test_truncations_name_their_byte(self, tmp_path, cut, what):
        p = self.corrupt(tmp_path, "t.pasg", raw("sig.pasg")[:cut])
        with pytest.raises(FormatError, match=what):
            F.read_signals(p)

    def test_volume_truncated_origin(self, tmp_path):
        p = self.corrupt(tmp_path, "o.pavx", raw("vol.pavx")[:40])
        with pytest.raises(FormatError, match="volume origin at byte 28"):
            F.read_volume(p)

    def test_trailing_bytes(self, tmp_path):
        p = self.corrupt(tmp_path, "x.pcbg", raw("cloud.pcbg") + b"\x00\x01")
        with pytest.raises(FormatError, match="2 unexpected trailing bytes at byte 92"):
            F.read_cloud(p)

    def test_missing_file(self, tmp_path):
        with pytest.raises(FormatError, match="cannot read"):
            F.read_volume(tmp_path / "nope.pavx")

    def test_csv_rejections(self, tmp_path):
        cases = {"empty.csv": ("\n\n", "empty sensor file"), "hdr.csv": ("a,b,c\n1,2,3\n", "bad header"),
                 "width.csv": ("x,y,z\n1,2\n", "line 2 has 2 fields"),
                 "num.csv": ("x,y,z\n1,2,3\n1,q,3\n", "line 3 is not numeric")}
        for name, (text, msg) in cases.items():
            (tmp_path / name).write_text(text)
            with pytest.raises(FormatError, match=msg):
                F.read_sensors_csv(tmp_path / name)

    def test_csv_blank_lines_and_spaced_header(self, tmp_path):
        (tmp_path / "s.csv").write_text("x, y, z\n\n1,2,3\n\n4,5,6\n")
        a = F.read_sensors_csv(tmp_path / "s.csv")
        np.testing.assert_array_equal(a.positions, [[1, 2, 3], [4, 5, 6]])
