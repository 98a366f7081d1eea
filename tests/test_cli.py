"""MRC2014 I/O (include/ballmatch_b200_io.hpp) and the ballmatch-b200 CLI contract
(reference tools/main.cpp:25-26: 0 ok, 2 usage, 3 non-convergence, 4 I/O)."""
import json
import subprocess
from pathlib import Path

import numpy as np
import pytest

from mrcio import read_mrc, write_mrc

ROOT = Path(__file__).resolve().parents[1]
CLI = ROOT / "paper_2509_01180_b200" / "bin" / "ballmatch-b200"


def _make_cpp():
    subprocess.run(["make", "-C", str(ROOT / "oracle")], check=True, capture_output=True)
    r = subprocess.run(["make", "-C", str(ROOT / "tests" / "cpp")], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


def test_mrc_reader_writer_modes_orders_errors(tmp_path):
    _make_cpp()
    z, y, x = np.meshgrid(np.arange(8), np.arange(8), np.arange(8), indexing="ij")
    v = (x + 10 * y + 100 * z - 50).astype(np.float64)  # stored x fastest: array [z][y][x]
    write_mrc(tmp_path / "m2_le.mrc", v, voxel=2.5)
    write_mrc(tmp_path / "m2_be.mrc", v, big_endian=True)
    write_mrc(tmp_path / "m0.mrc", ((x + y + z) % 100 - 50), mode=0)
    write_mrc(tmp_path / "m1.mrc", v, mode=1)
    write_mrc(tmp_path / "m6.mrc", v + 50, mode=6)
    # MAPC/MAPR/MAPS = 3,2,1: file columns run along z, rows along y, sections along x
    write_mrc(tmp_path / "m2_perm.mrc", np.transpose(v, (2, 1, 0)), axes=(3, 2, 1))
    write_mrc(tmp_path / "m2_ext.mrc", v, ext=96)
    write_mrc(tmp_path / "nostamp.mrc", v, stamp=False)
    write_mrc(tmp_path / "mode3.mrc", v, mode=3)
    write_mrc(tmp_path / "short.mrc", v, truncate=40)
    r = subprocess.run([str(ROOT / "tests" / "cpp" / "_build" / "test_mrc"), str(tmp_path)], capture_output=True,
                       text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert np.allclose(read_mrc(tmp_path / "rt_stack.mrc").shape, (16, 8, 8))


def test_cli_usage_and_io_exit_codes(tmp_path):
    assert CLI.exists(), "build first: __graft_entry__.build()"
    assert subprocess.run([str(CLI), "--version"], capture_output=True).returncode == 0
    assert subprocess.run([str(CLI)], capture_output=True).returncode == 2
    assert subprocess.run([str(CLI), "frobnicate"], capture_output=True).returncode == 2
    assert subprocess.run([str(CLI), "align", "--template", "t.mrc"], capture_output=True).returncode == 2
    r = subprocess.run([str(CLI), "align", "--template", str(tmp_path / "none.mrc"), "--subtomo", "x.mrc"],
                       capture_output=True, text=True)
    assert r.returncode == 4 and "not readable" in r.stderr
    write_mrc(tmp_path / "bad.mrc", np.zeros((8, 8, 8)), stamp=False)
    r = subprocess.run([str(CLI), "align-batch", "--template", str(tmp_path / "bad.mrc"), "--stack",
                        str(tmp_path / "bad.mrc")], capture_output=True, text=True)
    assert r.returncode == 4 and "MAP " in r.stderr
    r = subprocess.run([str(CLI), "align", "--template", "a", "--subtomo", "b", "--lmax", "x"], capture_output=True)
    assert r.returncode == 2


@pytest.mark.gpu
def test_cli_align_batch_matches_oracle(cuda_device, tmp_path):
    """align-batch on an MRC particle stack vs the oracle's align() per particle, plus
    the averaged map (synthesize of the coefficient-space average)."""
    import math

    from oracle import bmo
    n, L = 32, 8
    tmpl = bmo.gaussian_blob_template(n, 20, 7).astype(np.float32).astype(np.float64)
    parts = []
    for p in range(3):
        s, _, _ = bmo.make_particle(tmpl, 40 + p, 2, 1.0, 60.0)
        parts.append(s)
    write_mrc(tmp_path / "t.mrc", tmpl)
    write_mrc(tmp_path / "stack.mrc", np.concatenate(parts, axis=0))
    rep = tmp_path / "r.json"
    cmd = [str(CLI), "align-batch", "--template", str(tmp_path / "t.mrc"), "--stack", str(tmp_path / "stack.mrc"),
           "--bands", "4,8", "--lmax", "8", "--lambda-cut", str(8 * math.pi), "--max-candidates", "8",
           "--shift-radius", "2", "--wedge", "60", "--report", str(rep), "--average", str(tmp_path / "avg.mrc")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode in (0, 3), r.stdout + r.stderr
    res = json.loads(rep.read_text())["results"]
    ocfg = bmo.make_config(l_max=L, lambda_cut=8 * math.pi, bands=(4, 8), max_candidates=8, shift_radius=2)
    for p in range(3):
        ref = bmo.align(tmpl, parts[p], ocfg, wedge_deg=60.0)
        got = res[p]
        assert tuple(got["shift_voxels"]) == ref["shift"]
        assert bmo.geodesic_degrees(got["rotation"]["quaternion_wxyz"], ref["quat"]) < 0.5
        assert got["score"] == pytest.approx(ref["score"], rel=1e-4)
    avg = read_mrc(tmp_path / "avg.mrc")
    assert avg.shape == (n, n, n)
    assert np.corrcoef(avg.ravel(), tmpl.ravel())[0, 1] > 0.5
