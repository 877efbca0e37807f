"""Snapshot format and CLI against the reference's own outputs
(tests/golden/cli.npz, written by the reference CLI / save_field).  CPU-only parts."""

import numpy as np
import pytest

from paper_1806_01422_b200 import cli
from paper_1806_01422_b200.errors import ValidationError
from paper_1806_01422_b200.grid import grid_1d, load_field, save_field
from semtest_util import golden


def _body(text):
    return [ln for ln in text.splitlines() if not ln.startswith("#")]


def test_snapshot_bytes_identical_and_roundtrip(tmp_path):
    g = golden("cli.npz")
    grid = grid_1d(-1.0, 1.0, 3, 4, "dirichlet0")
    path = tmp_path / "s.field"
    save_field(str(path), grid, g["snapshot_values"])
    assert path.read_bytes() == bytes(g["snapshot"])            # byte-identical to the reference
    ref = tmp_path / "ref.field"
    ref.write_bytes(bytes(g["snapshot"]))
    gr, vals = load_field(str(ref))
    assert gr.nglobal == grid.nglobal and gr.axis.bc == "dirichlet0" and gr.axis.degree == 4
    assert np.array_equal(vals, g["snapshot_values"])          # bit-exact round trip
    fwd = tmp_path / "fwd.field"
    fwd.write_bytes(bytes(g["forward_field"]))
    gf, vf = load_field(str(fwd))
    save_field(str(tmp_path / "again.field"), gf, vf)
    assert (tmp_path / "again.field").read_bytes() == bytes(g["forward_field"])


def test_snapshot_errors(tmp_path):
    bad = tmp_path / "bad.field"
    bad.write_bytes(b"not a snapshot\nend-header\n")
    with pytest.raises(ValidationError):
        load_field(str(bad))
    g = golden("cli.npz")
    trunc = tmp_path / "trunc.field"
    trunc.write_bytes(bytes(g["snapshot"])[:-16])
    with pytest.raises(ValidationError):
        load_field(str(trunc))
    with pytest.raises(ValidationError):
        save_field(str(tmp_path / "x.field"), grid_1d(-1.0, 1.0, 3, 4), np.zeros(5))


def test_schedule_command_matches_reference(tmp_path):
    g = golden("cli.npz")
    out = tmp_path / "sched.csv"
    assert cli.main(["schedule", "--steps", "30", "--checkpoint-slots", "5", "--output", str(out)]) == 0
    ref = bytes(g["schedule"]).decode()
    assert _body(out.read_text()) == _body(ref)
    mine = [ln for ln in out.read_text().splitlines() if ln.startswith("# ")][1:]
    assert mine == [ln for ln in ref.splitlines() if ln.startswith("# ")][1:]   # steps/slots/recomputed


def test_exit_codes_and_config(tmp_path):
    assert cli.main(["forward", "--problem", "nosuch", "--output", str(tmp_path / "x")]) == 2
    assert cli.main(["forward", "--bogus"]) == 2
    assert cli.main(["schedule"]) == 2                              # --steps is required
    cfg = tmp_path / "c.cfg"
    cfg.write_text("nonexistent_key = 3\n")
    assert cli.main(["forward", "--config", str(cfg), "--output", str(tmp_path / "x")]) == 2
    cfg.write_text("problem = diffusion1d  # comment\nsteps = 12\nadaptive = true\ndt = 1e-3\n")
    vals = cli._read_config(str(cfg), cli.build_parser())
    assert vals == {"problem": "diffusion1d", "steps": 12, "adaptive": True, "dt": 1e-3}
    # file entries are defaults: an invalid grid from the file is a validation error (2)
    cfg.write_text("elements = 0\n")
    assert cli.main(["forward", "--config", str(cfg), "--output", str(tmp_path / "x")]) == 2
