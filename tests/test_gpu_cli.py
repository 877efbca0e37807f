"""CLI commands on the GPU backend vs the reference CLI's own outputs (tests/golden/cli.npz)."""

import io

import numpy as np
import pytest

from paper_1806_01422_b200 import cli
from paper_1806_01422_b200.grid import load_field
from semtest_util import golden, rel_err

pytestmark = pytest.mark.gpu


def _rows(text):
    lines = [ln for ln in text.splitlines() if not ln.startswith("#")]
    return lines[0], [ln.split(",") for ln in lines[1:]]


def _meta(text, key):
    for ln in text.splitlines():
        if ln.startswith(f"# {key} = "):
            return ln.split(" = ", 1)[1]
    return None


@pytest.mark.parametrize("name,extra", [("forward", []), ("forward_cn", ["--scheme", "cn"])])
def test_forward_command_matches_reference(cuda, tmp_path, name, extra):
    g = golden("cli.npz")
    steps = "40" if name == "forward" else "8"
    argv = ["forward", "--problem", "burgers1d", "--elements", "5", "--degree", "8", "--steps", steps,
            "--horizon", "0.4", "--output", str(tmp_path / "f")] + extra
    assert cli.main(argv) == 0
    mine = (tmp_path / "f.csv").read_text()
    ref = bytes(g[f"{name}_csv"]).decode()
    hm, rm = _rows(mine)
    hr, rr = _rows(ref)
    assert hm == hr and len(rm) == len(rr)
    for a, b in zip(rm, rr):                         # fixed-dt step log: identical text
        assert a == b
    assert abs(float(_meta(mine, "terminal_l2_error")) - float(_meta(ref, "terminal_l2_error"))) <= \
        1e-10 * float(_meta(ref, "terminal_l2_error"))
    _, vm = load_field(str(tmp_path / "f.field"))
    refp = tmp_path / "ref.field"
    refp.write_bytes(bytes(g[f"{name}_field"]))
    _, vr = load_field(str(refp))
    assert rel_err(vm, vr) <= 1e-12


def test_gradcheck_command_matches_reference(cuda, tmp_path):
    g = golden("cli.npz")
    out = tmp_path / "gc.csv"
    assert cli.main(["gradcheck", "--problem", "burgers1d", "--elements", "4", "--degree", "6", "--steps",
                     "20", "--horizon", "0.2", "--ndirs", "2", "--eps", "1e-4,1e-5",
                     "--output", str(out)]) == 0
    mine, ref = out.read_text(), bytes(g["gradcheck"]).decode()
    assert abs(float(_meta(mine, "J0")) - float(_meta(ref, "J0"))) <= 1e-9 * abs(float(_meta(ref, "J0")))
    _, rm = _rows(mine)
    _, rr = _rows(ref)
    for a, b in zip(rm, rr):
        assert a[:2] == b[:2]
        assert abs(float(a[3]) - float(b[3])) <= 1e-9 * abs(float(b[3]))      # adjoint directional derivative
        assert abs(float(a[2]) - float(b[2])) <= 1e-6 * abs(float(b[2]))      # finite difference
    assert float(_meta(mine, "max_rel_error")) <= 1e-6


def test_optimize_and_bench_commands(cuda, tmp_path):
    assert cli.main(["optimize", "--problem", "burgers1d", "--elements", "4", "--degree", "6", "--steps",
                     "10", "--horizon", "0.1", "--max-iters", "2", "--output", str(tmp_path / "o")]) in (0, 4)
    assert (tmp_path / "o.field").exists() and "# status = " in (tmp_path / "o.csv").read_text()
    assert cli.main(["bench", "--problem", "burgers1d", "--elements", "8", "--steps", "5", "--horizon",
                     "0.05", "--degrees", "7,8", "--reps", "3", "--output", str(tmp_path / "b.csv")]) == 0
    head, rows = _rows((tmp_path / "b.csv").read_text())
    assert head == "operation,degree,unknowns,seconds" and len(rows) == 10
