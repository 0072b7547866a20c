"""Benchmark front end (paper_1704_03092_b200/cli.py): argument handling and
spec synthesis on the CPU (no GPU needed), one device run under -m gpu."""

import subprocess
import sys

import pytest

import paper_1704_03092_b200 as stc
from paper_1704_03092_b200 import cli


def test_synthesize_spec_matrix_and_split():
    s = cli.synthesize_spec(6, 7, 8)
    assert (s.labels_c, s.labels_a, s.labels_b) == ("ab", "ac", "cb")
    assert (s.n_i, s.n_j, s.n_p) == (6, 7, 8)
    s = cli.synthesize_spec(12, 7, 16, "split")
    assert (s.n_i, s.n_j, s.n_p) == (12, 7, 16)
    assert s.extents["a"] * s.extents["b"] == 12 and s.extents["a"] == 4  # ceil(sqrt(12)) = 4 divides 12
    assert (s.extents["c"], s.extents["d"]) == (7, 1)  # ceil(sqrt(7)) = 3 does not divide 7
    assert (s.extents["e"], s.extents["f"]) == (4, 4)
    with pytest.raises(ValueError):
        cli.synthesize_spec(2, 2, 2, "cube")


def test_operands_follow_the_seed_convention():
    spec = cli.synthesize_spec(3, 4, 5)
    a, b, c = cli.make_operands(spec, 7)
    ref = stc.make_dense_tensor(spec.tensor_extents(spec.labels_b), "random", 8)
    assert (b.data == ref.data).all() and a.extents == (3, 5) and c.extents == (3, 4)


@pytest.mark.parametrize("argv, msg", [
    (["-m", "4", "-n", "4"], "together"),
    (["-m", "4", "-n", "4", "-k", "4", "-file", "x"], "not both"),
    (["-m", "0", "-n", "4", "-k", "4"], ">= 1"),
    (["-m", "4", "-n", "4", "-k", "4", "-niter", "0"], "-niter"),
    (["-m", "4", "-n", "4", "-k", "4", "-impl", "0", "-level", "1"], "level 0"),
    (["-m", "4", "-n", "4", "-k", "4", "-blocking", "1,2,3"], "six"),
])
def test_argument_errors(argv, msg, capsys):
    assert cli.main(argv) == 2
    assert msg in capsys.readouterr().err


def test_bad_benchmark_file(tmp_path, capsys):
    f = tmp_path / "bench.txt"
    f.write_text("abij abef efij & a:2;b:2;i:2;j:2;e:2;\n")  # f has no extent
    assert cli.main(["-file", str(f)]) == 1
    assert "error" in capsys.readouterr().err


@pytest.mark.gpu
def test_cli_runs_and_reports_accuracy(tmp_path):
    f = tmp_path / "bench.txt"
    f.write_text("aibj eafb jfie & a:8;b:32;i:8;j:32;e:16;f:16;\nabij abef efij & a:6;b:7;i:5;j:9;e:4;f:3;\n")
    out = subprocess.run([sys.executable, "-m", "paper_1704_03092_b200", "-file", str(f), "-level", "2",
                          "-impl", "1", "-niter", "2", "-csv", str(tmp_path / "r.csv")],
                         capture_output=True, text=True, check=True).stdout.splitlines()
    assert out[0].startswith("# size")
    recs = [line.split("\t") for line in out[1:]]
    assert len(recs) == 2 and recs[0][0].startswith("aibj-eafb-jfie=")
    for r in recs:
        assert float(r[1]) > 0 and float(r[3]) > 0 and float(r[4]) <= 1e-12
    assert (tmp_path / "r.csv").read_text().startswith("size,seconds")
