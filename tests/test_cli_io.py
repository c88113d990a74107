"""SGT1 I/O parity with files written by the reference (tests/golden/*.sgt) and
the GPU-backed CLI (reference tests/test_cli.py:70-106 restated)."""

import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import GOLDEN, ROOT, golden, rel_err
from paper_2509_10613_b200.errors import FormatError
from paper_2509_10613_b200.sgt_io import read_array, write_array


@pytest.mark.parametrize("name,key", [("ref_f64_3d", "a3"), ("ref_f32_2d", "a2"),
                                      ("ref_int_1d", "a1")])
def test_reads_reference_files_and_writes_identical_bytes(tmp_path, name, key):
    g = golden("sgt_contents")
    path = os.path.join(GOLDEN, name + ".sgt")
    got = read_array(path)
    want = g[key]
    assert got.shape == want.shape
    np.testing.assert_array_equal(got, want.astype(got.dtype))
    out = tmp_path / "o.sgt"
    write_array(want, out)
    assert open(out, "rb").read() == open(path, "rb").read()


def test_malformed_files(tmp_path):
    p = tmp_path / "bad.sgt"
    p.write_bytes(b"SGT")
    with pytest.raises(FormatError) as e:
        read_array(p)
    assert e.value.offset == 3
    p.write_bytes(b"XXXX\x00\x01" + (1).to_bytes(8, "little") + b"\x00" * 8)
    with pytest.raises(FormatError) as e:
        read_array(p)
    assert e.value.offset == 0
    p.write_bytes(b"SGT1\x07\x01" + (1).to_bytes(8, "little") + b"\x00" * 8)
    with pytest.raises(FormatError) as e:
        read_array(p)
    assert e.value.offset == 4
    p.write_bytes(b"SGT1\x00\x01" + (2).to_bytes(8, "little") + b"\x00" * 8)
    with pytest.raises(FormatError) as e:
        read_array(p)
    assert e.value.offset == 14
    c = tmp_path / "p.csv"
    c.write_text("0,1\n1,2\n")
    np.testing.assert_array_equal(read_array(c), [[0, 1], [1, 2]])


def run_cli(*args):
    return subprocess.run([sys.executable, "-m", "paper_2509_10613_b200.cli", *args],
                          capture_output=True, text=True, cwd=ROOT)


def test_cli_usage_error_without_gpu(tmp_path):
    x = tmp_path / "x.sgt"
    write_array(np.zeros((3, 1)), x)
    r = run_cli("kernel", "--input", str(x), "--input2", str(x), "--cotangent", str(x))
    assert r.returncode == 2  # usage error before any device work


@pytest.mark.gpu
class TestCliGpu:
    def test_constant_paths_print_one(self, tmp_path):
        c = tmp_path / "c.sgt"
        write_array(np.zeros((3, 1)), c)
        r = run_cli("kernel", "--input", str(c), "--input2", str(c))
        assert r.returncode == 0, r.stderr
        assert r.stdout.strip() == "1.0"

    def test_backward_outputs_match_facade(self, tmp_path):
        from paper_2509_10613_b200 import sigcore_compat as sc
        x, y, cot = tmp_path / "x.sgt", tmp_path / "y.sgt", tmp_path / "c.sgt"
        gx, gy = tmp_path / "gx.sgt", tmp_path / "gy.sgt"
        rng = np.random.default_rng(0)
        xa = rng.standard_normal((1, 4, 2)) * 0.5
        ya = rng.standard_normal((1, 5, 2)) * 0.5
        write_array(xa, x)
        write_array(ya, y)
        write_array(np.array([2.0]), cot)
        r = run_cli("kernel", "--input", str(x), "--input2", str(y), "--dyadic-x", "1",
                    "--cotangent", str(cot), "--grad-output-x", str(gx),
                    "--grad-output-y", str(gy))
        assert r.returncode == 0, r.stderr
        _, wx, wy = sc.kernel_batch_backward(xa, ya, sc.KernelConfig(1, 0), np.array([2.0]))
        np.testing.assert_array_equal(read_array(gx), wx)
        np.testing.assert_array_equal(read_array(gy), wy)

    def test_gram_symmetric_and_matches_oracle(self, tmp_path, oracle):
        inp, out = tmp_path / "x.sgt", tmp_path / "g.sgt"
        X = np.random.default_rng(1).standard_normal((3, 4, 2))
        write_array(X, inp)
        r = run_cli("gram", "--input", str(inp), "--output", str(out))
        assert r.returncode == 0, r.stderr
        g = read_array(out)
        assert g.shape == (3, 3)
        np.testing.assert_array_equal(g, g.T)
        assert rel_err(g, oracle.kernel_gram(X)) < 1e-10

    def test_rbf_flag(self, tmp_path, oracle):
        x, y, out = tmp_path / "x.sgt", tmp_path / "y.sgt", tmp_path / "k.sgt"
        rng = np.random.default_rng(2)
        xa, ya = rng.standard_normal((2, 6, 3)), rng.standard_normal((2, 5, 3))
        write_array(xa, x)
        write_array(ya, y)
        r = run_cli("kernel", "--input", str(x), "--input2", str(y), "--dyadic-x", "1",
                    "--rbf-sigma", "0.9", "--output", str(out))
        assert r.returncode == 0, r.stderr
        assert rel_err(read_array(out), oracle.kernel_batch(xa, ya, 1, 0, ("rbf", 0.9))) < 1e-10

    def test_bad_file_is_data_error(self, tmp_path):
        p = tmp_path / "bad.sgt"
        p.write_bytes(b"nope")
        r = run_cli("gram", "--input", str(p), "--output", str(tmp_path / "g.sgt"))
        assert r.returncode == 1


def test_bench_report_schema_cpu():
    """The GPU bench report keeps the reference's fields and validates against
    schemas/bench_report_gpu.schema.json (no GPU needed for the report object)."""
    import json
    import os

    import jsonschema

    from paper_2509_10613_b200.bench_tasks import TASKS, BenchReport
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    schema = json.load(open(os.path.join(root, "schemas", "bench_report_gpu.schema.json")))
    for task in TASKS:
        r = BenchReport(task=task, shape={"B": 4, "L": 16, "d": 3, "dyadic_x": 0, "dyadic_y": 1},
                        repetitions=3, times=[0.3, 0.2, 0.25], cells=4 * 15 * 30)
        d = json.loads(r.to_json())
        jsonschema.validate(d, schema)
        assert d["minimum"] == 0.2 and abs(d["cells_per_s"] - 1800 / 0.2) < 1e-6
        for k in ("task", "shape", "repetitions", "times", "minimum", "threads", "scalar_width"):
            assert k in d  # the reference report's fields (sigcore/bench.py:38-47)


def test_bench_parser_accepts_reference_flags():
    from paper_2509_10613_b200 import cli
    a = cli.build_parser().parse_args(["bench", "--task", "kernel-fwd", "--batch", "8",
                                       "--length", "64", "--dim", "4", "--dyadic-x", "1",
                                       "--reps", "5", "--json"])
    assert a.task == "kernel-fwd" and a.reps == 5 and a.json


@pytest.mark.gpu
@pytest.mark.parametrize("task", ["kernel-fwd", "kernel-bwd", "gram-fwd", "gram-bwd",
                                  "gram-value-grad"])
def test_bench_tasks_gpu(task, tmp_path):
    """Every bench task runs on the GPU through the CLI and emits a report that
    validates against the extended schema."""
    import json

    import jsonschema
    out = tmp_path / "r.json"
    r = subprocess.run([sys.executable, "-m", "paper_2509_10613_b200.cli", "bench", "--task", task,
                        "--batch", "9", "--length", "40", "--dim", "6", "--reps", "3",
                        "--roofline", "--output", str(out)],
                       cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    d = json.loads(out.read_text())
    schema = json.load(open(os.path.join(ROOT, "schemas", "bench_report_gpu.schema.json")))
    jsonschema.validate(d, schema)
    assert d["task"] == task and d["cells_per_s"] > 0 and d["roofline_frac"] > 0
