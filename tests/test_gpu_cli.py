"""The `poas` CLI on B200 units: profile -> plan -> run on
the tensor and CUDA-core units (resident and host operands), C written by
`run --out-c` checked against the fp64 oracle under the plan semantics, and
`evaluate` producing the reference's report schema with measured
standalone runs."""
import json
import subprocess

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
CLI = ROOT / "paper_2209_10245_b200" / "bin" / "poas"
UNITS = ("gpu0.tc=xpu:dev=0:sms=16:dtype=bf16:elem=2:link=hbm:probe=256-1024;"
         "gpu0.simt=gpu:dev=0:sms=4:exclusive=1:elem=4:link=hbm:probe=128-512")
PROF = "probes=4,repetitions=2,bandwidth_payload=8388608"


def run(*args):
    return subprocess.run([str(CLI), *args], capture_output=True, text=True, timeout=600)


@pytest.fixture(scope="module")
def gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")


def _planted(text, slope):
    out = []
    for line in text.splitlines():
        p = line.split()
        if len(p) == 2 and p[0] == "slope":
            line = f"slope {slope!r}"
        elif len(p) == 2 and p[0] == "intercept":
            line = "intercept 0"
        out.append(line)
    return "\n".join(out) + "\n"


@pytest.mark.parametrize("host", [False, True])
def test_run_gpu_units_c_matches_oracle(gpu, tmp_path, host):
    import oracle

    units = UNITS if not host else UNITS.replace("link=hbm", "link=pcie")
    prof = tmp_path / "p.profile"
    r = run("profile", "--units", units, "--profiling", PROF, "--out", str(prof))
    assert r.returncode == 0, r.stderr
    # a machine on which both units get rows: both kernels write C
    prof.write_text(_planted(prof.read_text(), 2e-13))
    m, n, k = 1000, 768, 520
    sched = tmp_path / "s.json"
    r = run("plan", "--profile", str(prof), "--dims", f"{m}x{n}x{k}", "--out", str(sched))
    assert r.returncode == 0, r.stderr
    sd = json.loads(sched.read_text())
    assert all(d["rows"] > 0 for d in sd["devices"]), sd["devices"]
    c_path = tmp_path / "C.bin"
    args = ["run", "--schedule", str(sched), "--units", units, "--repeats", "2", "--seed", "7",
            "--out-c", str(c_path)] + (["--host"] if host else [])
    r = run(*args)
    assert r.returncode == 0, r.stderr
    C = np.fromfile(c_path, dtype=np.float32).reshape(m, n)
    sa, sb = oracle.stream_seed(7, "A"), oracle.stream_seed(7, "B")
    exp = oracle.expected_c(sd, oracle.fill_uniform(m, k, sa), oracle.fill_uniform(k, n, sb),
                            {"gpu0.tc": 2, "gpu0.simt": 0})
    assert oracle.rel_frobenius(C, exp) <= 2e-5
    rep = json.loads((tmp_path / "s.report.json").read_text())
    assert rep["repeats"] == 2 and rep["measured_makespan"] > 0


def test_evaluate_gpu_units(gpu, tmp_path):
    inputs = tmp_path / "in.json"
    inputs.write_text(json.dumps([{"name": "a", "m": 2048, "n": 1024, "k": 1024},
                                  {"name": "b", "m": 1000, "n": 2000, "k": 512}]))
    out = tmp_path / "ev"
    r = run("evaluate", "--units", UNITS, "--inputs", str(inputs), "--profiling", PROF, "--repeats", "3",
            "--out-dir", str(out))
    assert r.returncode == 0, r.stderr
    rep = json.loads((out / "report.json").read_text())
    assert rep["devices"] == ["gpu0.tc", "gpu0.simt"]
    for e in rep["inputs"]:
        assert e["measured_makespan"] > 0 and e["predicted_makespan"] > 0
        assert sum(d["rows"] for d in e["devices"]) == e["dims"]["m"]
        for d in e["devices"]:
            assert d["standalone_makespan"] > 0 and d["speedup"] > 0
        assert e["b200"]["standalone_measured"]  # small shapes: measured, not predicted
    assert {x["id"] for x in rep["rmse"]} == {"gpu0.tc", "gpu0.simt"}
