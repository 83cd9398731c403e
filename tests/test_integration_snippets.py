"""INTEGRATION.md's reference-side bindings compile and run.

Every ``<!-- snippet: NAME -->`` code block of INTEGRATION.md is extracted
verbatim. The C++ ones are compiled into tests/integration/harness.cpp
against the REFERENCE library itself (oracle/_ref/obj: /root/reference/proj/
src built unchanged with -Dpoas=poasref, so ``poas::`` in the snippets is the
reference) and linked with libpoas_b200.so; the harness profiles a host-CPU
unit through the snippet's B200Backend inside the reference's own
run_compute_probes / fit_machine, plans with the reference planner, executes
through poas_b200_execute, runs poas_b200_run_dynamic and the overlapped
path. The ctypes snippet is executed as written. CPU only (a host unit).
"""
import json
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT

REF_INC = Path("/root/reference/proj/include")
REF_OBJ = ROOT / "oracle" / "_ref" / "obj"
JSON_DIR = Path("/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann")


def snippets() -> dict:
    text = (ROOT / "INTEGRATION.md").read_text()
    out = {}
    for m in re.finditer(r"<!-- snippet: (\w+) -->\n```(\w+)\n(.*?)```", text, re.S):
        out[m.group(1)] = (m.group(2), m.group(3))
    return out


def test_snippets_present():
    s = snippets()
    assert set(s) >= {"backend", "execute", "ctypes", "dynamic", "overlap", "sharded"}, sorted(s)


def test_cpp_snippets_compile_and_run_against_reference(tmp_path):
    if not REF_INC.is_dir() or not (REF_OBJ / "profiler.o").exists():
        pytest.skip("reference sources / oracle/_ref objects not available (make -C oracle ref)")
    for name, (lang, body) in snippets().items():
        if lang == "cpp":
            (tmp_path / f"snippet_{name}.inc").write_text(body)
    objs = [str(p) for p in sorted(REF_OBJ.glob("*.o")) if p.name != "ref_shim.o"]
    exe = tmp_path / "harness"
    cmd = ["g++", "-std=c++20", "-O1", "-Dpoas=poasref", f"-I{tmp_path}", f"-I{REF_INC}", f"-I{JSON_DIR}",
           f"-I{ROOT / 'include'}", str(ROOT / "tests" / "integration" / "harness.cpp"), *objs,
           "-fopenmp", f"-L{ROOT / 'paper_2209_10245_b200'}", "-lpoas_b200",
           f"-Wl,-rpath,{ROOT / 'paper_2209_10245_b200'}", "-o", str(exe)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-4000:]
    m, n, k = 160, 96, 72
    r = subprocess.run([str(exe), str(tmp_path), str(m), str(n), str(k)], capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0 and r.stdout.strip() == "ok", (r.returncode, r.stdout, r.stderr[-3000:])

    import oracle

    prof = (tmp_path / "profile.txt").read_text()
    assert "device cpu0" in prof and "kind cpu" in prof
    # the reference planner's schedule for the B200-backend profile
    assert (tmp_path / "schedule.json").read_text() == oracle.ref.plan(prof, m, n, k)
    A = np.fromfile(tmp_path / "A.bin", dtype=np.float32).reshape(m, k)
    B = np.fromfile(tmp_path / "B.bin", dtype=np.float32).reshape(k, n)
    exp = A.astype(np.float64) @ B.astype(np.float64)
    for cname in ("C.bin", "C_ovl.bin"):
        C = np.fromfile(tmp_path / cname, dtype=np.float32).reshape(m, n)
        assert np.linalg.norm(C - exp) / np.linalg.norm(exp) <= 2e-5, cname
    rep = json.loads((tmp_path / "report.json").read_text())
    assert rep["repeats"] == 2 and rep["measured_makespan"] > 0
    dyn = json.loads((tmp_path / "dynamic.json").read_text())
    assert len(dyn["iterations"]) == 2 and "profile" in dyn
    sh = json.loads((tmp_path / "sharded.json").read_text())
    assert sh["rows"] == [m] and sh["row0"] == [0]
    assert sum(d["rows"] for d in sh["plans"][0]["devices"]) == m


def test_ctypes_snippet_runs(poas):
    lang, body = snippets()["ctypes"]
    assert lang == "python"
    prof = (ROOT / "tests" / "golden" / "profiles").glob("*.profile")
    profile_text = next(iter(sorted(prof))).read_text()
    import os

    cwd = os.getcwd()
    os.chdir(ROOT)
    try:
        env = {"profile_text": profile_text}
        exec(compile(body, "INTEGRATION.md:ctypes", "exec"), env)
    finally:
        os.chdir(cwd)
    assert env["rc"] == 0
    assert env["schedule"] == poas.plan(profile_text, 16384, 16384, 16384)
