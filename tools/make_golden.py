"""Regenerates tests/golden/ from the REFERENCE planner (oracle/_ref, built
from /root/reference by oracle/Makefile). Run here, where /root/reference
exists; the fixtures are committed so parity tests also run without it.

    python tools/make_golden.py
"""
import hashlib
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import oracle  # noqa: E402

REF = Path("/root/reference/proj")
OUT = ROOT / "tests" / "golden"

# Planning cases: (profile name, m, n, k). Table 3 inputs (reference
# proj/data/table3.json), the BASELINE configs, and the survey's examples.
DIMS = [
    (30000, 30000, 30000), (60000, 20000, 35000), (130000, 20000, 20000),
    (40000, 80000, 20000), (40000, 30000, 60000), (56000, 40000, 40000),
    (16000, 16000, 16000), (2048, 2048, 2048), (8192, 8192, 8192), (16384, 16384, 16384),
    (65536, 8192, 8192), (1024, 1024, 1024), (32768, 32768, 32768), (16003, 4000, 4000),
    (20011, 3000, 3000),
]

CPU_ONLY = ("poas-machine v1\n\nbus true\n\ndevice cpu0\nkind cpu\ntrue_slope 2e-12\n"
            "true_intercept 0.0005\nelem_size 4\nnoise 0\ndrift 0\ncache_bytes 314572800\n")

# The survey's illustrative B200-like machine.
B200_LIKE = ("poas-machine v1\n\nbus true\n\nprofiling\naccel_min_side 3000\naccel_max_side 6000\n\n"
             "device cpu0\nkind cpu\ntrue_slope 2e-12\ntrue_intercept 0.0005\nelem_size 4\nnoise 0\n"
             "drift 0\n\ndevice gpu0.simt\nkind gpu\ntrue_slope 3.5e-14\ntrue_intercept 2e-05\n"
             "true_bandwidth 6500000000000\nelem_size 4\nnoise 0\ndrift 0\n\n"
             "device gpu0.tc\nkind xpu\ntrue_slope 1.45e-15\ntrue_intercept 2e-05\n"
             "true_bandwidth 6500000000000\nelem_size 2\nnoise 0\ndrift 0\nalign 8\n")


def main():
    oracle.build(with_ref=True)
    r = oracle.ref
    OUT.mkdir(parents=True, exist_ok=True)
    mach2 = r.machine_config_roundtrip((REF / "data" / "mach2.cfg").read_text())
    (OUT / "mach2.cfg").write_text(mach2)
    (OUT / "table3.json").write_text((REF / "data" / "table3.json").read_text())

    profiles = {
        "mach2_exact": r.exact_profile(mach2),
        "mach2_seed7": r.profile_synthetic(mach2, 7),
        "mach2_seed1": r.profile_synthetic(mach2, 1),
        "cpu_only": r.exact_profile(CPU_ONLY),
        "b200_like": r.exact_profile(B200_LIKE),
    }
    (OUT / "profiles").mkdir(exist_ok=True)
    for name, text in profiles.items():
        (OUT / "profiles" / f"{name}.profile").write_text(text)

    cases = []
    for name, text in profiles.items():
        for (m, n, k) in DIMS:
            try:
                sched = r.plan(text, m, n, k)
                split = r.solve_split(text, m, n, k)
                err = None
            except oracle.OracleError as e:
                sched, split, err = None, None, e.code
            digest = hashlib.sha256(sched.encode()).hexdigest() if sched else None
            cases.append({"profile": name, "m": m, "n": n, "k": k,
                          "schedule": sched if sched and len(sched) < 12000 else None,
                          "schedule_sha256": digest, "split": split, "error": err})
    (OUT / "plans.json").write_text(json.dumps(cases, indent=0))

    rng = {"for_stream_20261017_A": r.rng_draw(20261017, "A", 0),
           "for_stream_20261017_B": r.rng_draw(20261017, "B", 0),
           "for_stream_20261017_A_draw9": r.rng_draw(20261017, "A", 9)}
    (OUT / "rng.json").write_text(json.dumps(rng, indent=1))
    print(f"wrote {len(cases)} plan cases, {len(profiles)} profiles to {OUT}")


if __name__ == "__main__":
    main()
