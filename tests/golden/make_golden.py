"""Regenerates tests/golden/cases.json from the UNMODIFIED reference simulator
(oracle/_ref/libservesim_ref.so, compiled from /root/reference/proj/src by
oracle/Makefile). Run here (where /root/reference exists):

    python tests/golden/make_golden.py

Each entry pins, for one parity case of tests/cases.py: the reference's
event_hash, arrival_hash, decisions and byte-exact summary_json.
"""
import json
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from cases import static_cases, trace_cases  # noqa: E402
from oracle_lib import Ref  # noqa: E402
from paper_2509_23384_b200 import sim  # noqa: E402


def main():
    ref = Ref()
    out = {}
    with tempfile.TemporaryDirectory() as td:
        allc = dict(static_cases())
        allc.update(trace_cases(td, sim.synth_generate))
        for name, cfg in allc.items():
            r = ref.run(cfg)
            out[name] = {k: r[k] for k in ("event_hash", "arrival_hash", "decisions", "arrived",
                                           "completed", "rejected", "unfinished", "summary_json")}
    # known answers of the perf model (proj/tests/test_perf_model.cpp:43-51, 91-117)
    dst = Path(__file__).with_name("cases.json")
    dst.write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")
    print(f"wrote {len(out)} cases to {dst}")


if __name__ == "__main__":
    main()
