"""Generate tests/golden/models.json: per-step digests of the COMPILED
REFERENCE Engine (src/engine.cpp over SimNet, oracle/_ref) on the benchmark
models C2-C4 (tests/model_cases.py).

Run here (where /root/reference exists):  python -m oracle.make_golden_models [name...]
Test infrastructure only.  Each case stores FNV-1a digests (util.hpp:73-80)
of node 0's flushed outputs per step (the reference checks every node equal)
and the plan swaps the adaptive engine logged.
"""
from __future__ import annotations

import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import RefOracle  # noqa: E402
from tests.model_cases import cases, layers  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests",
                   "golden", "models.json")


def main(names):
    ref = RefOracle()
    old = {}
    if os.path.exists(OUT):
        with open(OUT) as f:
            old = {c["name"]: c for c in json.load(f)["cases"]}
    done = []
    for c in cases():
        if names and c["name"] not in names:
            if c["name"] in old:
                done.append(old[c["name"]])
            continue
        t = time.time()
        dig, ev = ref.engine_run(c["nodes"], layers(c["model"]), c["steps"], c["tag"],
                                 c.get("plan"), c.get("adaptive"), c.get("step_seed", 1), 0)
        swaps = [json.loads(x) for x in ev.splitlines()]
        c = dict(c, digests=dig,
                 plan_swaps=[[e["step"], e["payload"]["bits"]] for e in swaps
                             if e["event"] == "plan_swap"],
                 ref_seconds=round(time.time() - t, 1))
        print(c["name"], c["digests"], f"{c['ref_seconds']} s", flush=True)
        done.append(c)
        with open(OUT, "w") as f:
            json.dump(dict(source="compiled reference src/engine.cpp via SimNet (oracle/_ref); "
                                  "cases: tests/model_cases.py", cases=done), f, indent=0)


if __name__ == "__main__":
    main(sys.argv[1:])
