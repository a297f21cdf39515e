"""Generate tests/golden/*.json from the COMPILED REFERENCE (oracle/_ref).

Run here (where /root/reference exists):  python -m oracle.make_golden
The fixtures hold input recipes plus FNV-1a digests (util.hpp:73-80) of the
reference's outputs, so they stay small and travel to the GPU box, where the
reference tree does not exist.

Input recipes (``gen``) are rebuilt by ``tests/golden_inputs.py`` with the
keyed normal01 generator (util.hpp:32-38) plus deterministic edits that cover
the edge cases SURVEY §4 lists: zero buckets, -0.0, single-spike buckets,
ragged tails, tiny and empty vectors.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import MODE_QUANTIZE, MODE_UNCOMPRESSED, Oracle, RefOracle  # noqa: E402
from tests.golden_inputs import make_input  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests",
                   "golden")


def codec_cases():
    cases = []
    kinds = ["normal", "zeros_mixed", "negzero", "spike", "tiny_scale", "huge_scale",
             "integers"]
    lengths = [0, 1, 7, 33, 128, 1000, 4099, 65537]
    buckets = [1, 8, 64, 128, 512, 1024, 7, 1000]
    k = 0
    for bits in range(1, 9):
        for bucket in buckets:
            for n in lengths:
                if bucket == 1 and n > 4099:
                    continue
                kind = kinds[k % len(kinds)]
                k += 1
                cases.append(dict(n=n, bits=bits, bucket=bucket, seed=1000003 * k + 17,
                                  gen=dict(kind=kind, seed=k)))
    # the C1-style configuration at a moderate size
    cases.append(dict(n=1 << 20, bits=4, bucket=128, seed=42,
                      gen=dict(kind="normal", seed=0x5eed, scale=1e-3)))
    return cases


def sra_cases():
    cases = []
    k = 0
    for nodes in [2, 3, 4, 5, 8]:
        for layout in ["single", "mixed", "raw"]:
            k += 1
            d = 10007 + 131 * nodes
            if layout == "single":
                segs = [[0, d, MODE_QUANTIZE, 4, 128]]
            elif layout == "raw":
                segs = [[0, d, MODE_UNCOMPRESSED, 0, 0]]
            else:
                segs = [[0, 300, MODE_UNCOMPRESSED, 0, 0], [300, 5000, MODE_QUANTIZE, 4, 128],
                        [5300, 2000, MODE_QUANTIZE, 2, 512], [7300, 64, MODE_UNCOMPRESSED, 0, 0],
                        [7364, d - 7364, MODE_QUANTIZE, 8, 64]]
            for average in [True, False]:
                cases.append(dict(nodes=nodes, d=d, segments=segs, step_seed=1000 + k,
                                  average=average, gen=dict(kind="normal", seed=77 * k)))
    return cases


RESNETISH = [("conv1.w", 9408, 0, 1e-3), ("bn1.w", 64, 2, 1e-2), ("bn1.b", 64, 1, 1e-2),
             ("layer1.conv.w", 36864, 0, 1e-3), ("layer1.bn.w", 64, 2, 1e-2),
             ("layer2.conv.w", 73728, 0, 2e-3), ("small.w", 1000, 0, 1e-2),
             ("fc.w", 20480, 0, 1e-2), ("fc.b", 10, 1, 1e-2)]


def engine_cases():
    plan = json.dumps({"defaults": {"bits": 4, "bucket": 128},
                       "layers": {"fc.w": {"bits": 8, "bucket": 64},
                                  "layer2.conv.w": {"bits": 2, "bucket": 512},
                                  "conv1.w": {"mode": "uncompressed"}}})
    adaptive = json.dumps({"method": "kmeans", "palette": [2, 4, 8], "stats_period": 3,
                           "stats_window": 2})
    linear = json.dumps({"method": "linear", "palette": [2, 3, 4, 5, 6, 8], "stats_period": 2,
                         "stats_window": 1, "pair_buckets": True})
    return [
        dict(name="static_default_n2", nodes=2, layers=RESNETISH, steps=3, tag=0xC2),
        dict(name="static_default_n5", nodes=5, layers=RESNETISH, steps=2, tag=0xC3),
        dict(name="static_plan_n4_small_fuse", nodes=4, layers=RESNETISH, steps=3, tag=0xC4,
             plan=plan, fuse_limit=200000, step_seed=99),
        dict(name="adaptive_kmeans_n3", nodes=3, layers=RESNETISH, steps=5, tag=0xC5,
             adaptive=adaptive),
        dict(name="adaptive_linear_pairs_n2", nodes=2, layers=RESNETISH, steps=4, tag=0xC6,
             adaptive=linear),
    ]


def main():
    ref = RefOracle()
    o = Oracle()
    os.makedirs(OUT, exist_ok=True)
    codec = []
    for c in codec_cases():
        v = make_input(c["n"], c["gen"])
        norms, packed = ref.quantize(v, c["bits"], c["bucket"], c["seed"])
        deq = ref.dequantize(norms, packed, c["n"], c["bits"], c["bucket"])
        wire = ref.serialize(v, c["bits"], c["bucket"], c["seed"])
        c.update(norms_fnv=o.fnv1a64(norms), packed_fnv=o.fnv1a64(packed),
                 deq_fnv=o.fnv1a64(deq), wire_fnv=o.fnv1a64(wire), packed_len=int(packed.size),
                 input_fnv=o.fnv1a64(v))
        if c["n"] <= 64:
            c["packed_hex"] = packed.tobytes().hex()
            c["norms_hex"] = norms.tobytes().hex()
        codec.append(c)
    with open(os.path.join(OUT, "codec.json"), "w") as f:
        json.dump(dict(source="compiled reference src/codec.cpp via oracle/_ref",
                       cases=codec), f, indent=0)

    sra = []
    for c in sra_cases():
        inputs = [make_input(c["d"], dict(c["gen"], seed=c["gen"]["seed"] + r))
                  for r in range(c["nodes"])]
        outs, sent, ctr = ref.allreduce(inputs, [tuple(s) for s in c["segments"]],
                                        c["step_seed"], c["average"])
        assert all((x.view(np.uint32) == outs[0].view(np.uint32)).all() for x in outs)
        c.update(out_fnv=o.fnv1a64(outs[0]), bytes_sent=sent, counters=ctr)
        sra.append(c)
    with open(os.path.join(OUT, "sra.json"), "w") as f:
        json.dump(dict(source="compiled reference src/collectives.cpp run_sra via SimNet",
                       cases=sra), f, indent=0)
    eng = []
    for c in engine_cases():
        dig, ev = ref.engine_run(c["nodes"], c["layers"], c["steps"], c["tag"], c.get("plan"),
                                 c.get("adaptive"), c.get("step_seed", 1), c.get("fuse_limit", 0))
        swaps = [json.loads(x) for x in ev.splitlines()]
        c.update(digests=dig, plan_swaps=[[e["step"], e["payload"]["bits"]] for e in swaps
                                          if e["event"] == "plan_swap"])
        eng.append(c)
    with open(os.path.join(OUT, "engine.json"), "w") as f:
        json.dump(dict(source="compiled reference src/engine.cpp via SimNet (oracle/_ref)",
                       cases=eng), f, indent=0)
    print(f"wrote {len(codec)} codec, {len(sra)} sra, {len(eng)} engine cases to {OUT}")


if __name__ == "__main__":
    main()
