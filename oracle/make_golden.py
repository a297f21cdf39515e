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
    print(f"wrote {len(codec)} codec and {len(sra)} sra cases to {OUT}")


if __name__ == "__main__":
    main()
