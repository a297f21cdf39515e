"""Per-rank SRA kernel time of one step for the BASELINE configs C2-C4, every
rank's kernels on this B200 (exchange in device memory; see
scripts/sra_emul_bench.py): C2 ResNet-50 4b/128, C3 VGG-16 2b and 8b /
bucket 512, C4 BERT-base at the static 4b/128 plan and at a mixed-width plan
over the adaptive palette {2,3,4,5,6,8} (bucket 128; the widths the adaptive
planner picks vary by layer and window, so the emulation cycles the palette
over the compressed layers).  Writes gpurun_out/sra_emul_configs.json.
Development / evidence tool (GPU box)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2111_08617_b200 import _gcomm as G  # noqa: E402
from paper_2111_08617_b200.ddp import load_layout, resolve_codecs  # noqa: E402


def per_rank_ms(layers, codecs, nodes, rng):
    bufs = G.pack_fused_buffers([n for _, n, _ in layers], 64 << 20)
    total = 0.0
    for fb in bufs:
        req = G.ReduceRequest()
        req.inputs = [(rng.standard_normal(fb.total_elements) * 1e-3).astype(np.float32)
                      for _ in range(nodes)]
        req.segments = [G.Segment(s.buffer_offset, s.length, codecs[s.tensor_index].mode,
                                  codecs[s.tensor_index].bits, codecs[s.tensor_index].bucket_size)
                        for s in fb.segments]
        req.op = G.ReduceOp.average
        req.step_seed = 7
        G.allreduce(req, nodes)
        total += min(G.allreduce(req, nodes).trace.device_time_s for _ in range(3))
    return total * 1e3 / nodes, len(bufs)


def plan(bits, bucket):
    return G.CompressionPlan.from_json(json.dumps({"defaults": {"bits": bits, "bucket": bucket}}))


def main():
    rng = np.random.default_rng(0)
    out = []
    cfgs = [("C2 ResNet-50 4b/128", "resnet50", plan(4, 128), None),
            ("C3 VGG-16 2b/512", "vgg16", plan(2, 512), None),
            ("C3 VGG-16 8b/512", "vgg16", plan(8, 512), None),
            ("C4 BERT-base 4b/128 (static plan)", "bert_base", plan(4, 128), None),
            ("C4 BERT-base mixed {2,3,4,5,6,8}/128", "bert_base", plan(4, 128), [2, 3, 4, 5, 6, 8])]
    for name, model, pl, palette in cfgs:
        layers = load_layout(model)
        codecs = resolve_codecs(layers, pl)
        if palette:
            k = 0
            for c in codecs:
                if c.mode == G.CodecMode.quantize:
                    c.bits = palette[k % len(palette)]
                    k += 1
        elems = sum(n for _, n, _ in layers)
        for nodes in (2, 8):
            ms, nb = per_rank_ms(layers, codecs, nodes, rng)
            row = {"config": name, "nodes": nodes, "elements": elems, "buffers": nb,
                   "per_rank_kernel_ms": ms,
                   "kernel_busbw_GBps": 4 * elems / (ms * 1e-3) * 2 * (nodes - 1) / nodes / 1e9}
            out.append(row)
            print(row, flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", "sra_emul_configs.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
