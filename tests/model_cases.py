"""BASELINE configs C2-C4 as engine-parity cases.

Layer lists come from paper_2111_08617_b200/layouts/*.json (torchvision /
transformers parameter shapes, derived offline).  Each layer gets the
reference engine's kind and a gradient scale; node r, layer t, step k get
``scale_t * normal01(H(H(H(tag, k), r), t), i)`` (oracle.engine_inputs, the
recipe oracle/ref_shim.cpp:ref_engine_run uses).

* C2  ResNet-50, 161 tensors, default filter + plan (4 bits / bucket 128),
      64 MiB fused buffers (2 buffers), step_seed 1, N in {2,3,4,5,8}.
* C3  VGG-16, 32 tensors (fc6 split over 6 buffers, 10 buffers), plan
      defaults {2, 8} bits / bucket 512, N = 8.
* C4  BERT-base, 206 tensors, adaptive k-means over the palette
      {2,3,4,5,6,8}, alpha 1, a short stats period / window, N = 8; scales
      banded like the reference's canned transformer population
      (/root/reference/proj/src/bench.cpp:204-216): embeddings 1e-3,
      attention 1e-2, MLP 1.2e-2, pooler / prediction heads 0.3.
"""
from __future__ import annotations

import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LAYOUTS = os.path.join(ROOT, "paper_2111_08617_b200", "layouts")
KIND = {"weight": 0, "bias": 1, "norm": 2, "embedding": 3, "other": 4}


def _layers(model):
    with open(os.path.join(LAYOUTS, f"{model}.json")) as f:
        return json.load(f)["layers"]


def _bert_scale(name):
    if ".embeddings." in name:
        return 1e-3
    if ".attention." in name:
        return 1e-2
    if ".intermediate." in name or ".output." in name:
        return 1.2e-2
    return 0.3  # pooler and prediction heads: the small hot layers


def layers(model):
    """(name, elements, kind_int, scale) per tensor."""
    out = []
    for x in _layers(model):
        scale = _bert_scale(x["name"]) if model == "bert_base" else 1e-3
        out.append((x["name"], int(x["elements"]), KIND[x["kind"]], scale))
    return out


def plan_json(bits, bucket):
    return json.dumps({"defaults": {"bits": bits, "bucket": bucket}})


C4_ADAPTIVE = json.dumps({"method": "kmeans", "palette": [2, 3, 4, 5, 6, 8], "alpha": 1.0,
                          "stats_period": 2, "stats_window": 1})


def cases():
    """Engine-parity cases over the benchmark models (golden: models.json)."""
    out = []
    for n in (2, 3, 4, 5, 8):
        out.append(dict(name=f"C2_resnet50_n{n}", model="resnet50", nodes=n, steps=3, tag=0xC2))
    for bits in (2, 8):
        out.append(dict(name=f"C3_vgg16_{bits}b_n8", model="vgg16", nodes=8, steps=2, tag=0xC3,
                        plan=plan_json(bits, 512)))
    out.append(dict(name="C4_bert_base_adaptive_n8", model="bert_base", nodes=8, steps=4,
                    tag=0xC4, adaptive=C4_ADAPTIVE))
    return out
