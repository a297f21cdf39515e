"""Run bench.py with each compile-time variant of libgcx.so in
paper_2111_08617_b200/variants/ swapped in (development tool, GPU box):
prints value, pipelined / serial step time and K1 time per variant."""
import os, sys, json, subprocess, shutil
ROOT = "/root/repo"
lib = os.path.join(ROOT, "paper_2111_08617_b200", "libgcx.so")
shutil.copy(lib, "/tmp/libgcx_orig.so")
res = {}
names = ["orig"] + sorted(f[:-3] for f in os.listdir(os.path.join(ROOT, "paper_2111_08617_b200", "variants")) if f.endswith(".so"))
for name in names:
    src = "/tmp/libgcx_orig.so" if name == "orig" else os.path.join(ROOT, "paper_2111_08617_b200", "variants", name + ".so")
    shutil.copy(src, lib)
    out = subprocess.run([sys.executable, "bench.py", "--steps", "20", "--warmup", "5"], capture_output=True, text=True, cwd=ROOT).stdout
    d = json.loads(out.strip().splitlines()[-1])
    res[name] = (d["value"], d["ms_per_step"], d["config"]["ms_per_step_serial"], d["config"]["quantize_ms"], d["config"]["dequantize_ms"])
    print(name, res[name], flush=True)
shutil.copy("/tmp/libgcx_orig.so", lib)
