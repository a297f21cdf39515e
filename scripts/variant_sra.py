"""Emulated N = 8 SRA per-rank kernel time (scripts/sra_emul_bench.py's
measurement) for libgcx.so and each compile-time variant in
paper_2111_08617_b200/variants/ (swapped in by copying; development tool)."""
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = os.path.join(ROOT, "paper_2111_08617_b200", "libgcx.so")
shutil.copy(lib, "/tmp/libgcx_orig.so")
vdir = os.path.join(ROOT, "paper_2111_08617_b200", "variants")
names = ["orig"] + sorted(f[:-3] for f in os.listdir(vdir) if f.endswith(".so"))
for name in names:
    src = "/tmp/libgcx_orig.so" if name == "orig" else os.path.join(vdir, name + ".so")
    shutil.copy(src, lib)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "sra_emul_bench.py")],
                         capture_output=True, text=True, cwd=ROOT).stdout
    print(name, out.strip().splitlines()[-3:], flush=True)
shutil.copy("/tmp/libgcx_orig.so", lib)
