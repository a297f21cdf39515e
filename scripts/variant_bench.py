"""Time K1 (gcx_quantize) of the compile-time variants in
paper_2111_08617_b200/variants/ on C1 and check they are bit-identical to
the shipped libgcx.so.  Development tool, run under gpurun."""
import ctypes as C
import glob
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def load(path):
    lib = C.CDLL(path)
    lib.gcx_quantize.argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.c_uint64, C.c_uint64,
                                 C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    lib.gcx_quantize.restype = C.c_int
    lib.gcx_quantize_prefixed.argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.c_uint64, C.c_uint64,
                                          C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                          C.c_void_p]
    lib.gcx_quantize_prefixed.restype = C.c_int
    lib.gcx_make_prefix.argtypes = [C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p]
    lib.gcx_prefix_slots.argtypes = [C.c_uint64]
    lib.gcx_prefix_slots.restype = C.c_uint64
    return lib


def main():
    n, bits, bucket = 25_557_032, 4, 128
    torch.cuda.set_device(0)
    g = torch.Generator(device="cuda").manual_seed(1)
    xs = [torch.randn(n, generator=g, device="cuda") * 1e-3 for _ in range(4)]
    nb = (n + bucket - 1) // bucket
    cap = 4 * ((n * (bits + 1) + 31) // 32)
    norms = torch.empty(nb, device="cuda")
    packed = torch.empty(cap, dtype=torch.uint8, device="cuda")
    bad = torch.empty(1, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream()
    libs = [os.path.join(ROOT, "paper_2111_08617_b200", "libgcx.so")] + sorted(
        glob.glob(os.path.join(ROOT, "paper_2111_08617_b200", "variants", "*.so")))
    ref_packed = None
    out = {}
    for path in libs:
        lib = load(path)
        prefix = torch.empty(lib.gcx_prefix_slots(n), dtype=torch.int64, device="cuda")
        assert lib.gcx_make_prefix(n, bucket, prefix.data_ptr(), st.cuda_stream) == 0
        use_prefix = os.environ.get("VARIANT_PREFIX", "1") == "1"

        def q(x, seed):
            if use_prefix:
                rc = lib.gcx_quantize_prefixed(x.data_ptr(), n, bits, bucket, seed,
                                               prefix.data_ptr(), norms.data_ptr(),
                                               packed.data_ptr(), bad.data_ptr(), st.cuda_stream)
            else:
                rc = lib.gcx_quantize(x.data_ptr(), n, bits, bucket, seed, norms.data_ptr(),
                                      packed.data_ptr(), bad.data_ptr(), st.cuda_stream)
            assert rc == 0
        for k in range(5):
            q(xs[k % 4], 42)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for k in range(20):
            q(xs[k % 4], 42 + k)
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        q(xs[0], 7)
        torch.cuda.synchronize()
        pk = packed.clone()
        same = True if ref_packed is None else bool(torch.equal(pk, ref_packed))
        if ref_packed is None:
            ref_packed = pk
        out[os.path.basename(path)] = {"quantize_us": ms * 1e3, "bit_identical": same}
        print(os.path.basename(path), f"{ms*1e3:.1f} us", "identical" if same else "DIFFERENT",
              flush=True)
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", "variants.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
