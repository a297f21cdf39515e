"""Time K3 (gcx_dequantize) of the compile-time variants in
paper_2111_08617_b200/variants/ on C1 and check they are bit-identical to
the shipped libgcx.so.  Development tool, run under gpurun."""
import ctypes as C
import glob
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    n, bits, bucket = 25_557_032, 4, 128
    torch.cuda.set_device(0)
    nb = (n + bucket - 1) // bucket
    cap = 4 * ((n * (bits + 1) + 31) // 32)
    g = torch.Generator(device="cuda").manual_seed(1)
    sets = [(torch.rand(nb, generator=g, device="cuda") + 0.5,
             torch.randint(0, 256, (cap,), generator=g, device="cuda", dtype=torch.uint8)) for _ in range(4)]
    out = torch.empty(n, device="cuda")
    st = torch.cuda.current_stream()
    libs = [os.path.join(ROOT, "paper_2111_08617_b200", "libgcx.so")] + sorted(
        glob.glob(os.path.join(ROOT, "paper_2111_08617_b200", "variants", "*.so")))
    ref = None
    for path in libs:
        lib = C.CDLL(path)
        lib.gcx_dequantize.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int, C.c_uint64,
                                       C.c_void_p, C.c_void_p]
        def d(k):
            nr, pk = sets[k % 4]
            assert lib.gcx_dequantize(nr.data_ptr(), pk.data_ptr(), n, bits, bucket, out.data_ptr(),
                                      st.cuda_stream) == 0
        for k in range(5):
            d(k)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for k in range(40):
            d(k)
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 40
        d(0)
        torch.cuda.synchronize()
        o = out.clone()
        same = ref is None or bool(torch.equal(o, ref))
        ref = o if ref is None else ref
        print(os.path.basename(path), f"{ms*1e3:.1f} us", "identical" if same else "DIFFERENT",
              f"{(4*n + cap + 4*nb)/ms/1e6:.0f} GB/s", flush=True)


if __name__ == "__main__":
    main()
