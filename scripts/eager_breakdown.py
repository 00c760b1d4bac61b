"""Where the host time of an eager 512x512x32 call goes: the public call, the
same C ABI call made directly through ctypes with prepared arguments, the
Python argument preparation alone, and an empty ctypes round trip; with the
default plan, K2s (IH_SMALL=1) and without PDL (IH_NO_PDL=1) -- one JSON line."""
import ctypes, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1711_01919_b200 import device, _native

img = device.upload_image(np.random.default_rng(0).integers(0, 256, (512, 512), dtype=np.uint8))
lut = ((np.arange(256) * 32) // 256).astype(np.uint8)
out = device.empty_output(1, 32, 512, 512, "cuda")[0]
L = _native.lib()


def per_call(fn, n=3000):
    for _ in range(100):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return round((time.perf_counter() - t0) / n * 1e6, 2)


res = {"mode": os.environ.get("MODE", "default")}
res["public_us"] = per_call(lambda: device.integral_histogram(img, lut, 32, out=out))
a = device._prepare_args(img, lut, 32, None, "auto", None)
ws = device._workspace_for(a, None)
args = (a.images.data_ptr(), a.frames, a.H, a.W, a.pitch, a.fstride, device._lut_ptr(a), a.bins,
        a.lo, a.hi, out.data_ptr(), ws.data_ptr(), ws.numel() * ws.element_size(), a.kernel, a.stream)
res["abi_us"] = per_call(lambda: L.ih_integral_histogram(*args))
res["prepare_args_us"] = per_call(lambda: device._prepare_args(img, lut, 32, None, "auto", None))
res["ctypes_empty_us"] = per_call(lambda: L.ih_abi_version())
res["plan"] = device.plan(1, 512, 512, 32)["launches"]
print(json.dumps(res), flush=True)
