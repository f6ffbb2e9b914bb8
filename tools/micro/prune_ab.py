"""A/B timing of sf_prune_topk_rows from two builds of the library on the
same box (run once per build: `prune_ab.py old`, `prune_ab.py new`) (BERT-base x~, 12.6M, keep 0.1, row pointers): L2 flushed by a
256 MB write, back to back, and right after a GEMM."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch

here = os.path.dirname(os.path.abspath(__file__))
# one library per process (each links its own static cudart): argv[1] = old | new
which = sys.argv[1] if len(sys.argv) > 1 else "new"
libs = {which: ctypes.CDLL(os.path.join(here, "libslimfit_old.so") if which == "old" else
                           os.path.join(here, "..", "..", "paper_2305_18513_b200", "libslimfit_b200.so"))}
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn(16384, 768, generator=g, device="cuda")
x = (x - x.mean(-1, keepdim=True)) / x.std(-1, keepdim=True)
n, H = x.numel(), 768
k = -(-n // 10)
fl = torch.empty(64 << 20, device="cuda")
a_ = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
for _ in range(100):
    a_ @ a_
for name, lib in libs.items():
    lib.sf_prune_workspace_bytes.restype = ctypes.c_size_t
    lib.sf_prune_workspace_bytes.argtypes = [ctypes.c_int64]
    lib.sf_prune_topk_rows.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    ws = torch.empty(lib.sf_prune_workspace_bytes(n), dtype=torch.uint8, device="cuda")
    vals = torch.empty(k, device="cuda")
    idx = torch.empty(k, dtype=torch.int32, device="cuda")
    rp = torch.empty(n // H + 1, dtype=torch.int32, device="cuda")
    for mode in ("flushed", "back-to-back", "after-gemm"):
        ts = []
        for it in range(30):
            if mode == "flushed":
                fl.fill_(float(it))
            elif mode == "after-gemm":
                a_ @ a_
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            rc = lib.sf_prune_topk_rows(x.data_ptr(), n, k, 1, vals.data_ptr(), idx.data_ptr(), H, rp.data_ptr(),
                                        ws.data_ptr(), None)
            assert rc == 0, (name, rc)
            e1.record()
            if mode != "back-to-back":
                torch.cuda.synchronize()
            ts.append((e0, e1))
        torch.cuda.synchronize()
        t = sorted(a.elapsed_time(b) * 1e3 for a, b in ts[5:])
        ref = torch.sort(x.reshape(-1).abs(), descending=True).values[k - 1]
        assert vals.abs().min() >= ref, name      # the kept set really is the top k
        print(f"{name} {mode:13s}: median {t[len(t) // 2]:.1f} us, min {t[0]:.1f} us")
