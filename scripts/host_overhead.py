"""Probe (GPU box): host time of one product call vs its kernel time
(BERT layers): the Python API (TwPlan.run, gemm_cto) and the raw C ABI."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2402_10876_b200 as tw  # noqa: E402
from paper_2402_10876_b200 import _native  # noqa: E402


def main():
    lib = _native.load_library()
    for k, n in [(768, 768), (768, 3072), (3072, 768)]:
        w = tw.round_to(tw.synthetic_matrix(0, k, n, 0), "fp16")
        _, tsm = tw.prune_tw(w, 0.75, 128)
        enc = tw.encode_cto(tsm)
        p = tw.TwPlan(enc, row_layout="runs")
        a = tw.round_to(tw.synthetic_matrix(0, 8192, k, 1), "fp16")
        x = p.prepare(torch.from_numpy(a).cuda())
        ct = torch.empty((p.info.n_condensed, 8192), dtype=torch.float16, device="cuda")
        s = _native.stream_handle()
        for _ in range(10):
            p.run(x, out=ct)
        torch.cuda.synchronize()
        N = 2000
        t0 = time.perf_counter()
        for _ in range(N):
            lib.tw_gemm_ex(p._handle, x.data_ptr(), 8192, x.stride(0), ct.data_ptr(), ct.stride(0),
                           1, 1, s)
        t_c = (time.perf_counter() - t0) / N * 1e6
        import os
        os.environ["TW_DEBUG_FLAGS"] = "64"
        t0 = time.perf_counter()
        for _ in range(N):
            lib.tw_gemm_ex(p._handle, x.data_ptr(), 8192, x.stride(0), ct.data_ptr(), ct.stride(0),
                           1, 1, s)
        t_nl = (time.perf_counter() - t0) / N * 1e6
        t0 = time.perf_counter()
        for _ in range(N):
            lib.tw_abi_version()
        t_ct = (time.perf_counter() - t0) / N * 1e6
        os.environ.pop("TW_DEBUG_FLAGS")
        print(f"  no-launch host {t_nl:.2f} us, bare ctypes call {t_ct:.2f} us")
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(N):
            p.run(x, out=ct)
        t_py = (time.perf_counter() - t0) / N * 1e6
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(200):
            p.run(x, out=ct)
        e1.record()
        torch.cuda.synchronize()
        t_k = e0.elapsed_time(e1) * 1e3 / 200
        a_dev = torch.from_numpy(a).cuda()
        tw.gemm_cto(a_dev, enc)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(200):
            tw.gemm_cto(a_dev, enc)
        t_api = (time.perf_counter() - t0) / 200 * 1e6
        torch.cuda.synchronize()
        print(f"{k}x{n}: host per call: C ABI {t_c:.1f} us, TwPlan.run {t_py:.1f} us, "
              f"gemm_cto (device A) {t_api:.1f} us; stream time per call {t_k:.1f} us")


if __name__ == "__main__":
    main()
