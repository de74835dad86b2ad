"""Measures pinned host<->device copy bandwidth on the box (1D contiguous, one direction and
both directions at once) -- the bound of the end-to-end (skinny round trip) number."""
import json
import sys

import torch


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 720 * 1000 * 1000
    h1 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    res = {}
    for name, fn in [("h2d", lambda: d1.copy_(h1, non_blocking=True)),
                     ("d2h", lambda: h2.copy_(d2, non_blocking=True))]:
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            fn()
        e1.record()
        torch.cuda.synchronize()
        res[name + "_GBps"] = 3 * n / (e0.elapsed_time(e1) * 1e-3) / 1e9
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        with torch.cuda.stream(s1):
            d1.copy_(h1, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    res["bidir_total_GBps"] = 2 * 3 * n / (e0.elapsed_time(e1) * 1e-3) / 1e9
    print(json.dumps(res))


if __name__ == "__main__":
    main()


def stepper_copies():
    """Pitched 3D copies of the stepper (hc_stepper_upload/download) at 256^3 O3."""
    import os
    import time
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2211_13295_b200 import hydro
    g = hydro.make_geometry(256, 256, 256, 3)
    st = hydro.Stepper(g, hydro.make_params(3))
    host = torch.empty((g.mz, g.my, g.mx, 5), dtype=torch.float64, pin_memory=True).numpy()
    st.upload(host)
    st.download(host)
    t0 = time.perf_counter()
    for _ in range(3):
        st.upload(host)
        st.sync()
    t1 = time.perf_counter()
    for _ in range(3):
        st.download(host)
    t2 = time.perf_counter()
    print(json.dumps({"stepper_upload_GBps": 3 * host.nbytes / (t1 - t0) / 1e9,
                      "stepper_download_GBps": 3 * host.nbytes / (t2 - t1) / 1e9}))


if __name__ == "__main__" and len(sys.argv) > 2:
    stepper_copies()
