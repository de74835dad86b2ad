"""Generates tests/golden/ from the REFERENCE library (oracle/_ref/libhydro_ref.so, built by
`make -C oracle ref` from the unmodified /root/reference/proj sources). Run in the build
container: python tests/golden/make_golden.py"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from oracle import pyoracle as po  # noqa: E402
from tests.golden import golden  # noqa: E402


def main():
    ref = po.Reference()
    ref.set_threads(8)
    man = {}
    for name, meta in golden.CASES.items():
        out = golden.run_case(ref, meta)
        man[name] = dict(meta=meta, digests={k: golden.digest(v) for k, v in out.items()})
        if not meta.get("digest_only"):
            keep = {k: out[k] for k in ("skinny", "dts", "rate")}
            np.savez_compressed(os.path.join(golden.HERE, name + ".npz"), **keep)
        print(name, man[name]["digests"]["skinny"][:16], out["dts"])
    with open(golden.MANIFEST, "w") as f:
        json.dump(man, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
