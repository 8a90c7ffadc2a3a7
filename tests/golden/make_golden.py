"""Write tests/golden/config1_golden.json -- calls ONLY oracle/ and synth/ (never the CUDA path).

BASELINE config 1: single W4A4 linear, M=16 tokens, K=1024, N=1024, group 128, 128 INT8 outliers,
seed 0.  Stores sha256 digests of every oracle intermediate plus a few sampled values, so that an
accidental change of the oracle's arithmetic (without a commit naming the paper passage that
justifies it) fails tests/test_oracle_golden.py.
"""
import hashlib
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import oracle  # noqa: E402
import synth   # noqa: E402


def digests(M=16, N=1024, K=1024, seed=0):
    X, W, perm = synth.problem(M, N, K, seed)
    r = oracle.quantized_linear(X, perm, W, K)
    out = {k: hashlib.sha256(np.ascontiguousarray(v).tobytes()).hexdigest() for k, v in r.items()}
    out["inputs"] = hashlib.sha256(X.tobytes() + W.tobytes() + perm.tobytes()).hexdigest()
    out["c_samples"] = {f"{m},{n}": float(r["c"][m, n]) for m, n in [(0, 0), (7, 511), (15, 1023)]}
    return out


if __name__ == "__main__":
    d = digests()
    d["_about"] = ("BASELINE config 1 (M=16,K=1024,N=1024,seed 0) oracle digests; written by "
                   "tests/golden/make_golden.py from oracle/ only")
    (Path(__file__).parent / "config1_golden.json").write_text(json.dumps(d, indent=1) + "\n")
    print(json.dumps(d, indent=1))
