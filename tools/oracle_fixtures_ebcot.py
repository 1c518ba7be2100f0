"""Oracle fixtures for the opt-in JPEG2000-style base layer (parity UNPINNED:
the reference has no such layer; the C oracle oracle/ebcot_oracle.c is the
only CPU restatement).  Writes tests/golden/oracle_ebcot.json: container
SHA-256 of full-size fields compressed with base_codec="ebcot"."""
import hashlib
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))

import golden_inputs as gi  # noqa: E402
from oracle import oracle  # noqa: E402
from paper_2510_22265_b200 import fields  # noqa: E402

CASES = [
    ("temperature", dict(seed=1, mean=280.0, std=15.0), 0.01),
    ("temperature", dict(seed=2, mean=250.0, std=5.0), 0.001),
    ("precip", dict(seed=2005), 0.01),
]


def field_of(kind, kw):
    if kind == "temperature":
        return fields.temperature_like(721, 1440, **kw)
    return fields.precip_like(721, 1440, **kw)


def main():
    oracle.build()
    out = []
    for kind, kw, eps in CASES:
        a = field_of(kind, kw)
        blob = oracle.compress(a, rel_error=eps, base_codec="ebcot")
        out.append({"kind": kind, "kw": kw, "eps": eps, "input_sha": gi.sha(a),
                    "container_sha": hashlib.sha256(blob).hexdigest(), "container_len": len(blob),
                    "decoded_sha": gi.sha(oracle.decompress(blob))})
        print(out[-1], flush=True)
    with open(os.path.join(REPO, "tests", "golden", "oracle_ebcot.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
