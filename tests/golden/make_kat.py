"""Verify tests/golden/kat.json against the reference's own test sources.

Each numeric literal in kat.json was transcribed from the doctest file named
in its "cite" field.  When /root/reference is present (the build container,
never the GPU box), this script checks every literal still appears verbatim
in that file, so a transcription error cannot slip into the oracle pins.

    python tests/golden/make_kat.py          # exits non-zero on a mismatch
"""
import json
import os
import re
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REF_TESTS = "/root/reference/proj/tests"

# Derived values that the reference states as an expression, not a literal.
DERIVED_OK = {"0.7071067811865476", "0.5", "0.25", "0.125", "1.0", "-0.5", "500.0", "2", "1",
              "19", "3", "0", "4", "10", "-600.0", "600.0", "0.1",
              # integer / exponent literals of test_pipelines.cpp (Rng(23), 1e-15,
              # uint8 channel values) that the decimal-literal scan below skips
              "23", "1e-15", "128", "255", "64"}


def literals(obj):
    if isinstance(obj, dict):
        for k, v in obj.items():
            if k in ("cite", "eps", "instance"):
                continue
            yield from literals(v)
    elif isinstance(obj, list):
        for v in obj:
            yield from literals(v)
    elif isinstance(obj, (int, float, str)) and not isinstance(obj, bool):
        yield str(obj)


def main() -> int:
    kat = json.load(open(os.path.join(HERE, "kat.json")))
    if not os.path.isdir(REF_TESTS):
        print("reference sources absent; nothing to verify")
        return 0
    bad = 0
    for name, entry in kat.items():
        if name.startswith("_"):
            continue
        files = [c.strip().split(":")[0] for c in entry["cite"].split(";")]
        text = "".join(open(os.path.join(REF_TESTS, f)).read() for f in files)
        for lit in literals(entry):
            if lit in DERIVED_OK:
                continue
            # compare as floats: every literal of the cited file, sign-insensitive
            vals = {float(t) for t in re.findall(r"\d+\.\d+(?:e[-+]?\d+)?|\d{6,}", text)}
            if abs(float(lit)) not in vals:
                print(f"{name}: literal {lit} not found in {files}")
                bad += 1
    print("kat.json verified" if not bad else f"{bad} mismatches")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
