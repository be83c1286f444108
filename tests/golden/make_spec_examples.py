"""Regenerates tests/golden/spec_examples.json: the SPEC.md worked examples
evaluated directly from the SPEC formulas in pure Python (independent of the
oracle), used to pin the oracle's perfmodel."""
import json
import math
import os


def prefill(P, hidden, layers, nd, peak, ce, lens):
    return (2.0 * P * sum(lens) + (4 * hidden * layers) * sum(l * l for l in lens)) / (nd * peak * ce)


def decode(P, byts, layers, kvh, hd, nd, bw, me, peak, ce, lens):
    kvb = 2 * layers * kvh * hd * byts
    mem = (P * byts + sum(lens) * kvb) / (nd * bw * me)
    comp = (2.0 * P * len(lens)) / (nd * peak * ce)
    return max(mem, comp)


if __name__ == "__main__":
    g = {
        "source": "SPEC.md worked examples, recomputed by tests/golden/make_spec_examples.py (pure Python)",
        "prefill": {"h100_512_s": prefill(70e9, 8192, 80, 4, 989e12, 0.5, [512]),
                    "910b2_1000_s": prefill(70e9, 8192, 80, 4, 400e12, 0.5, [1000])},
        "decode": {"h100_32x500_s": decode(70e9, 2, 80, 8, 128, 4, 3.35e12, 1.0, 989e12, 1.0, [500] * 32)},
        "capacity": {"7b_h100": math.floor((4 * 80e9 * 0.9 - 7e9 * 2) / 524288)},
    }
    json.dump(g, open(os.path.join(os.path.dirname(__file__), "spec_examples.json"), "w"), indent=1)
