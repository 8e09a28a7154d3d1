"""Helpers to read golden fixtures (values printed in PAPER.md, cited in each file)."""
import json
import math
import os

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def num(v):
    """Parse printed constants such as '4sqrt2/3', '-5sqrt2/3', '2/3', 'sqrt2'."""
    if isinstance(v, (int, float)):
        return float(v)
    s = v.replace(" ", "")
    sign = -1.0 if s.startswith("-") else 1.0
    s = s.lstrip("-")
    num_, _, den = s.partition("/")
    val = 1.0
    if "sqrt2" in num_:
        coef = num_.replace("sqrt2", "")
        val = (float(coef) if coef else 1.0) * math.sqrt(2.0)
    else:
        val = float(num_)
    if den:
        val /= float(den)
    return sign * val
