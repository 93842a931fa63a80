"""Flatten a bench.py JSON line (key = value), for reading results."""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
skip = set(sys.argv[2:])


def show(d, p=""):
    for k, v in d.items():
        if k in skip:
            continue
        if isinstance(v, dict):
            show(v, p + k + ".")
        else:
            print(p + k, "=", str(v)[:160])


show(d)
