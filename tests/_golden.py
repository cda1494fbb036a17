import os

_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def paper_observations():
    out = {}
    with open(os.path.join(_DIR, "paper_observations.txt")) as f:
        for line in f:
            line = line.split("#", 1)[0].strip()
            if not line:
                continue
            k, v = (t.strip() for t in line.split("=", 1))
            out[k] = float(v)
    return out
