"""Parser for tests/golden/*.dag (format in tests/golden/README.md)."""
import os

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(fname):
    cases = {}
    cur = None
    with open(os.path.join(GOLDEN, fname)) as f:
        for raw in f:
            line = raw.split("#", 1)[0].strip()
            if not line:
                continue
            t = line.split()
            if t[0] == "case":
                cur = dict(name=t[1], trace=[], vertices=[], edges=set(), waits=None)
            elif t[0] == "end":
                cases[cur["name"]] = cur
                cur = None
            elif t[0] == "launch":
                args = []
                for a in t[2:]:
                    arr, mode = a.split(":")
                    args.append((arr, mode))
                cur["trace"].append(("launch", t[1], args))
            elif t[0] == "host":
                cur["trace"].append(("host", t[1], t[2], int(t[3]), int(t[4])))
            elif t[0] == "sync":
                cur["trace"].append(("sync",))
            elif t[0] == "expect":
                if t[1] == "vertex":
                    cur["vertices"].append((int(t[2]), t[3], int(t[4])))
                elif t[1] == "edge":
                    cur["edges"].add((int(t[2]), int(t[3]), t[4]))
                elif t[1] == "waits":
                    cur["waits"] = int(t[2])
                else:
                    raise ValueError(line)
            else:
                raise ValueError(line)
    return cases


def all_cases():
    out = []
    for fn in sorted(os.listdir(GOLDEN)):
        if fn.endswith(".dag"):
            for name, c in load(fn).items():
                out.append((f"{fn}:{name}", c))
    return out
