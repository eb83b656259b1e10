"""Golden outputs of the reference's own parsers (oracle/_ref) for the cases
in tests/ingest_cases.py.   python tests/golden/make_ingest_golden.py"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, ".."))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
from ingest_cases import FASTA, OVERLAPS, SEEDS  # noqa: E402
from oracle_py import Ref  # noqa: E402


def enc(r):
    if isinstance(r, tuple) and r and r[0] == "error":
        return {"error": r[1], "line": r[2], "message": r[3]}
    return r


def main():
    R = Ref()
    out = {"fasta": [], "seeds": [], "overlaps": []}
    for text, allowed in FASTA:
        r = R.parse_fasta(text.encode(), allowed)
        if r[0] == "error":
            out["fasta"].append(enc(r))
        else:
            out["fasta"].append({"symbols": r[0].decode(), "offsets": r[1].tolist(), "names": r[2]})
    for text in SEEDS:
        r = R.parse_tasks(text.encode(), False)
        out["seeds"].append(enc(r) if isinstance(r, tuple) else {"tasks": r.tolist()})
    for text in OVERLAPS:
        r = R.parse_tasks(text.encode(), True)
        out["overlaps"].append(enc(r) if isinstance(r, tuple) else {"tasks": r.tolist()})
    json.dump(out, open(os.path.join(HERE, "ingest.json"), "w"), indent=1)
    print({k: len(v) for k, v in out.items()})


if __name__ == "__main__":
    main()
