"""Golden vectors of the reference's prompt assembly (TEST INFRASTRUCTURE; needs
/root/reference, i.e. oracle/_ref built): random templates in the placeholder text form
over random exchange histories -- clamped and out-of-range slices, missing exchanges,
literal words with mixed whitespace, malformed placeholders -- through the unmodified
parse_prompt_template + assemble_prompt / assemble_resolvable_prefix (prompt.cpp:75-164,
oracle/ref_shim.cpp pref_assemble).  Writes tests/golden/prompt_golden.json.gz.

  python tests/golden/make_prompt_golden.py
"""
import gzip
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

WORDS = ["alpha", "beta", "gamma", "delta", "plan", "code", "x", "y2", "zeta-3", "ünï"]
WS = [" ", "  ", "\t", "\n", " \t ", "\r\n"]


def rand_template(rng, ids, missing):
    parts = []
    for _ in range(int(rng.integers(1, 7))):
        k = rng.random()
        if k < 0.35:
            n = int(rng.integers(0, 5))
            txt = "".join(str(rng.choice(WS)) + str(rng.choice(WORDS)) for _ in range(n))
            if rng.random() < 0.5:
                txt += str(rng.choice(WS))
            parts.append(txt)
        elif k < 0.95:
            rid = str(rng.choice(missing)) if (missing and rng.random() < 0.15) else \
                str(rng.choice(ids))
            src = "request" if rng.random() < 0.5 else "response"
            a = int(rng.integers(0, 400))
            b = a + int(rng.integers(1, 400))
            parts.append("${%s:%s:[%d,%d]}" % (rid, src, a, b))
        else:  # malformed placeholders (parse error in the reference)
            parts.append(str(rng.choice(["${a:request:[5,5]}", "${a:req:[0,1]}", "${a:request:0,1}",
                                          "${a:request:[3,1]}", "${nocolon}", "${a:request:[1,2]"])))
    return "".join(parts)


def main():
    from oracle.py_oracle import Reference
    ref = Reference(16)
    rng = np.random.default_rng(2604)
    cases = []
    for t in range(250):
        n_ex = int(rng.integers(1, 6))
        ids = [f"req_{t}_{k}" for k in range(n_ex)]
        ex = {}
        for k in ids:
            ex[k] = (rng.integers(0, 1 << 40, size=int(rng.integers(0, 300)), dtype=np.uint64),
                     rng.integers(0, 1 << 40, size=int(rng.integers(0, 300)), dtype=np.uint64))
        text = rand_template(rng, ids, [f"gone_{t}"])
        rec = {"text": text, "ex": {k: [v[0].tolist(), v[1].tolist()] for k, v in ex.items()}}
        for prefix in (0, 1):
            rc, toks, comp = ref.assemble(text, ex, prefix=bool(prefix))
            rec[f"rc{prefix}"] = rc
            rec[f"tok{prefix}"] = [] if toks is None else [int(x) for x in toks]
            rec[f"complete{prefix}"] = comp
        cases.append(rec)
    path = os.path.join(HERE, "prompt_golden.json.gz")
    with gzip.open(path, "wt") as f:
        json.dump({"cases": cases}, f)
    print("wrote", path, len(cases), "cases")


if __name__ == "__main__":
    main()
