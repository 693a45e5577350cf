"""Golden vectors for suffix drafting and greedy acceptance, produced by the
REAL reference (``shiftsim.spec_decode.propose`` / ``_greedy_accept``,
spec_decode.py:105-149).  Run in the build container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_spec_golden.py

Writes ``tests/golden/spec_golden.json`` (the GPU box only reads the fixture).
"""

import json
import sys
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from shiftsim.spec_decode import SuffixIndex, _greedy_accept, propose  # noqa: E402


def main():
    rng = np.random.default_rng(2507)
    drafts = []
    for case in range(400):
        n = int(rng.integers(1, 80))
        alphabet = int(rng.choice([2, 3, 5, 16, 256]))
        if case % 4 == 0:  # periodic histories: long matches, replay into the suffix
            period = [int(t) for t in rng.integers(0, alphabet, int(rng.integers(1, 7)))]
            hist = (period * (n // len(period) + 1))[:n]
        else:
            hist = [int(t) for t in rng.integers(0, alphabet, n)]
        mm, ms, win = int(rng.integers(1, 5)), int(rng.integers(1, 10)), int(rng.integers(1, 40))
        limit = None if case % 3 else int(rng.integers(0, 12))
        d = propose(SuffixIndex(hist, min_match=mm, max_spec=ms, window=win), limit=limit)
        drafts.append({"history": hist, "min_match": mm, "max_spec": ms, "window": win,
                       "limit": limit, "tokens": list(d.tokens), "match_len": d.match_len})
    accepts = []
    for case in range(200):
        k = int(rng.integers(0, 8))
        vocab = 6
        rows = rng.standard_normal((k + 1, vocab))
        if case % 5 == 0:  # ties: lowest index wins
            rows[:, 3] = rows[:, 1] = rows.max(axis=1) + 1.0
        targets = [int(np.argmax(r)) for r in rows]
        draft = [t if rng.random() < 0.7 else int(rng.integers(0, vocab)) for t in targets[:k]]
        accepts.append({"draft": draft, "rows": rows.tolist(),
                        "emitted": [int(t) for t in _greedy_accept(draft, rows)]})
    out = Path(__file__).with_name("spec_golden.json")
    out.write_text(json.dumps({"source": "shiftsim.spec_decode (spec_decode.py:105-149)",
                               "propose": drafts, "greedy_accept": accepts}))
    print(f"wrote {out}: {len(drafts)} drafts, {len(accepts)} accepts")


if __name__ == "__main__":
    main()
