"""Oracle text trace IO (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).

SPEC.md:132-139, 170: header ``#moeplace-trace v1 L=<L> E=<E> K=<K>``, then one line per token,
``chunk_id<TAB>layer0:e,..,e<TAB>...<TAB>layer{L-1}:e,..,e``; errors carry the 1-based line
number (header = line 1).  The product parses and writes on the device only; this plain-Python
restatement is the checker the tests compare it with (line numbers, regrouping, byte-identical
canonical output).
"""
from __future__ import annotations

import re

import numpy as np

HEADER = re.compile(r"^#moeplace-trace v1 L=(\d+) E=(\d+) K=(\d+)\s*$")
FIELD = re.compile(r"^(?:layer)?(\d+):(.*)$")


class TextParseError(ValueError):
    def __init__(self, msg: str, line_no: int):
        super().__init__(f"line {line_no}: {msg}")
        self.line_no = line_no


def parse_text(path):
    """-> (shape (L, E, K) or None for an empty file, selections int64 [N, L, K] in file order,
    chunk id per token int64 [N])."""
    with open(path, "r") as f:
        lines = f.read().split("\n")
    if lines and lines[-1] == "":
        lines.pop()
    if not lines:
        return None, np.zeros((0, 0, 0), np.int64), np.zeros(0, np.int64)
    m = HEADER.match(lines[0])
    if not m:
        raise TextParseError("missing or malformed header", 1)
    L, E, K = (int(m.group(i)) for i in (1, 2, 3))
    if L < 1 or E < 1 or K < 1 or K > E:
        raise TextParseError("bad model shape in header", 1)
    N = len(lines) - 1
    sel = np.empty((N, L, K), dtype=np.int64)
    cid = np.empty(N, dtype=np.int64)
    for i, line in enumerate(lines[1:]):
        ln = i + 2
        parts = line.rstrip("\r").split("\t")
        if len(parts) != L + 1:
            raise TextParseError(f"expected {L} layer fields, found {len(parts) - 1}", ln)
        try:
            cid[i] = int(parts[0])
        except ValueError:
            raise TextParseError(f"bad chunk id {parts[0]!r}", ln) from None
        if cid[i] < 0:
            raise TextParseError("negative chunk id", ln)
        for l in range(L):
            fm = FIELD.match(parts[l + 1])
            if not fm or int(fm.group(1)) != l:
                raise TextParseError(f"malformed field {parts[l + 1]!r}", ln)
            items = fm.group(2).split(",")
            if len(items) != K:
                raise TextParseError(f"layer {l}: expected {K} experts", ln)
            try:
                vals = [int(v) for v in items]
            except ValueError:
                raise TextParseError(f"layer {l}: non-integer expert index", ln) from None
            if any(v < 0 or v >= E for v in vals):
                raise TextParseError(f"layer {l}: expert index outside [0, {E})", ln)
            if len(set(vals)) != K:
                raise TextParseError(f"layer {l}: repeated expert index", ln)
            sel[i, l] = vals
    return (L, E, K), sel, cid


def regroup(sel, cid):
    """Stable regroup by ascending chunk id: (sel, chunk ids [C], bounds [C+1])."""
    order = np.argsort(cid, kind="stable")
    ids, counts = np.unique(cid[order], return_counts=True)
    return sel[order], ids.astype(np.int64), np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)


def write_text(path, shape, sel, cid_per_token) -> None:
    """Canonical text form of token-major selections (tokens in the given order)."""
    L, E, K = shape
    with open(path, "w") as f:
        f.write(f"#moeplace-trace v1 L={L} E={E} K={K}\n")
        prefixes = [f"layer{l}:" for l in range(L)]
        for t in range(sel.shape[0]):
            f.write(str(int(cid_per_token[t])) + "\t" + "\t".join(
                prefixes[l] + ",".join(str(int(v)) for v in sel[t, l]) for l in range(L)) + "\n")
