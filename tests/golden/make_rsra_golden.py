"""Add sha256 digests of REFERENCE-written .rsra files (and reference toy
runtime decodes) to golden.json.

Runs the reference package (rsrmv @ /root/reference) in the build container:
for every small case of make_golden.SMALL and every LARGE config it saves the
reference artifact with rsrmv.artifact_io.save (pkg/src/rsrmv/artifact_io.py)
and records sha256 + length of the file bytes under golden.json["rsra"].

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_rsra_golden.py
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import make_golden as mg  # noqa: E402  (puts the reference on sys.path)
from rsrmv import artifact_io, bench, preproc, toyrt  # noqa: E402

TOY = [  # (seed, d, V, depth, k, prompt, steps)
    (0, 64, 256, 2, 4, [1, 2, 3], 24),
    (7, 96, 128, 3, 5, [5], 16),
]


def rsra_digest(a):
    with tempfile.TemporaryDirectory() as td:
        fp = os.path.join(td, "a.rsra")
        artifact_io.save(a, fp)
        blob = open(fp, "rb").read()
    return dict(sha=hashlib.sha256(blob).hexdigest(), bytes=len(blob))


def main():
    out = {"small": {}, "large": {}}
    for i, (m, n, bw, k, tw, seed, dens, ws) in enumerate(mg.SMALL):
        p = mg.packed_for(m, n, bw, seed, dens, ws)
        out["small"][str(i)] = rsra_digest(preproc.preprocess(p, k, tile_width=tw))
    for name, m, n, bw, k, seed in mg.LARGE:
        p = bench.random_matrix(m, n, bw, seed)
        out["large"][name] = rsra_digest(preproc.preprocess(p, k))
        print(name, out["large"][name], flush=True)
    toy = []
    for seed, d, V, depth, k, prompt, steps in TOY:
        model = toyrt.build_toy_model(seed, d, V, depth, k=k)
        toks, _ = toyrt.greedy_decode(model, toyrt.RSR, prompt, steps)
        toy.append(dict(seed=seed, d=d, V=V, depth=depth, k=k, prompt=prompt, steps=steps,
                        tokens=toks, digest=model.digest()))
    path = os.path.join(HERE, "golden.json")
    g = json.load(open(path))
    g["rsra"] = out
    g["toyrt"] = toy
    with open(path, "w") as f:
        json.dump(g, f, indent=1)


if __name__ == "__main__":
    main()
