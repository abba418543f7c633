"""Device-side bounds checks (stands in for compute-sanitizer, which the GPU
pool refuses): the library rebuilt with -DRIANN_BOUNDS checks the index and
capacity invariants of every frame kernel (pool offsets and list lengths,
descriptor and query indices, drawn positions and anchors, window bounds,
candidate-block and survivor capacities, K2 positions) and reports the first
failing site.  A config-0 stream on both frame paths, a config-1 crop, the
batch query API, sharded tables and the first two frames of config 3 (the
multi-pass first frame) must run clean, with fields equal to the normal
build's."""

import hashlib
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import hashlib, json, sys
sys.path.insert(0, %(repo)r)
import numpy as np
import paper_1508_07953_b200 as R
from paper_1508_07953_b200 import _native as N
from paper_1508_07953_b200 import workloads as W
from dataclasses import replace
assert N.lib().riann_debug_checks() == 1, "not the bounds-checked build"

def digest(fields):
    h = hashlib.sha256()
    for f in fields:
        h.update(np.ascontiguousarray(f.indices).tobytes())
        h.update(np.ascontiguousarray(f.distances).tobytes())
    return h.hexdigest()

out = {}
cfg = W.CONFIGS[0]
clip = W.clip(cfg, 4)
model = R.ReferenceModel.from_refs(W.reference_set(cfg), cfg.patch)
for path in (0, 1):
    N.set_frame_path(path)
    out["cfg0_path%%d" %% path] = digest([f for _, f, _ in R.stream_fields(model, clip)])
N.set_frame_path(0)
q = R.frame_units(clip[1], model)[:500]
res = R.riann_query_batch(model, q, np.arange(500) %% model.n, R.SearchParams(max_rings=20), keys=list(range(500)))
out["batch"] = hashlib.sha256(res["idx"].tobytes() + res["dist"].tobytes()).hexdigest()
c1 = replace(W.CONFIGS[1], height=120, width=160, frames=4)
clip1 = W.clip(c1)
m1 = R.ReferenceModel.from_refs(W.reference_set(c1), c1.patch)
out["cfg1"] = digest([f for _, f, _ in R.stream_fields(m1, clip1)])
out["cfg1_bands3"] = digest([f for _, f, _ in R.stream_fields(m1, clip1, devices=[0], bands=3)])
ms = R.ReferenceModel.from_refs(W.reference_set(c1), c1.patch)
st = R.shard_model(ms, devices=[0, 0, 0], shards=3)
out["cfg1_shards"] = digest([f for _, f, _ in R.stream_fields(ms, clip1)])
st.close()
if %(cfg3)r:
    c3 = W.CONFIGS[3]
    m3 = R.ReferenceModel.from_refs(W.reference_set(c3), c3.patch, channels=3)
    out["cfg3"] = digest([f for _, f, _ in R.stream_fields(m3, W.iter_clip(c3, 2))])
print("BOUNDS_JSON " + json.dumps(out))
'''


def _digest(R, fields):
    h = hashlib.sha256()
    for f in fields:
        h.update(np.ascontiguousarray(f.indices).tobytes())
        h.update(np.ascontiguousarray(f.distances).tobytes())
    return h.hexdigest()


def test_bounds_checked_build(tmp_path):
    lib = str(tmp_path / "libriann_bounds.so")
    env = dict(os.environ, RIANN_LIB=lib, RIANN_NVCC_DEFS="-DRIANN_BOUNDS")
    b = subprocess.run([sys.executable, "-m", "paper_1508_07953_b200.build"], cwd=REPO, env=env,
                       capture_output=True, text=True, timeout=900)
    assert b.returncode == 0 and os.path.exists(lib), b.stderr[-2000:]
    script = tmp_path / "run.py"
    script.write_text(SCRIPT % {"repo": REPO, "cfg3": True})
    r = subprocess.run([sys.executable, str(script)], cwd=REPO, env=dict(os.environ, RIANN_LIB=lib),
                       capture_output=True, text=True, timeout=1200)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-3000:]
    got = json.loads(next(line for line in r.stdout.splitlines() if line.startswith("BOUNDS_JSON "))[12:])

    # the same runs on the normal build (this process)
    from dataclasses import replace

    import paper_1508_07953_b200 as R
    from paper_1508_07953_b200 import workloads as W

    cfg = W.CONFIGS[0]
    clip = W.clip(cfg, 4)
    model = R.ReferenceModel.from_refs(W.reference_set(cfg), cfg.patch)
    assert got["cfg0_path0"] == got["cfg0_path1"] == _digest(R, [f for _, f, _ in R.stream_fields(model, clip)])
    c1 = replace(W.CONFIGS[1], height=120, width=160, frames=4)
    clip1 = W.clip(c1)
    m1 = R.ReferenceModel.from_refs(W.reference_set(c1), c1.patch)
    want1 = _digest(R, [f for _, f, _ in R.stream_fields(m1, clip1)])
    assert got["cfg1"] == got["cfg1_bands3"] == got["cfg1_shards"] == want1
    c3 = W.CONFIGS[3]
    m3 = R.ReferenceModel.from_refs(W.reference_set(c3), c3.patch, channels=3)
    assert got["cfg3"] == _digest(R, [f for _, f, _ in R.stream_fields(m3, W.iter_clip(c3, 2))])
