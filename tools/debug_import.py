"""Debug: reference state at KF 100 (pickle) -> one reference step vs device import + one step."""
import json, os, pickle, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests")); sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import bench_ref
from helpers import device_kf
from paper_2511_02036_b200 import workload as W
from paper_2511_02036_b200.config import FuseConfig, MatchConfig
from paper_2511_02036_b200.session import LocalMapper, store_for
from paper_2511_02036_b200.snapshot import state_arrays

w = bench_ref.ReferenceWindow("c2", "baseline", start=100)
pre = state_arrays(w.pipe.model, w.pipe.store, w.pipe._recent)
w.step()
m = w.pipe.model
seq = W.generate_sequence(W.bench_world("c2"))
intr = seq.intrinsics()
dev = LocalMapper(intr, neighbor_count=20, match=MatchConfig(neighbor_count=20), fuse=FuseConfig(n1=20, n2=5),
                  store=store_for(200, 1264))
dev.import_state(pre, processed=w.pipe._processed - 1)
print("recent", len(pre["recent_id"]), "processed", w.pipe._processed - 1)
dev.process(device_kf(seq.records[100], intr))
s = dev.snapshot(with_covis=False)
obs = s.observations()
n = max(len(s.alive), len(m.points))
bad = 0
for i in range(n):
    p = m.points.get(i)
    if p is None or i >= len(s.alive):
        print("id space", i, len(s.alive), len(m.points)); break
    if bool(s.alive[i]) != p.alive:
        print("alive", i, bool(s.alive[i]), p.alive); bad += 1
    elif p.alive:
        if obs[i] != dict(sorted(p.observations.items())):
            print("obs", i, obs[i], sorted(p.observations.items())); bad += 1
        if (int(s.found[i]), int(s.visible[i])) != (p.found_count, p.visible_count):
            print("found/vis", i, (int(s.found[i]), int(s.visible[i])), (p.found_count, p.visible_count)); bad += 1
        if not np.array_equal(s.rep[i], p.rep_descriptor):
            print("rep", i); bad += 1
        if not np.array_equal(s.counts[i], m.counter_matrix[i]):
            print("counts", i, s.counts[i], m.counter_matrix[i]); bad += 1
    if bad > 15:
        break
print("bad", bad, "stats", dev.stats, dev.fused, dev.culled)
print("ref recent after", len(w.pipe._recent), "dev recent", len(dev.recent()))
print("borderline (epi, gates, fusion, rint) after the imported step:", list(dev.totals().borderline))
# the same keyframe natively from an empty map, for comparison
nat = LocalMapper(intr, neighbor_count=20, match=MatchConfig(neighbor_count=20), fuse=FuseConfig(n1=20, n2=5),
                  store=store_for(200, 1264))
for k in range(101):
    nat.process(device_kf(seq.records[k], intr))
t = nat.totals()
print("native run 0..100 borderline", list(t.borderline))
sn = nat.snapshot(with_covis=False)
for i in (902, 1292, 2010):
    print(i, "native vis", int(sn.visible[i]), "import vis", int(s.visible[i]), "ref", m.points[i].visible_count,
          "pos native-ref", np.abs(sn.pos[i] - m.points[i].position).max())
