"""Write the REAL reference's sequence file (synth.write_sequence, JSONL with hex
descriptors) for the orbit7 workload as a fixture for the ingest tests; run in the build
container where /root/reference is importable:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_jsonl.py
"""

import json
import os
import sys

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

from localmap import synth  # noqa: E402

GOLD = json.load(open(os.path.join(HERE, "golden.json")))
cfg = synth.WorldConfig(**GOLD["workloads"]["orbit7"]["config"])
synth.write_sequence(synth.generate_sequence(cfg), os.path.join(HERE, "orbit7_reference.jsonl"))
print("wrote", os.path.join(HERE, "orbit7_reference.jsonl"))
