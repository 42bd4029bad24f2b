"""Writes tests/golden/plan_json/: a small planned batch in the reference's file formats,
produced by the reference's own writers (write_sequences_jsonl, block_graph_to_json,
placement_to_json, plan_to_json; inc/io.hpp) through planner/_build/libdcpplanner.so,
plus bundle.npz = the same plan flattened by the planner shim (to compare against on
machines without the planner). Run here (needs /root/reference):
    python tests/golden/make_plan_json.py"""
import os
import shutil
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from common import MIXED_SPECS  # noqa: E402
from paper_2510_10620_b200 import planner as PL  # noqa: E402

OUT = os.path.join(HERE, "plan_json")


def main():
    shutil.rmtree(OUT, ignore_errors=True)
    b = PL.Batch.from_specs(MIXED_SPECS, 4, 2, 128)
    bundle = PL.plan(b, 2, 256, eps_intra=0.4, eps_data=0.6, json_dir=OUT)
    bundle.save(os.path.join(OUT, "bundle.npz"))
    for f in sorted(os.listdir(OUT)):
        print(f, os.path.getsize(os.path.join(OUT, f)))


if __name__ == "__main__":
    main()
