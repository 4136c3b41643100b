"""Run bench_sharded under torchrun with the given rank count (a 1-rank run
exercises the NCCL plumbing, the sharded state and the cut-off protocol on a
single GPU)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2408_11235_b200 as sk  # noqa: E402
from paper_2408_11235_b200 import sharding  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--steps", type=int, default=12)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--no-e2e", action="store_true")
ap.add_argument("--e2e-steps", type=int, default=2)
args = ap.parse_args()
args.gpus = int(os.environ.get("WORLD_SIZE", "1"))
cfg = sk.named_config(args.config)
sharding.bench_sharded(args, cfg, bench.METRIC, bench.UNIT, bench.config_dict(args, cfg))
