"""v-sharded multi-GPU step (placeholder until the sharded path lands)."""


def bench_sharded(args, cfg, metric, unit, config):
    raise NotImplementedError("v-sharded multi-GPU step not built yet")
