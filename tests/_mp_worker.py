"""Process body for the gloo world-size-2 tests (tests/test_search.py)."""

import os


def sharded_ga(rank: int, world: int, port: int, seed: int, out_dir: str, dedupe: bool = False) -> None:
    import json
    import random

    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from gpuoffload.evaluators import CostModelEvaluator
    from gpuoffload.ga import GAParams
    from gpuoffload.screen import screen_model

    from paper_2011_03602_b200.search import ShardedEvaluator, run_search_batched
    from _models import random_model

    class Counting(CostModelEvaluator):
        def __init__(self):
            super().__init__()
            self.calls = 0

        def measure(self, request):
            self.calls += 1
            return super().measure(request)

    class DedupeCounting(Counting):
        """Counting cost model with B200Evaluator's program-level dedupe keys."""

        dedupe = True

        @staticmethod
        def run_key(doc_key, payload):
            from paper_2011_03602_b200.evaluator import B200Evaluator

            return B200Evaluator.run_key(doc_key, payload)

        @staticmethod
        def _doc(model):
            from paper_2011_03602_b200.ir import document_of

            return document_of(model)

    model = random_model(random.Random(seed), max_depth=3)
    inner = DedupeCounting() if dedupe else Counting()
    ev = ShardedEvaluator(inner)
    stats = {}
    res = run_search_batched(model, screen_model(model), ev, GAParams(population_size=10, generations=6, seed=seed),
                             stats=stats)
    with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as f:
        json.dump({"best": list(res.best_genome), "time": res.best_time, "evals": res.evaluations_performed,
                   "hits": res.cache_hits, "local_calls": inner.calls,
                   "speculated_unused": stats["speculated_unused"],
                   "history": [[h.generation, h.best_time, h.mean_time, h.evaluations] for h in res.history]}, f)
    dist.barrier()
    dist.destroy_process_group()
