"""Batched and sharded GA drivers.

``run_search_batched`` is the reference GA (``run_search``, src/ga.py:246-285)
with one change: each generation's not-yet-cached genomes are measured in ONE
``evaluator.measure_batch`` call (all B200 workers in parallel, or all ranks of
a process group) instead of one ``measure`` at a time (src/ga.py:270).  The
operators, the RNG stream, the memo semantics, the cache-hit count, the
history and the final selection are the reference's own, so with a
deterministic evaluator the ``SearchResult`` is identical to ``run_search``'s
(tests/test_search.py).  SPEC.md:286 allows exactly this ("results are merged
in genome order so outcomes are independent of completion order").

**Speculative prefetch, commit on demand** (SURVEY.md §8e).  When the
evaluator measures ``parallel_width`` patterns at once (B200 workers x ranks)
and a generation's fresh genomes do not fill the last round, the idle slots
measure not-yet-requested genomes of the (small) genome space into a side
cache.  A side-cache result is committed -- counted in
``evaluations_performed``, reported to ``on_evaluation``, entered in the memo
-- only when the GA later asks for that genome, so the ``SearchResult`` is
still the reference's under a deterministic evaluator.  On Himeno L
(64-genome space, fresh genomes per generation 62, 0, 0, 0, 0, 1, 1, ...)
eight B200s then finish the whole search in the first round instead of
paying two more serial rounds later.

``ShardedEvaluator`` spreads a batch over the ranks of a ``torch.distributed``
process group (gloo, host-side results only: fitness units are independent,
so there is no data-path collective): requests are assigned longest-predicted
first (the reference cost model, src/evaluators.py:74-109) to the least
loaded rank, each rank measures its share on its own B200, and the results
are all-gathered so every rank continues with the same cache.
"""

from __future__ import annotations

from .evaluator import _result_cls


def _ga():
    import gpuoffload.ga as ga  # the reference GA (operators, dataclasses)

    return ga


class _BatchRunner:
    """GenomeEvaluator (src/ga.py:85-134) with batch submission."""

    def __init__(self, model, space, evaluator, backend, on_evaluation, speculate: bool | None = None):
        ga = _ga()
        from gpuoffload.evaluators import EvaluationRequest
        from gpuoffload.model import ModelIndex, ReplacedBlock

        self._Request = EvaluationRequest
        self.ga = ga
        self.model = model
        self.space = space
        self.evaluator = evaluator
        self.backend = backend
        self.on_evaluation = on_evaluation
        self.index = ModelIndex(model)
        self.cache: dict = {}
        self.evaluations = 0
        self.cache_hits = 0
        self.replaced_blocks = tuple(st for _, _, st in model.walk_statements() if isinstance(st, ReplacedBlock))
        self._needs_code = getattr(evaluator, "needs_code", True)
        self.width = max(1, int(getattr(evaluator, "parallel_width", 1)))
        if speculate is None:
            speculate = self.width > 1 and space.length <= SPECULATE_MAX_BITS
        self.speculate = speculate
        self.side: dict = {}       # speculative (request, result) by genome, not yet committed
        self.speculated = 0        # patterns measured speculatively

    def _request(self, bits, tags):
        from gpuoffload.codegen import emit_annotated
        from gpuoffload.patterns import pattern_from_genome
        from gpuoffload.transfers import plan_transfers

        pattern = pattern_from_genome(self.model, self.space, bits)
        plan = plan_transfers(self.model, pattern, self.index)
        code = emit_annotated(self.model, pattern, plan, self.backend) if self._needs_code else ""
        return self._Request(model=self.model, pattern=pattern, transfer_plan=plan, emitted_code=code,
                             backend=self.backend, replaced_blocks=self.replaced_blocks, tags=dict(tags))

    def _measure_all(self, requests) -> list:
        """Measure a batch; an ``OSError`` out of the evaluator (harness I/O,
        a missing compiler, a full disk) makes the affected requests
        ``runtime_error`` instead of aborting the search, as the reference's
        ``GenomeEvaluator.evaluate`` does (src/ga.py:124-128)."""
        if not requests:
            return []
        measure_batch = getattr(self.evaluator, "measure_batch", None)
        if measure_batch is not None:
            try:
                return measure_batch(requests)
            except OSError:
                pass  # re-measure one by one so only the failing requests are infeasible
        return [self._measure_one(r) for r in requests]

    def _measure_one(self, request):
        from gpuoffload.evaluators import MeasurementResult

        try:
            return self.evaluator.measure(request)
        except OSError as exc:
            return MeasurementResult(None, "runtime_error", getattr(self.evaluator, "evaluator_id", "unknown"),
                                     f"evaluator I/O failure: {exc}")

    def evaluate_population(self, population, tags) -> list:
        """Fitness of every individual, in population order.  First
        occurrences of uncached genomes are measured together; repeats (in
        this generation or earlier) are cache hits, exactly as the serial
        loop counts them."""
        ga = self.ga
        fresh: list[tuple] = []
        seen = set()
        for bits in population:
            bits = tuple(bits)
            if bits not in self.cache and bits not in seen:
                seen.add(bits)
                fresh.append(bits)
        fresh_res = {b: self.side.pop(b) for b in fresh if b in self.side}
        to_measure = [b for b in fresh if b not in fresh_res]
        extra: list[tuple] = []
        if self.speculate and to_measure and len(to_measure) % self.width:
            need = self.width - len(to_measure) % self.width
            known = set(self.cache) | set(self.side) | set(fresh)
            for g in self.space.all_genomes():
                if len(extra) == need:
                    break
                if tuple(g) not in known:
                    extra.append(tuple(g))
        batch = to_measure + extra
        requests = [self._request(b, tags) for b in batch]
        results = self._measure_all(requests)
        for bits, req, res in zip(batch, requests, results):
            if bits in seen:
                fresh_res[bits] = (req, res)
            else:
                self.side[bits] = (req, res)
                self.speculated += 1
        out = []
        for bits in population:
            bits = tuple(bits)
            if bits in self.cache:
                self.cache_hits += 1
                out.append(self.cache[bits])
                continue
            req, res = fresh_res[bits]
            fit = ga.Fitness(res.time_seconds, res.evaluator_id)
            self.cache[bits] = fit
            self.evaluations += 1
            if self.on_evaluation is not None:
                self.on_evaluation(bits, req, res)
            out.append(fit)
        return out


SPECULATE_MAX_BITS = 12  # speculate only in genome spaces of <= 4096 patterns


def run_search_batched(model, verdicts, evaluator, params, backend: str = "c_openacc", on_evaluation=None,
                       speculate: bool | None = None, stats: dict | None = None, confirm_top: int = 0,
                       confirm_repeats: int = 3):
    """``run_search`` (src/ga.py:246-285) with per-generation batch
    measurement (and speculative prefetch when ``speculate``; default: on
    when the evaluator is wider than one pattern).  ``stats`` (optional dict)
    receives ``speculated`` / ``speculated_unused`` counts.

    ``confirm_top=k`` (opt-in; off keeps the reference's final selection):
    patterns measured concurrently share host cores, host memory bandwidth
    and PCIe, so their fitness can drift from the solo time (tools/ga_drift.py:
    <= 9 % with two concurrent patterns, up to 1.6x with eight sharing one
    B200).  The k fastest feasible genomes are then re-measured one at a time
    (``evaluator.measure_solo``, best of ``confirm_repeats``; ``measure`` if
    the evaluator has none) and the fastest confirmed one is returned;
    ``stats["confirmed"]`` lists (genome, search time, solo time)."""
    ga = _ga()
    from gpuoffload.patterns import PatternError, build_genome_space

    space = build_genome_space(model, verdicts)
    if space.is_empty:
        raise PatternError("no offloadable loops; skip the search and use the CPU-only pattern")
    runner = _BatchRunner(model, space, evaluator, backend, on_evaluation, speculate)
    import random

    if space.length <= 2:
        fits = runner.evaluate_population(list(space.all_genomes()), {"generation": 0})
        history = (ga._generation_stats(0, fits, runner.evaluations),)
    else:
        rng = random.Random(params.seed)
        population = ga.init_population(space.length, params, rng)
        hist = []
        for gen in range(params.generations):
            fits = runner.evaluate_population(population, {"generation": gen})
            hist.append(ga._generation_stats(gen, fits, runner.evaluations))
            if gen + 1 < params.generations:
                population = ga.next_generation(population, fits, params, rng)
        history = tuple(hist)
    if stats is not None:
        stats.update(speculated=runner.speculated, speculated_unused=len(runner.side))
    best_bits, best_time, no_offload = ga._best_of_cache(runner.cache, space.length)
    if confirm_top > 0:
        best_bits, best_time = _confirm(runner, confirm_top, confirm_repeats, best_bits, best_time, stats)
    return ga.SearchResult(best_genome=best_bits, best_time=best_time, no_offload=no_offload,
                           evaluations_performed=runner.evaluations, cache_hits=runner.cache_hits,
                           history=history, genome_length=space.length)


def _confirm(runner, k: int, repeats: int, best_bits, best_time, stats):
    """Re-measure the k fastest feasible programs alone (see
    ``run_search_batched``).  Genomes that run the identical program (same
    GPU roots and plan: ``B200Evaluator.run_key``) are one candidate,
    represented by its first genome in the search's order, so measurement
    noise cannot pick between copies of one program; ties keep that order."""
    ranked = sorted((f.time, bits) for bits, f in runner.cache.items() if f.time is not None)
    solo = getattr(runner.evaluator, "measure_solo", None)
    run_key = getattr(runner.evaluator, "run_key", None)
    rows, seen = [], set()
    for t_search, bits in ranked:
        if len(rows) == k:
            break
        req = runner._request(bits, {"confirm": True})
        if run_key is not None:
            from .evaluator import payload_from_request

            key = run_key("", payload_from_request(req))
            if key in seen:
                continue
            seen.add(key)
        res = solo(req, repeats) if solo is not None else runner._measure_one(req)
        rows.append((bits, t_search, res.time_seconds))
    if stats is not None:
        stats["confirmed"] = [("".join(map(str, b)), t, s) for b, t, s in rows]
    ok = [(s, i, b) for i, (b, _, s) in enumerate(rows) if s is not None]
    if not ok:
        return best_bits, best_time
    s, _, b = min(ok)
    return b, s


def exhaustive_search_batched(model, verdicts, evaluator, cap: int = 14, backend: str = "c_openacc",
                              on_evaluation=None):
    """``exhaustive_search`` (src/ga.py:292-321): all 2^a genomes in one batch."""
    ga = _ga()
    from gpuoffload.patterns import PatternError, build_genome_space

    space = build_genome_space(model, verdicts)
    if space.is_empty:
        raise PatternError("no offloadable loops; nothing to enumerate")
    if space.length > cap:
        raise ga.ExhaustiveCapError(f"genome length {space.length} exceeds the exhaustive cap of {cap}")
    runner = _BatchRunner(model, space, evaluator, backend, on_evaluation)
    fits = runner.evaluate_population(list(space.all_genomes()), {"generation": 0})
    history = (ga._generation_stats(0, fits, runner.evaluations),)
    best_bits, best_time, no_offload = ga._best_of_cache(runner.cache, space.length)
    return ga.SearchResult(best_genome=best_bits, best_time=best_time, no_offload=no_offload,
                           evaluations_performed=runner.evaluations, cache_hits=runner.cache_hits,
                           history=history, genome_length=space.length)


def _predicted_cost(request) -> float:
    try:
        from gpuoffload.evaluators import CostModelParams, cost_model_time

        r = cost_model_time(request, CostModelParams())
        return r.time_seconds if r.time_seconds is not None else 0.0
    except ImportError:
        return 0.0


def lpt_assignment(costs: list[float], workers: int) -> list[int]:
    """Longest-processing-time-first: worker index per item (deterministic:
    ties by item order, then lowest worker index)."""
    order = sorted(range(len(costs)), key=lambda i: (-costs[i], i))
    load = [0.0] * workers
    owner = [0] * len(costs)
    for i in order:
        w = min(range(workers), key=lambda k: (load[k], k))
        owner[i] = w
        load[w] += max(costs[i], 1e-12)
    return owner


class ShardedEvaluator:
    """Evaluator protocol over a process group: ``measure_batch`` shards the
    batch across ranks (one B200 each) and all-gathers the results."""

    def __init__(self, inner, group=None):
        import torch.distributed as dist

        self.inner = inner
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.evaluator_id = getattr(inner, "evaluator_id", "sharded")
        self.concurrency_safe = True
        self.needs_code = getattr(inner, "needs_code", True)
        self.parallel_width = self.world * max(1, int(getattr(inner, "parallel_width", 1)))
        self._runs: dict = {}  # run key -> gathered (time, validity, evaluator, diagnostics)

    def measure(self, request):
        return self.measure_batch([request])[0]

    def _run_keys(self, requests) -> list | None:
        """Program-level dedupe keys (B200Evaluator.run_key) when the inner
        evaluator dedupes: identical programs are measured once across ALL
        ranks, and the results are shared through the gathered cache."""
        if not getattr(self.inner, "dedupe", False) or not hasattr(self.inner, "run_key"):
            return None
        from .evaluator import payload_from_request
        from .ir import document_digest

        return [self.inner.run_key(document_digest(self.inner._doc(r.model)), payload_from_request(r))
                for r in requests]

    def measure_batch(self, requests) -> list:
        keys = self._run_keys(requests)
        if keys is None:
            todo = list(range(len(requests)))
        else:
            firsts: dict = {}
            for i, k in enumerate(keys):
                if k not in self._runs and k not in firsts:
                    firsts[k] = i
            todo = sorted(firsts.values())
        owner = lpt_assignment([_predicted_cost(requests[i]) for i in todo], self.world)
        mine = [i for i, o in zip(todo, owner) if o == self.rank]
        inner_batch = getattr(self.inner, "measure_batch", None)
        reqs = [requests[i] for i in mine]
        res = inner_batch(reqs) if inner_batch else [self.inner.measure(r) for r in reqs]
        local = [(i, r.time_seconds, r.validity, r.evaluator_id, r.diagnostics) for i, r in zip(mine, res)]
        gathered: list = [None] * self.world
        self.dist.all_gather_object(gathered, local, group=self.group)
        cls = _result_cls()
        out: list = [None] * len(requests)
        for part in gathered:
            for i, t, validity, eid, diag in part:
                out[i] = cls(t, validity, eid, diag)
                if keys is not None:
                    self._runs[keys[i]] = (t, validity, eid, diag)
        if keys is not None:
            for i, k in enumerate(keys):
                if out[i] is None:
                    out[i] = cls(*self._runs[k])
        return out
