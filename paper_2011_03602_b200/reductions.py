"""Opt-in screen extension: reductions and private scalars on the GPU
(SURVEY.md §8 f4).

The reference screen rejects every loop whose subtree both reads and sets a
non-index scalar (``loop_carried_scalar``, src/screen.py:57-68; "reductions
land here").  Two such shapes are safe to offload with the right kernel:

* a **reduction** scalar ``s``: every statement of the subtree that touches
  ``s`` is ``s = s + e``, ``s = e + s`` or ``s = s - e`` with ``s`` not in
  ``e`` (the Himeno ``gosa = gosa + gs[idx]`` nest, the textbook
  ``gosa = gosa + ss * ss``).  The kernel accumulates per thread, combines
  with a warp-shuffle / shared-memory tree and finishes deterministically in
  the last CTA (compiler.py ``_reduction_epilogue``);
* a **private** scalar: every iteration writes it before reading it (the
  textbook Himeno ``s0``/``ss`` temporaries); each thread keeps its own copy
  and the thread of the sequentially last iteration stores the value the
  loop leaves behind (lastprivate, as for every scalar a kernel writes).

Turning this on changes the genome (more loops become genes), so it is OFF
for parity with the reference GA; enable it with
``screen_model_with_reductions`` for the GA's verdicts and ``"reductions":
true`` in the app spec for the compiler.  Float reductions are reassociated
(tree order instead of sequential), so their outputs differ from the
sequential CPU result by the sequential sum's own rounding error (~1e-4
relative for 4M fp32 terms): give them a matching ``rel_tol`` in the spec.
Integer reductions are exact.
"""

from __future__ import annotations

from .ir import Program, expr_vars


def reduction_stmt(st):
    """``(var, op, e)`` when ``st`` is ``s = s + e`` / ``s = e + s`` /
    ``s = s - e`` with ``s`` a scalar not occurring in ``e``, else None."""
    if st.kind != "assign" or st.target[0] != "var":
        return None
    s = st.target[1]
    v = st.value
    if v[0] != "bin" or v[1] not in "+-":
        return None
    a, b = v[2], v[3]
    if a == ("var", s) and s not in expr_vars(b):
        return s, v[1], b
    if v[1] == "+" and b == ("var", s) and s not in expr_vars(a):
        return s, "+", a
    return None


def carried_scalars(prog: Program, lid: int) -> set[int]:
    """Non-index scalars both read and set in the loop's subtree (the
    reference rule, src/screen.py:54-68)."""
    regions = set(prog.subtree_regions(lid))
    exempt = {prog.loops[x].index_var for x in prog.subtree_loops(lid)}
    reads, sets = set(), set()
    for o in prog.doc["occurrences"]:
        if o["region"] not in regions or prog.vars[o["var"]].is_array or o["var"] in exempt:
            continue
        if o["kind"] == "read":
            reads.add(o["var"])
        elif o["kind"] == "set":
            sets.add(o["var"])
    return reads & sets


def _first_touch(prog: Program, rid: int, s: int) -> str | None:
    """Walking one iteration's body in order: "write" when every path writes
    ``s`` before reading it, "read" when ``s`` may be read first, None when
    the region never touches it.  A nested loop that writes first may run
    zero times, so a later read of ``s`` in the same body counts as a read."""
    maybe_written = False
    for st in prog.regions[rid].statements:
        if st.kind == "loop":
            lo = prog.loops[st.loop]
            if s in expr_vars(lo.lower) or s in expr_vars(lo.upper) or lo.index_var == s:
                return "read"
            sub = _first_touch(prog, lo.body, s)
            if sub == "read":
                return "read"
            maybe_written = maybe_written or sub == "write"
            continue
        reads, writes = prog.stmt_access(st)
        if st.kind == "call" and (s in reads or s in writes):
            return "read"
        if s in reads:
            return "read"
        if s in writes:
            return "write"
    return "write" if maybe_written else None


def classify(prog: Program, lid: int) -> dict[int, str] | None:
    """``{scalar: "reduction" | "private"}`` for every carried scalar of loop
    ``lid``, or None when one of them is neither."""
    out: dict[int, str] = {}
    body = prog.loops[lid].body
    stmts = list(prog.walk(body))
    for s in carried_scalars(prog, lid):
        touching = []
        for st in stmts:
            if st.kind == "loop":
                lo = prog.loops[st.loop]
                if s in expr_vars(lo.lower) + expr_vars(lo.upper):
                    touching.append(None)
                continue
            r, w = prog.stmt_access(st)
            if s in r or s in w:
                touching.append(st)
        red = [reduction_stmt(st) if st is not None else None for st in touching]
        ops = {x[1] for x in red if x is not None and x[0] == s}
        if touching and all(x is not None and x[0] == s for x in red) and len(ops) == 1:
            out[s] = "reduction:" + ops.pop()
        elif _first_touch(prog, body, s) == "write":
            out[s] = "private"
        else:
            return None
    return out


def screen_model_with_reductions(model):
    """The reference's verdicts (``screen_model``, src/screen.py:82-84) with
    ``loop_carried_scalar`` rejections lifted when every carried scalar is a
    reduction or private and the rest of the reference rules pass.  Returns
    the reference's own ``ParallelizabilityVerdict`` objects, so
    ``build_genome_space`` / ``run_search`` take it unchanged."""
    from gpuoffload.screen import REASON_CARRIED_SCALAR, REASON_OK, ParallelizabilityVerdict, screen_model

    from .compiler import parallelizable
    from .ir import document_of

    base = screen_model(model)
    prog = Program(document_of(model))
    out = []
    for v in base:
        if v.reason == REASON_CARRIED_SCALAR and classify(prog, v.loop_id) is not None \
                and parallelizable(prog, v.loop_id, extended=True):
            out.append(ParallelizabilityVerdict(v.loop_id, True, REASON_OK))
        else:
            out.append(v)
    return out
