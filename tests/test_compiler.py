"""The compiler's analyses against the reference: the screen restatement must
reproduce the reference's verdicts (tests/golden/*.json, produced by
src/screen.py), kernel chains follow the screen, generated code is
deterministic, and the device-side integer division is exact."""

import json
import random

import pytest

from conftest import SMALL_APPS, golden
from paper_2011_03602_b200.compiler import (affine, compile_program, generate_sources, parallelizable,
                                            plan_nest, stencil_offset)
from paper_2011_03602_b200.ir import Program

ALL = SMALL_APPS + ["himeno_M", "himeno_L", "matmul_1024", "nasmg_258", "himeno_xs_noread"]


@pytest.mark.parametrize("name", ALL)
def test_screen_restatement_matches_reference(name):
    g = golden(name)
    prog = Program(g["doc"])
    for v in g["verdicts"]:
        assert parallelizable(prog, v["loop"]) == (v["reason"] == "ok"), (name, v)


def test_chains_follow_the_screen():
    prog = Program(golden("himeno_M")["doc"])
    assert plan_nest(prog, 1).chain == [1, 2, 3]      # Jacobi i-root: 3-D grid
    assert plan_nest(prog, 3).chain == [3]            # k-root: 1-D, i/j on the host
    assert plan_nest(prog, 0).chain == []             # n loop (carried gosa): sequential kernel
    mm = Program(golden("matmul_1024")["doc"])
    assert plan_nest(mm, 0).chain == [0, 1]           # k stays in-thread (non-affine write for k)
    assert plan_nest(mm, 1).chain == [1]


def test_kernel_shapes():
    prog = Program(golden("himeno_M")["doc"])
    jac, cpy = plan_nest(prog, 1), plan_nest(prog, 7)
    assert jac.shape == "flat" and jac.ppt == 2
    assert cpy.shape == "flat" and cpy.ppt == 4
    sten = plan_nest(prog, 1, enable_stencil=True)
    assert sten.shape == "stencil" and set(sten.staged) == {prog.var_by_name["p"].id}
    assert len(sten.streams) == 12


def test_affine_and_offsets():
    prog = Program(golden("himeno_M")["doc"])
    iv = [prog.loops[x].index_var for x in (1, 2, 3)]
    refs = []
    for st in prog.walk(prog.loops[3].body):
        def walk(e):
            if e[0] == "arr":
                refs.append(e)
                walk(e[2])
            elif e[0] == "bin":
                walk(e[2]); walk(e[3])
        walk(st.value)
    p = prog.var_by_name["p"].id
    offs = {stencil_offset(r[2], iv, 129 * 257, 257) for r in refs if r[1] == p}
    assert len(offs) == 19 and (0, 0, 0) in offs and (1, 1, 0) in offs and (-1, 0, -1) in offs
    assert affine(("bin", "/", ("num", 4, False), ("var", iv[0])), set(iv)) is None


def test_generation_is_deterministic():
    g = golden("nasmg_18")
    assert generate_sources(g["doc"], g["spec"]) == generate_sources(json.loads(json.dumps(g["doc"])), g["spec"])


def test_compile_builds_host_module_and_cubin():
    g = golden("four_loops")
    c = compile_program(g["doc"], g["spec"])
    assert c.host_so.exists() and c.cubin.exists()
    assert c.cubin.read_bytes()[:4] == b"\x7fELF"


def _fastdiv(n, d):
    s = 0
    while s < 32 and (1 << s) < d:
        s += 1
    mul = (((1 << 32) * ((1 << s) - d)) // d + 1) & 0xFFFFFFFF
    hi = (n * mul) >> 32
    return (hi + n) >> s


def test_fastdiv_exact():
    rng = random.Random(5)
    ds = [1, 2, 3, 7, 127, 255, 257, 4096, 65535, 2**31 - 1, 2**31, 2**32 - 1] + \
         [rng.randrange(1, 2**32) for _ in range(200)]
    ns = [0, 1, 2**31 - 1, 2**31, 2**32 - 1] + [rng.randrange(0, 2**32) for _ in range(200)]
    for d in ds:
        for n in ns:
            assert _fastdiv(n, d) == n // d, (n, d)


def _c_int(expr: str, tid: int) -> int:
    """Evaluate a generated non-negative C integer index expression."""
    py = expr.replace("threadIdx.x", str(tid)).replace("/", "//")
    return eval(py, {})  # noqa: S307 -- generated arithmetic on literals only


@pytest.mark.parametrize("opts", [{}, {"ktile_swz": False}])
def test_ktile_staging_covers_each_tile_element_once(opts):
    """The k-tile kernel's shared-memory staging map (matmul 1024, i-root):
    over all threads and stage slots every (k, row) element of each operand
    tile is stored exactly once; with the default swizzle every warp's
    transposed stores of the k-contiguous operand hit 32 distinct banks."""
    import re

    g = golden("matmul_1024")
    dev = generate_sources(g["doc"], dict(g["spec"], **opts))[1]
    body = dev[dev.find("b2o_k0("):]
    body = body[:body.find("__syncthreads();")]  # the prologue stores
    decl = dict((int(t), (int(bk), int(ext))) for t, bk, ext in
                re.findall(r"__shared__ __align__\(16\) float s(\d+)_\[(\d+)\]\[(\d+)\];", dev))
    stores = re.findall(r"\n  s(\d+)_\[(.+?)\]\[(.+?)\] = p\d+_(\d+);", body)
    assert stores and decl
    nthr = 256
    for t, (bk, pitch) in decl.items():
        mine = [(kk, oo) for tt, kk, oo, _ in stores if int(tt) == t]
        seen = {}
        for kk, oo in mine:
            for tid in range(nthr):
                key = (_c_int(kk, tid), _c_int(oo, tid))
                seen[key] = seen.get(key, 0) + 1
        ext = pitch - 4
        assert set(seen) == {(k, o) for k in range(bk) for o in range(ext)}, t
        assert set(seen.values()) == {1}, t
        if not opts and t == 0:  # A(i, k): k has unit stride -> transposed stores
            for kk, oo in mine:
                for w in range(nthr // 32):
                    banks = {(_c_int(kk, tid) * pitch + _c_int(oo, tid)) % 32 for tid in range(32 * w, 32 * w + 32)}
                    assert len(banks) == 32, (kk, oo, w, len(banks))


def test_ktile_shape_that_cannot_stage_is_rejected():
    """A k-tile edge whose staging does not divide evenly over the threads
    (60 x 60 tiles: 225 threads) would leave operands unstaged; the compiler
    refuses it instead of producing wrong sums."""
    import pytest as _pt

    from paper_2011_03602_b200.compiler import CompileError, generate_sources

    g = golden("matmul_48")
    with _pt.raises(CompileError, match="k-tile shape"):
        generate_sources(g["doc"], dict(g["spec"], ktile_tile=60))
    generate_sources(g["doc"], dict(g["spec"], ktile_tile=32))  # supported shapes still build
