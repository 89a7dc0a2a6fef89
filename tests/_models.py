"""Seeded random loop forests for GA tests, built with the reference's
ModelBuilder (the same shape of generator the reference's own tests use,
tests/conftest.py:59-152 of the reference, written independently here)."""

from gpuoffload.build import ModelBuilder
from gpuoffload.model import BinOp, Num, VarRef


def random_model(rng, max_depth=3, n_arrays=3):
    b = ModelBuilder()
    idx = [b.declare(f"i{d}", "int") for d in range(max_depth)]
    arrs = [b.declare(f"a{k}", "float", is_array=True, length=rng.choice([16, 32, 64])) for k in range(n_arrays)]
    sc = b.declare("s", "float", initializer=Num(0.0, True))
    names = {v: b.var_name(v) for v in idx + arrs + [sc]}

    def nest(region, depth):
        _, body = b.for_loop(region, names[idx[depth]], Num(0), Num(rng.choice([2, 4, 8, 16])),
                             cpu_cost_per_iter=rng.choice([0.5, 1.0, 2.0]),
                             gpu_cost_per_iter=rng.choice([0.05, 0.2, 1.5]))
        dst, src = rng.choice(arrs), rng.choice(arrs)
        if rng.random() < 0.25:
            b.assign(body, b.ref(names[sc]), b.at(names[src], VarRef(idx[depth])))
        else:
            b.assign(body, b.at(names[dst], VarRef(idx[depth])),
                     BinOp("+", b.at(names[src], VarRef(idx[depth])), Num(1.0, True)))
        if depth + 1 < max_depth and rng.random() < 0.6:
            nest(body, depth + 1)

    for _ in range(rng.randint(2, 4)):
        nest(b.root, 0)
    m = b.finish()
    return m if len(m.loops) >= 3 else random_model(rng, max_depth, n_arrays)
