"""One-off large differential fuzz (not part of the committed suite).

  build  (here, with the reference importable):
      PYTHONPATH=/root/reference/pkg/src python tools/fuzz_big.py build N [BASE]
      -> tools/_bigfuzz.json: N general + N shape programs with the
         reference's plans for up to 64 genomes each (general seeds from
         BASE, shape seeds from BASE + 1000; default 5000)
  run    (on a B200):   python tools/fuzz_big.py run [fp32|fp64]
      -> every genome vs the C oracle, bit for bit; prints a summary line
"""

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
OUT = ROOT / "tools" / "_bigfuzz.json"


def build(n: int, base: int = 5000) -> None:
    sys.path.insert(0, str(ROOT / "tests" / "golden"))
    sys.argv = ["make_golden.py"]
    import make_golden as mg
    from gpuoffload.minilang import parse_mini_source
    from gpuoffload.screen import screen_model

    import _fuzz
    import _fuzz_shapes
    from paper_2011_03602_b200.reductions import screen_model_with_reductions

    rec = {}
    for seed in range(base, base + n):
        m = parse_mini_source(_fuzz.program(seed))
        rec[f"g{seed}"] = mg.app_record(f"g{seed}", m, _fuzz.spec(seed), all_genomes_cap=64)
    for seed in range(base + 1000, base + 1000 + n):
        m = parse_mini_source(_fuzz_shapes.program(seed))
        sp = _fuzz_shapes.spec(seed)
        scr = screen_model_with_reductions if sp.get("reductions") else screen_model
        rec[f"s{seed}"] = mg.app_record(f"s{seed}", m, sp, all_genomes_cap=64, screen=scr)
    OUT.write_text(json.dumps(rec))
    print(len(rec), "programs,", sum(len(r["patterns"]) for r in rec.values()), "genomes")


def run(precision: str = "fp32") -> None:
    import numpy as np

    from oracle.cgen import CProgram
    from paper_2011_03602_b200 import appspec
    from paper_2011_03602_b200.evaluator import B200Evaluator
    from paper_2011_03602_b200.ir import Program

    rec = json.loads(OUT.read_text())
    bad, n = [], 0
    for name, r in rec.items():
        r["spec"]["precision"] = precision
        prog = Program(r["doc"])
        want = CProgram(r["doc"], precision).run(appspec.initial_state(prog, r["spec"]))
        ev = B200Evaluator(r["spec"], devices=[0], timeout_seconds=60)
        try:
            app = ev.app_for(r["doc"])
        except Exception as exc:  # noqa: BLE001
            bad.append((name, "build", str(exc)[:200]))
            continue
        outs = [prog.var_by_name[o].id for o in r["spec"]["outputs"]]
        for g in sorted(r["patterns"]):
            n += 1
            res = ev.measure_payloads(r["doc"], [r["patterns"][g]])[0]
            if res["validity"] != "valid":
                bad.append((name, g, res["diag"][:200]))
                continue
            for vid in outs:
                got = app.read(vid, worker=res["worker"])
                if got.tobytes() != np.asarray(want[vid], dtype=got.dtype).tobytes():
                    bad.append((name, g, prog.vars[vid].name))
                    break
        ev.close()
    print(json.dumps({"precision": precision, "programs": len(rec), "genomes": n, "failures": len(bad),
                      "first": bad[:10]}))


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build(int(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 5000)
    else:
        run(sys.argv[2] if len(sys.argv) > 2 else "fp32")
