"""Compile service behind the C ABI's ``b2o_app_load`` (include/b2o.h).

SURVEY.md §8(b) asks for ``app_load(model_json, app_spec_json) -> app`` at the
C boundary, so a consumer without Python bindings can measure patterns.  The
per-program compiler is this package's Python code (compiler.py: IR document
-> host module + sm_100a cubin), so ``b2o_app_load`` runs it as a build step
the way the reference's external harness runs its ``build_cmd``
(src/evaluators.py:189-204):

    python -m paper_2011_03602_b200.compile_cli DOC.json SPEC.json OUT_DIR

It compiles (or fetches from the module cache) the program, writes the
initial value of every variable as a raw little-endian file (the app spec's
inputs, zero elsewhere; appspec.initial_state), and a line-oriented manifest
the C side parses without a JSON library::

    host <path of app_host.so>
    cubin <path of app.cubin>
    loops <n_loops>
    var <id> <bytes> <path> <name>

Exit status 0 on success; 2 with the reason on stderr for a program the
compiler rejects (the caller reports compile_error) or a malformed request.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np


def main(argv: list[str]) -> int:
    if len(argv) != 3:
        print("usage: python -m paper_2011_03602_b200.compile_cli DOC.json SPEC.json OUT_DIR", file=sys.stderr)
        return 2
    from . import appspec
    from .compiler import CompileError, compile_program
    from .ir import Program

    try:
        doc = json.loads(Path(argv[0]).read_text())
        spec = json.loads(Path(argv[1]).read_text())
        prog = Program(doc)
        compiled = compile_program(doc, spec)
        state = appspec.initial_state(prog, spec)
    except (CompileError, ValueError, KeyError) as exc:
        print(f"compile_error: {exc}", file=sys.stderr)
        return 2
    out = Path(argv[2])
    out.mkdir(parents=True, exist_ok=True)
    lines = [f"host {compiled.host_so}", f"cubin {compiled.cubin}", f"loops {compiled.n_loops}"]
    for v in prog.vars:
        arr = np.ascontiguousarray(state[v.id])
        f = out / f"var{v.id}.bin"
        arr.tofile(f)
        lines.append(f"var {v.id} {arr.nbytes} {f} {v.name}")
    (out / "manifest.txt").write_text("\n".join(lines) + "\n")
    return 0


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
