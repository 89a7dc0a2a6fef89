"""Language edges: real Python and Java source ->
the reference's language-neutral IR document.

The paper analyses C, Python and Java programs with one common flow
(PAPER.md:104,112,122-124); the reference only ships its C-like mini
language and a JSON IR document that "other languages feed ... without
linking against it" (src/irdoc.py:1-4), tagged ``python_like`` /
``java_like``.  These frontends accept the loop-nest subset of
each language that the mini language can express, lower it to mini-language
text, parse that with the reference's own parser (``parse_mini_source``,
src/minilang.py:520) and tag the resulting document with the source
language, so everything downstream -- screen, genome, transfer plan, GA,
block matching, and the B200 backend -- is unchanged.

Both raise :class:`FrontendError` (with a line number) for constructs
outside the subset instead of guessing their semantics.
"""

from __future__ import annotations


class FrontendError(ValueError):
    """The source uses a construct outside the supported subset."""

    def __init__(self, msg: str, line: int | None = None):
        super().__init__(f"line {line}: {msg}" if line else msg)
        self.line = line


def to_document(mini_source: str, language: str) -> dict:
    """Parse mini-language text with the reference parser and return its IR
    document tagged with ``language`` (validated by the reference loader)."""
    import json

    from gpuoffload.irdoc import load_ir_document, model_to_document
    from gpuoffload.minilang import parse_mini_source

    doc = model_to_document(parse_mini_source(mini_source))
    doc["language"] = language
    return model_to_document(load_ir_document(json.dumps(doc)))
