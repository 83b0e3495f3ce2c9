"""Exception types of the decode path.

Same class names and hierarchy as the reference (pkg/src/ctcwfst/errors.py:4-65)
so callers' ``except`` clauses keep working after the switch. Only the types
the decode path (graph load, decoding, boosting, streaming) raises are here.
"""


class CtcWfstError(Exception):
    """Root of every error raised by the decoder package."""


class _LineError(CtcWfstError):
    """An error that may point at a 1-based input line."""

    def __init__(self, message, lineno=None):
        self.lineno = lineno
        super().__init__(message if lineno is None else f"line {lineno}: {message}")


class FstParseError(_LineError):
    """Malformed AT&T FST text or symbol table (wfst.read_fst_text / read_symbols)."""


class SymbolTableError(CtcWfstError):
    """Inconsistent symbol <-> id mapping."""


class GraphError(CtcWfstError):
    """Decoding graph unusable (e.g. empty)."""


class DecodeError(CtcWfstError):
    """Beam search failure: epsilon iteration cap, dead beam, bad frame width,
    or misuse (boost after frames, best path before any frame)."""


class BoostError(CtcWfstError):
    """Invalid word-boost table or misuse."""


class BoostParseError(_LineError, BoostError):
    """Malformed boost table text."""


class StreamError(CtcWfstError):
    """Streaming pool misuse (capacity, state machine, unknown stream)."""
