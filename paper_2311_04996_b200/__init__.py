"""B200-native batched WFST beam-search decoding for CTC models.

Drop-in for the decode path of the reference package ``ctcwfst``
(pkg/src/ctcwfst/__init__.py:10-53): graph load, batched offline decode,
streaming decode over per-utterance channels and word boosting. The frame
loop runs as hand-written sm_100a CUDA kernels (csrc/) behind a C-ABI
(include/ctcwfst_b200.h); there is no CPU fallback.
"""

from .boosting import BoostTable, attach_boost, boost_costs, build_boost_fsa, load_boost_table
from .decoder import (DecodeFailure, DecoderConfig, DecodeState, FlatGraph, Hypothesis, Token, advance,
                      best_path, create_channel, decode_batch, decode_utterance, flatten, prune)
from .errors import BoostError, BoostParseError, CtcWfstError, DecodeError, FstParseError, GraphError, StreamError
from .kernels import KERNEL_NAME, compiled_available
from .graphio import load_graph, save_graph
from .lattice import Lattice, PhraseBoost, decode_lattices, nbest_lattices
from .streaming import BatcherConfig, Chunk, StreamPool
from .wfst import Arc, SymbolTable, Wfst, arc_sort, read_fst_text, read_symbols, write_fst_text, write_symbols

__version__ = "0.1.0"
