"""B200-native memory-restricted X-drop seed extension (arXiv 2304.08662 path).

The product is the C-ABI shared library (include/xdrop_b200.h) built from
csrc/ for sm_100a; this package only binds it (capi), mirrors the reference
xband API on top of it (xband), and generates the BASELINE configs (synth).
"""
from . import capi, synth, xband  # noqa: F401
from .xband import (BandBuffers, BandExceededError, DanglingReference, DevicePool, Dir,  # noqa: F401
                    ExtensionResult, ExtensionTask, InputError, OutOfRange, ScoringScheme,
                    SeedAlignment, SeedOutOfBounds, SeqView, Sequence, SequenceStore, SubMatrix,
                    UnknownSymbol, extend_batch, extend_seed, extend_tasks, extend_units, full,
                    gcups, make_view, parse_submatrix, sim, split_lr, estimate_cost, sweep_band,
                    xdrop_extend, parse_fasta, parse_seeds, parse_overlaps, FastaRecords,
                    MissingHeader, EmptyRecord, InvalidSymbol, MalformedLine, NegativeIndex,
                    BadHeader, IndexOutOfDeclaredShape)

__all__ = ["capi", "synth", "xband"]
