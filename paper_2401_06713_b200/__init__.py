"""B200-native Picasso conflict-graph builder.

The hot path of arXiv 2401.06713 (Picasso) — per-iteration conflict-graph construction
(palettecolor.conflict.build, /root/reference/pkg/src/palettecolor/conflict.py:89-167) — as
hand-written sm_100a CUDA behind a C ABI (include/picasso_b200.h), with the host side of the
reference's API around it (palette assignment, list coloring, residue iteration) so a whole
Picasso run produces the reference's coloring.

Drop-in use with the reference package::

    import palettecolor, paper_2401_06713_b200 as b200
    b200.install_into(palettecolor)      # palettecolor.conflict.build -> CUDA builder
"""

from __future__ import annotations

from .conflict import ConflictGraph, build, build_reference, lists_intersect
from .driver import (
    UNCOLORED,
    ColoringResult,
    ColorLists,
    IterationPlan,
    IterationRecord,
    PaletteParams,
    assign_random_lists,
    color_unconflicted,
    plan_iteration,
    run,
)
from .errors import (
    DeviceError,
    EdgeBudgetExceededError,
    IterationLimitError,
    PaletteColorError,
)
from .graph import EdgeOracleView, ExplicitGraph, graph_view, iter_pair_blocks, pauli_view
from .list_coloring import (
    ConflictColoringOutcome,
    color_conflict_graph,
    color_dynamic,
    color_static,
)
from .pauli import (
    EncodedPauli,
    PauliSet,
    anticommutes_chars,
    anticommutes_fast,
    anticommutes_oracle,
    complement_edge,
    decode,
    encode,
    parse_pauli_text,
    pauli_file_text,
    random_pauli_strings,
)

__version__ = "0.1.0"


def install_into(reference_module) -> None:
    """Route ``reference_module.conflict.build`` (and the package-level ``build``) to the
    CUDA builder for Pauli views.  Explicit-graph views keep the reference's own builder:
    they are a different oracle mode outside this builder's scope, not a fallback."""
    conflict_mod = reference_module.conflict
    original = getattr(conflict_mod, "_reference_build", conflict_mod.build)

    def routed(view, lists, **kw):
        if view.mode == "implicit-complement":
            return build(view, lists, **kw)
        return original(view, lists, **kw)

    conflict_mod._reference_build = original
    conflict_mod.build = routed
    reference_module.build = routed
