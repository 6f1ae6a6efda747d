"""Exception types of the drop-in API.

The names and the base-class relations are those of the reference package
(/root/reference/pkg/src/spreadsim/errors.py:1-57) so that callers catching
``spreadsim`` exceptions keep working.  Two additions: ``InvalidConfigError``
also derives from ``ValueError`` (the C ABI reports bad arguments with it),
and ``FlashSpreadNativeError`` signals a missing library / device or a CUDA
failure — the engine has no CPU fallback and fails loudly instead.
"""

from __future__ import annotations


class SpreadSimError(Exception):
    """Root of every error raised by this package."""


def _derive(name: str, base: type, doc: str) -> type:
    return type(name, (base,), {"__doc__": doc, "__module__": __name__})


GraphError = _derive("GraphError", SpreadSimError, "Invalid graph structure or graph file.")
IndexOutOfRangeError = _derive("IndexOutOfRangeError", GraphError, "Node id or offset outside its range.")
DuplicateEdgeError = _derive("DuplicateEdgeError", GraphError, "The same (src, dst) pair given twice.")
NegativeWeightError = _derive("NegativeWeightError", GraphError, "Edge weight below zero.")
SelfLoopError = _derive("SelfLoopError", GraphError, "Edge from a node to itself.")
EmptyGraphError = _derive("EmptyGraphError", GraphError, "Operation undefined on an edgeless graph.")
InfeasibleDegreeSequenceError = _derive(
    "InfeasibleDegreeSequenceError", GraphError, "No simple graph realises the requested degrees."
)
GraphFileError = _derive("GraphFileError", GraphError, "Malformed graph file.")
InvalidMomentsError = _derive("InvalidMomentsError", SpreadSimError, "Holding-time moments cannot be inverted.")
ReconfigureAfterStartError = _derive(
    "ReconfigureAfterStartError", SpreadSimError, "Storage format changed after the first step."
)
GridMismatchError = _derive("GridMismatchError", SpreadSimError, "Trajectories on different grids.")
DegenerateFitError = _derive("DegenerateFitError", SpreadSimError, "Regression input is degenerate.")


class InvalidConfigError(SpreadSimError, ValueError):
    """Bad configuration or argument (also a ValueError)."""


class FlashSpreadNativeError(SpreadSimError, RuntimeError):
    """The native library or CUDA device is missing, or a CUDA call failed."""
