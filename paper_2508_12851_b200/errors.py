"""Exception types of the reference API (domain.py:32-37, cost.py:34-35).

When the reference package `moeplace` is importable the very same classes are
re-exported, so callers that catch `moeplace.DimensionMismatch` /
`InfeasibleError` / `UnplacedExpertError` keep working with the B200 path.
"""

from __future__ import annotations

import sys
from pathlib import Path

_REF_INSTALL = Path(__file__).resolve().parent.parent / "baseline" / "_ref"


def import_moeplace():
    """Import the reference package (installed copy under baseline/_ref if needed); None if absent."""
    try:
        import moeplace  # noqa: F401
        return moeplace
    except ImportError:
        pass
    if _REF_INSTALL.is_dir() and str(_REF_INSTALL) not in sys.path:
        sys.path.append(str(_REF_INSTALL))
        try:
            import moeplace  # noqa: F401
            return moeplace
        except ImportError:
            return None
    return None


_mp = import_moeplace()
if _mp is not None:
    from moeplace.domain import DimensionMismatch, InfeasibleError  # type: ignore
    from moeplace.cost import UnplacedExpertError  # type: ignore
else:  # same names and bases as the reference
    class DimensionMismatch(ValueError):
        """A placement's shape disagrees with the cluster or model geometry."""

    class InfeasibleError(RuntimeError):
        """The requested configuration cannot satisfy coverage within memory."""

    class UnplacedExpertError(RuntimeError):
        """An invocation targets a server that holds no copy of the expert."""

__all__ = ["DimensionMismatch", "InfeasibleError", "UnplacedExpertError", "import_moeplace"]
