"""The reference's exception hierarchy (errors.py), for the errors this
package raises on the reference's paths: callers catching the reference's
classes by name keep working (a maintainer wiring the drop-in aliases
these to ``inspectour.errors``)."""


class PlanningError(Exception):
    """errors.py:4 - base class for the package's planning errors."""


class InfeasibleViewpointError(PlanningError):
    """errors.py:16 - a viewpoint lies in occupied space (graph.py:47-50)."""


class OccupiedEndpointError(PlanningError, ValueError):
    """errors.py:24 - a path query starts or ends on an occupied voxel
    (voxel.py:121-123).  Also a ValueError, as before."""


class InvalidTourError(PlanningError):
    """errors.py:28 - not a closed tour over the graph (graph.py:81-96)."""
