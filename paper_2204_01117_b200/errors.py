"""Exception types of the reference's step path, same names and bases:
ProjectionError (solver.py:113-116), SingularSystemError (linalg.py:23-24),
ScenarioError (scenario.py:40-46), MeshError / ClassificationError
(geometry.py:26-31)."""
from __future__ import annotations


class ProjectionError(RuntimeError):
    def __init__(self, report):
        super().__init__(f"pressure solve did not converge: {report}")
        self.report = report


class SingularSystemError(ValueError):
    """Pressure system has the all-constants nullspace (no outlet anywhere)."""


class ScenarioError(ValueError):
    """Carries the complete list of validation problems, not just the first."""

    def __init__(self, errors: list[str]):
        super().__init__("invalid scenario:\n  - " + "\n  - ".join(errors))
        self.errors = errors


class MeshError(ValueError):
    """Malformed mesh (open surface, bad indices, empty)."""


class ClassificationError(RuntimeError):
    """A point could not be classified inside/outside a mesh."""


class NativeError(RuntimeError):
    """CUDA / extension failure."""
