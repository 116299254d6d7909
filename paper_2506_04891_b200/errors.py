"""Exception types of the drop-in API.

Same three names and meanings as the reference (`pkg/src/layersim/errors.py:4-13`),
so callers that catch the reference's exceptions keep working. The C-ABI status codes
map onto them in `_native.py` (1 -> ValueError, 2 -> PlanMismatchError,
3 -> CapacityError, 4 -> RuntimeError).
"""


class CapacityError(Exception):
    """The request does not fit the configured element budget or device memory."""


class PlanMismatchError(Exception):
    """A plan was built for a different circuit / qubit count / variant set."""


class CorrectnessError(Exception):
    """Two executions that must agree (e.g. planned vs default) disagree."""
