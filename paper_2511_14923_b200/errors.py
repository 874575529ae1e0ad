"""Exception hierarchy, mirroring gbsemu/errors.py:8-29 (exit codes 2/3/4).

The C ABI returns the same numbers as status codes (include/mps_sampler.h);
:func:`raise_for_status` maps them back onto these classes.
"""


class GbsError(Exception):
    """Base class for all package errors (C-ABI status 1: CUDA runtime failure)."""

    exit_code = 1


class ValidationError(GbsError):
    """Bad user input: shapes, ranges, dtypes, missing sites (status 2)."""

    exit_code = 2


class ResourceGuardError(GbsError):
    """Refused for lack of a resource: no B200, out of HBM, over budget (status 3)."""

    exit_code = 3


class NumericalError(GbsError):
    """A computation produced values outside its certified range (status 4)."""

    exit_code = 4


_BY_STATUS = {1: GbsError, 2: ValidationError, 3: ResourceGuardError, 4: NumericalError}


def raise_for_status(status: int, message: str = "") -> None:
    if status == 0:
        return
    raise _BY_STATUS.get(int(status), GbsError)(message or f"native status {status}")
