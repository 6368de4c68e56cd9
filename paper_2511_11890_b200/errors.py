"""Exception hierarchy of the drop-in (errors.py:4-41 of the reference) and
its mapping from the C-ABI status codes of include/harpia_b200.h.

Class names and constructor signatures match the reference so callers that
``except BudgetTooSmallError as e: e.minimum_bytes`` keep working.
"""

from __future__ import annotations


class HarpiaError(Exception):
    """Root of every error the library raises (reference errors.py:4)."""


class ParameterError(HarpiaError):
    """Bad operator/tool parameter (errors.py:8); C status HB_EPARAM."""


class CorruptInputError(HarpiaError):
    """Volume bytes disagree with their declared geometry (errors.py:12)."""


class UnsupportedFormatError(HarpiaError):
    """dtype or layout outside the supported set (errors.py:16); HB_EUNSUPPORTED."""


class BudgetUnavailableError(HarpiaError):
    """The backend could not report free memory (errors.py:20); on B200 this is
    cudaMemGetInfo failing or no CUDA device; HB_EBUDGET_UNAVAILABLE."""


class BudgetTooSmallError(HarpiaError):
    """Budget cannot hold one padded chunk (errors.py:24-29); HB_EBUDGET_SMALL."""

    def __init__(self, message, minimum_bytes=None):
        super().__init__(message)
        self.minimum_bytes = minimum_bytes


class ChunkExecutionError(HarpiaError):
    """An operator (kernel) failed on a chunk (errors.py:32-37); HB_ECHUNK and
    HB_ECUDA both surface as this, carrying the failing chunk index."""

    def __init__(self, message, chunk_index):
        super().__init__(message)
        self.chunk_index = chunk_index


class JobCancelled(HarpiaError):
    """Cancelled at a chunk boundary; partial output is discarded (errors.py:40)."""


# C-ABI status codes (include/harpia_b200.h, enum hb_status)
HB_OK = 0
HB_EPARAM = 1
HB_EBUDGET_SMALL = 2
HB_EBUDGET_UNAVAILABLE = 3
HB_ECHUNK = 4
HB_ECANCELLED = 5
HB_ECUDA = 6
HB_EUNSUPPORTED = 7


def raise_for_status(code: int, message: str, *, failed_chunk: int = -1,
                     minimum_bytes: int = 0) -> None:
    """Translate a non-zero hb_status into the matching reference exception."""
    if code == HB_OK:
        return
    if code == HB_EPARAM:
        raise ParameterError(message)
    if code == HB_EBUDGET_SMALL:
        raise BudgetTooSmallError(message, minimum_bytes=int(minimum_bytes) or None)
    if code == HB_EBUDGET_UNAVAILABLE:
        raise BudgetUnavailableError(message)
    if code in (HB_ECHUNK, HB_ECUDA):
        raise ChunkExecutionError(message, chunk_index=int(failed_chunk))
    if code == HB_ECANCELLED:
        raise JobCancelled(message)
    if code == HB_EUNSUPPORTED:
        raise UnsupportedFormatError(message)
    raise HarpiaError(f"unknown status {code}: {message}")
