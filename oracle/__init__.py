"""TEST INFRASTRUCTURE ONLY — the CPU oracle (liboracle.so, built from
yo_oracle.c by oracle/Makefile) and, when it was built here, the reference
itself (oracle/_ref/librelsim_capi.so).  Both export the C-ABI of
include/yasps_b200.h (prefixes `yo_` / `yr_`), so the product's Engine drives
them unchanged when a test injects the library.  Only tests/, the driver's
smoke() and bench.py's CPU baseline / reference arm import this module; the
product package never does."""
from __future__ import annotations

from pathlib import Path

from paper_2605_23088_b200._lib import Library

HERE = Path(__file__).resolve().parent
_LIBS: dict[str, Library] = {}


def library() -> Library:
    """The oracle restatement of the reference's algorithm (yo_oracle.c)."""
    if "oracle" not in _LIBS:
        _LIBS["oracle"] = Library(HERE / "liboracle.so", "yo_")
    return _LIBS["oracle"]


def reference_library() -> Library:
    """The unmodified reference sources compiled here (oracle/ref_build.sh)."""
    if "ref" not in _LIBS:
        _LIBS["ref"] = Library(HERE / "_ref" / "librelsim_capi.so", "yr_")
    return _LIBS["ref"]


def reference_available() -> bool:
    return (HERE / "_ref" / "librelsim_capi.so").exists()


def for_backend(backend: str):
    """None (the product's default: the B200 library) for "gpu"."""
    if backend == "gpu":
        return None
    if backend == "oracle":
        return library()
    if backend == "reference":
        return reference_library()
    raise ValueError(backend)
