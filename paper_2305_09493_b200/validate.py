"""Validator API (reference ``spirvkit/validate.py``) on the CUDA batch kernel.

``validate_module`` keeps the reference signature and diagnostics contract
(validate.py:45-94, 223-234, 299-301); the checks themselves run in
``skg_validate`` (csrc/skg_validate.cu), which emits the diagnostics_text
lines parsed back into ``Diagnostic`` objects here.
"""

from __future__ import annotations

from dataclasses import dataclass

from . import _native


@dataclass(frozen=True)
class Diagnostic:
    severity: str
    code: str
    location: int | None
    message: str

    def __str__(self):
        where = "module" if self.location is None else str(self.location)
        return f"{self.severity} {self.code} {where} {self.message}"


def _parse(text: str):
    out = []
    for line in text.split("\n")[:-1]:
        sev, code, where, msg = line.split(" ", 3)
        out.append(Diagnostic(sev, code, None if where == "module" else int(where), msg))
    return out


def _as_bytes(module):
    if isinstance(module, (bytes, bytearray)):
        return bytes(module)
    # a builder ModuleScope (serialized as the reference does, validate.py:64-70);
    # int also has a to_bytes method but is not a module
    to_bytes = None if isinstance(module, int) else getattr(module, "to_bytes", None)
    if callable(to_bytes):
        return to_bytes()
    raise TypeError("validate_module expects bytes or a ModuleScope")


def validate_batch(modules, spec=None):
    """list[bytes] -> list[list[Diagnostic] | Exception]."""
    batch = modules if isinstance(modules, _native.DeviceBatch) else \
        _native.DeviceBatch.from_modules([_as_bytes(m) for m in modules])
    return [r if isinstance(r, BaseException) else _parse(r.decode("utf-8"))
            for r in _native.run_texts("validate", batch, 0, spec)]


def validate_module(module, spec=None):
    out = validate_batch([_as_bytes(module)], spec)[0]
    if isinstance(out, BaseException):
        raise out
    return out


def check_capability_closure(module, spec=None):
    """validate.py:223-234: closure findings only (decode error -> CorruptStream)."""
    diags = validate_module(module, spec)
    if diags and diags[0].code in ("NotSpirv", "TruncatedStream", "CorruptStream"):
        return [Diagnostic("error", "CorruptStream", None, diags[0].message)]
    return [d for d in diags if d.code == "MissingCapability" and d.location is not None]


def diagnostics_text(diagnostics) -> str:
    return "\n".join(str(d) for d in diagnostics)
