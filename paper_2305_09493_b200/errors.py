"""Exception classes of the codec path.

Names, bases and message formats are the reference contract
(``spirvkit/errors.py:4-94``): callers catch these by class, and the GPU path
reproduces ``str(exc)`` byte for byte.  Device kernels report a per-module
status code (see ``STATUS_*`` in :mod:`._native`) plus the message text; the
host shim maps the code back to one of these classes.
"""


class SpirvKitError(Exception):
    pass


class GrammarError(SpirvKitError):
    pass


class GrammarParseError(GrammarError):
    def __init__(self, message, line=None, column=None):
        super().__init__(message)
        self.line, self.column = line, column


class GrammarSchemaError(GrammarError):
    pass


class NotFoundError(GrammarError, KeyError):
    # KeyError.__str__ would repr-quote the message; keep it plain.
    __str__ = Exception.__str__


class CodecError(SpirvKitError):
    pass


class NotSpirvError(CodecError):
    pass


class TruncatedStreamError(CodecError):
    pass


class CorruptStreamError(CodecError):
    pass


class GenerationError(SpirvKitError):
    pass


class ScopeError(SpirvKitError):
    pass


class SsaError(SpirvKitError):
    pass


class StructureError(SpirvKitError):
    pass


class SerializationError(SpirvKitError):
    pass


class IdExhaustedError(SpirvKitError):
    pass


class AsmDiagnostic:
    """A 1-based (line, column) assembler message."""

    __slots__ = ("line", "column", "message")

    def __init__(self, line, column, message):
        self.line, self.column, self.message = line, column, message

    def __str__(self):
        return f"{self.line}:{self.column}: {self.message}"

    def __repr__(self):
        return f"AsmDiagnostic({self.line}, {self.column}, {self.message!r})"

    def __eq__(self, other):
        return (isinstance(other, AsmDiagnostic)
                and (self.line, self.column, self.message)
                == (other.line, other.column, other.message))


class AssemblyError(SpirvKitError):
    """All diagnostics of one failed assembly, one ``line:col: msg`` per line."""

    def __init__(self, diagnostics):
        self.diagnostics = list(diagnostics)
        body = "\n".join(map(str, self.diagnostics))
        super().__init__(f"{len(self.diagnostics)} error(s):\n{body}")
