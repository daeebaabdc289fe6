"""pytest plugin: run the REFERENCE's own test files with its hot-path names bound
to this package (tests/test_gpu_reference_suite.py loads it with -p).

The reference package (oracle/_ref/spirvkit, installed by __graft_entry__.build)
stays importable for what the tests use to build inputs -- the module builder,
the instruction factory, the grammar loaders, codegen -- while every function
on the codec hot path and the types / exceptions those
functions exchange with the tests are replaced, in the package namespace and in
its submodules, by the GPU-backed ones of paper_2305_09493_b200.
"""

import os
import sys

ROOT = os.environ["SKG_REPO_ROOT"]
sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))
sys.path.insert(0, ROOT)

import spirvkit as R  # noqa: E402  (the reference: builder / grammar / codegen for inputs)
from spirvkit import asm as R_asm, codec as R_codec, disasm as R_disasm, errors as R_errors  # noqa: E402
from spirvkit import cli as R_cli, grammar as R_grammar, validate as R_validate  # noqa: E402

import paper_2305_09493_b200 as G  # noqa: E402
from paper_2305_09493_b200 import asm as G_asm, codec as G_codec, disasm as G_disasm  # noqa: E402
from paper_2305_09493_b200 import cli as G_cli, errors as G_errors, grammar as G_grammar  # noqa: E402
from paper_2305_09493_b200 import validate as G_validate  # noqa: E402

BINDINGS = {
    R_codec: (G_codec, ["decode_module", "encode_header", "encode_instruction", "encode_string_literal",
                        "encode_context_dependent_literal", "encode_module", "ModuleHeader", "RawInstruction"]),
    R_disasm: (G_disasm, ["Disassembler", "DisassemblerOptions", "disassemble_module", "format_instruction",
                          "RenderContext"]),
    R_validate: (G_validate, ["validate_module", "check_capability_closure", "diagnostics_text", "Diagnostic"]),
    R_asm: (G_asm, ["Assembler", "assemble_module", "tokenize_line", "TextInstruction", "Token", "SymbolTable"]),
    R_grammar: (G_grammar, ["capability_dependency_graph", "DependencyReport"]),
    R_cli: (G_cli, ["run_cli", "build_parser"]),
}
ERRORS = ["SpirvKitError", "CodecError", "CorruptStreamError", "TruncatedStreamError", "NotSpirvError",
          "AssemblyError", "AsmDiagnostic", "StructureError", "SerializationError", "NotFoundError"]
BOUND = []
for mod, (src, names) in BINDINGS.items():
    for n in names:
        setattr(mod, n, getattr(src, n))
        if hasattr(R, n):
            setattr(R, n, getattr(src, n))
        BOUND.append(f"{mod.__name__}.{n}")
for n in ERRORS:
    setattr(R, n, getattr(G_errors, n))
    setattr(R_errors, n, getattr(G_errors, n))


def pytest_report_header(config):
    return [f"refsuite: reference spirvkit from {os.path.dirname(R.__file__)}; hot path bound to "
            f"{os.path.dirname(G.__file__)} ({len(BOUND)} names + {len(ERRORS)} exception classes)"]
