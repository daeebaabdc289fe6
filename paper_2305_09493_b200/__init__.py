"""B200-native SPIR-V codec path (disassemble / assemble / validate / decode) behind the
``spirvkit`` (arXiv 2305.09493 reference) API.  See DESIGN.md."""

from .asm import (Assembler, SymbolTable, TextInstruction, Token, assemble_batch, assemble_module,
                  tokenize_line, tokenize_lines)
from .codec import (ModuleHeader, RawInstruction, TypedFloat, TypedInt, decode_module,
                    encode_context_dependent_literal, encode_context_dependent_literals, encode_header,
                    encode_instruction, encode_module, encode_modules, encode_string_literal,
                    encode_string_literals, serialize_modules)
from .disasm import (Disassembler, DisassemblerOptions, RenderContext, disassemble_batch,
                     disassemble_module, disassemble_validate_batch, format_instruction)
from .errors import (AsmDiagnostic, AssemblyError, CodecError, CorruptStreamError,
                     GenerationError, GrammarError, GrammarParseError, GrammarSchemaError,
                     IdExhaustedError, NotFoundError, NotSpirvError, ScopeError,
                     SerializationError, SpirvKitError, SsaError, StructureError,
                     TruncatedStreamError)
from .grammar import (DependencyReport, EnumerantDef, ExtInstGrammar, GrammarSpec, InstructionDef,
                      OperandKindDef, OperandSlot, capability_dependency_graph, load_core_grammar,
                      load_extended_grammar, load_pinned, load_pinned_extended, transitive_capabilities)
from .validate import (Diagnostic, check_capability_closure, diagnostics_text, validate_batch,
                       validate_module)

__version__ = "0.1.0"
