/* libskgpu -- B200 (sm_100a) batch SPIR-V codec: the C-ABI drop-in boundary.
 *
 * The reference (spirvkit 0.1.0) is pure Python and has no FFI layer; its hot
 * path is the Python API listed in SURVEY.md 8(b).  Each entry point below
 * replaces the loop body of one of those functions for a whole batch of
 * modules at once; paper_2305_09493_b200/_native.py binds them with ctypes and
 * keeps the reference's Python signatures on top.
 *
 * Conventions
 *  - All data pointers are DEVICE pointers (cudaMalloc / torch CUDA tensors),
 *    stream-ordered on `stream` (a cudaStream_t, or NULL for the legacy
 *    stream).  Nothing is synchronised inside the library.
 *  - A batch is a byte arena `data` with per-module byte offset/length arrays
 *    (int64).  Module starts SHOULD be 16-byte aligned (vectorised loads);
 *    unaligned starts are accepted and loaded bytewise.
 *  - Content errors (what the reference raises or reports) never fail a call:
 *    they become per-module status codes (SKG_ST_*) plus an error record with
 *    the exact str(exc) text.  Return values report API misuse / CUDA errors.
 *  - Thread-safe for distinct workspaces; tables are immutable after create.
 */
#ifndef SKGPU_H
#define SKGPU_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* per-module status = exception class the reference raises/reports */
enum {
  SKG_ST_OK = 0,
  SKG_ST_TRUNCATED = 1,    /* TruncatedStreamError */
  SKG_ST_NOTSPIRV = 2,     /* NotSpirvError */
  SKG_ST_CORRUPT = 3,      /* CorruptStreamError */
  SKG_ST_CODEC = 4,        /* CodecError */
  SKG_ST_UNICODE = 5,      /* UnicodeDecodeError */
  SKG_ST_KEY = 6,          /* KeyError */
  SKG_ST_VALUE = 7,        /* ValueError */
  SKG_ST_OVERFLOW = 8,     /* OverflowError (struct.pack of a float literal) */
  SKG_ST_ASSEMBLY = 9,     /* AssemblyError (message = all diagnostics) */
  SKG_ST_STRUCTURE = 10,   /* StructureError */
  SKG_ST_SERIALIZATION = 11, /* SerializationError */
  SKG_ST_INTERNAL = 99     /* scratch/capacity problem: rerun with more workspace */
};

/* disassembler option bits (DisassemblerOptions, disasm.py:46-54; strict :103) */
enum {
  SKG_OPT_HIGHLIGHT = 1, SKG_OPT_INLINE_NAMES = 2, SKG_OPT_NO_INDENT = 4,
  SKG_OPT_GROUP = 8, SKG_OPT_NO_HEADER = 16, SKG_OPT_STRICT = 32
};

/* one error record (256 bytes): module index, status, detail words, message */
typedef struct skg_error {
  int32_t module;
  int32_t status;
  uint32_t a, b, c, d;   /* UnicodeDecodeError: start, end, reason(1 start,2 cont,3 end), byte */
  int32_t len;           /* message length (may exceed the stored 227 bytes) */
  char msg[228];
} skg_error;

typedef struct skg_tables skg_tables;

/* Upload a grammar table blob (paper_2305_09493_b200/tables.py) to the device.
 * Replaces: grammar.load_pinned()/load_pinned_extended() lookups
 * (reference grammar.py:97-154) as seen by ops.py / disasm.py / validate.py. */
int skg_tables_create(const uint32_t* host_blob, uint64_t n_words, skg_tables** out);
void skg_tables_destroy(skg_tables* t);

/* Device workspace (bytes) for a batch of n_mod modules whose largest module
 * has max_words words.  Includes the counters (ticket, errors, allocator) and the per-warp
 * overflow scratch of the persistent grid. */
uint64_t skg_workspace_bytes(uint32_t n_mod, uint32_t max_words);

/* Batch disassembly.
 * Replaces: Disassembler.to_text / disassemble_module(data, options, strict=...)
 * (reference disasm.py:117-127, 392-398) for every module of the batch.
 * Output: text arena `text` (capacity text_cap bytes); module m's text is
 * text[text_span[2m] : text_span[2m] + text_span[2m+1]].  Modules reserve their
 * bytes with an atomic bump allocator, so the arena holds the modules' texts in
 * completion order (no inter-module ordering wait on the device).
 * status[m] = SKG_ST_*; errors[] gets one record per failing module (up to
 * err_cap; counters: see skg_last_counts).  If the arena is too small the
 * modules that do not fit are not written, the overflow flag is set and the
 * required size is reported by skg_last_counts. */
int skg_disasm(const skg_tables* t, const uint8_t* data, const int64_t* mod_off,
               const int64_t* mod_len, uint32_t n_mod, uint32_t opts, uint32_t max_words,
               uint8_t* text, uint64_t text_cap, int64_t* text_span, int32_t* status,
               skg_error* errors, uint32_t err_cap, void* workspace, uint64_t workspace_bytes,
               void* stream);

/* skg_disasm with explicit id refs for every module of the batch: the text of
 * format_instruction(spec, inst, context) with a RenderContext whose `refs`
 * name some ids (reference disasm.py:57-67, 380-389).  ref_ids: n_refs
 * entries of 3 uint32 (id, byte offset into ref_text, byte length), ascending
 * by id; an id listed there renders as exactly that text (result column and
 * operands); all other ids render as usual. */
int skg_disasm_refs(const skg_tables* t, const uint8_t* data, const int64_t* mod_off,
                    const int64_t* mod_len, uint32_t n_mod, uint32_t opts, uint32_t max_words,
                    uint8_t* text, uint64_t text_cap, int64_t* text_span, int32_t* status,
                    skg_error* errors, uint32_t err_cap, void* workspace, uint64_t workspace_bytes,
                    void* stream, const uint32_t* ref_ids, const uint8_t* ref_text, uint32_t n_refs);

/* Fused decode -> validate -> disassemble: ONE pass over the batch
 * produces both skg_disasm's outputs (text, text_span, status, errors) and
 * skg_validate's (vtext, vtext_span, vstatus, verrors) from a single read and a
 * single decode of every module (shared boundary pass, grammar walk, id tables
 * and prescan).  Counters: skg_last_counts(workspace) for the text,
 * skg_last_counts((char*)workspace + 128) for the diagnostics arena. */
int skg_disasm_validate(const skg_tables* t, const uint8_t* data, const int64_t* mod_off,
                        const int64_t* mod_len, uint32_t n_mod, uint32_t opts, uint32_t max_words,
                        uint8_t* text, uint64_t text_cap, int64_t* text_span, int32_t* status,
                        skg_error* errors, uint32_t err_cap, uint8_t* vtext, uint64_t vtext_cap,
                        int64_t* vtext_span, int32_t* vstatus, skg_error* verrors, uint32_t verr_cap,
                        void* workspace, uint64_t workspace_bytes, void* stream);

/* Batch structural + capability validation.
 * Replaces: validate_module(bytes) (reference validate.py:73-94).
 * Output: diagnostics_text-formatted lines ("severity code location message\n")
 * per module in the `text` arena (same span convention as skg_disasm);
 * non-codec exceptions that escape the reference validator are reported
 * through status/errors exactly like skg_disasm. */
int skg_validate(const skg_tables* t, const uint8_t* data, const int64_t* mod_off,
                 const int64_t* mod_len, uint32_t n_mod, uint32_t max_words, uint8_t* text,
                 uint64_t text_cap, int64_t* text_span, int32_t* status, skg_error* errors,
                 uint32_t err_cap, void* workspace, uint64_t workspace_bytes, void* stream);

/* Instruction-boundary pass only (header + per-instruction offsets).
 * Replaces: codec.decode_module (reference codec.py:199-231).
 * inst_off receives, for module m, the word offsets of its instructions at
 * inst_off[inst_base[m] ...]; inst_base (n_mod+1) is computed by the caller as
 * an exclusive bound (the library writes inst_count[m]).  header: 5 words per
 * module (byte-order normalised). */
int skg_decode(const uint8_t* data, const int64_t* mod_off, const int64_t* mod_len, uint32_t n_mod,
               uint32_t* header, uint32_t* inst_off, const int64_t* inst_base, uint32_t* inst_count,
               uint32_t* words_out, const int64_t* words_base, int32_t* status, skg_error* errors,
               uint32_t err_cap, void* workspace, uint64_t workspace_bytes, void* stream);

/* Batch assembly (text -> binary).
 * Replaces: Assembler.assemble / assemble_module(text) (reference asm.py:133-180,
 * 365-368) together with the builder serialization it drives (builder.py:108-242).
 * Input: UTF-8 text arena `text` (module starts 16-byte aligned, arena padded
 * to 16 bytes) with int64 per-module offsets/lengths read at index m * mod_stride
 * (stride 2 accepts skg_disasm's interleaved text_span directly, so a
 * disassemble -> assemble round trip needs no host work).  Output arena `out`:
 * module m's result is out[out_span[2m] : out_span[2m] + out_span[2m+1]] -- the
 * module binary when status[m] == SKG_ST_OK, otherwise the exact str(exc) text
 * (UTF-8) of the exception class status[m] names.  Bytes are reserved with an
 * atomic bump allocator (skg_last_counts reports overflow / bytes used, as for
 * skg_disasm).  `slot_bytes` is the per-warp scratch (skg_asm_slot_hint); a
 * module that needs more reports SKG_ST_INTERNAL and can be rerun with a
 * larger slot.  `workspace` must hold skg_asm_workspace_bytes(slot_bytes, n_mod).
 * default_version = major << 16 | minor: the Assembler's default_version
 * (asm.py:128), used when the text has no "; Version:" comment. */
uint64_t skg_asm_slot_hint(uint64_t max_text_bytes);
uint64_t skg_asm_workspace_bytes(uint64_t slot_bytes, uint32_t n_mod);
int skg_asm(const skg_tables* t, const uint8_t* text, const int64_t* mod_off, const int64_t* mod_len,
            uint32_t mod_stride, uint32_t n_mod, uint64_t slot_bytes, uint8_t* out, uint64_t out_cap, int64_t* out_span,
            int32_t* status, void* workspace, uint64_t workspace_bytes, void* stream,
            uint32_t default_version);

/* decode_module for ONE large module (config-3 sizes), parallel over 4096-word
 * tiles of the stream: speculative per-tile boundary walks, a sequential link
 * pass that only walks until the true chain merges with a tile's speculative
 * chain, then per-tile count / scan / write (skg_bigdecode.cuh).
 * Replaces: codec.decode_module (reference codec.py:199-231) like skg_decode,
 * for one module of nbytes bytes at `data` (device).  max_opcode (the grammar's
 * largest opcode, 0 = no filter) only steers the speculation, never the result.
 * header[5] = major, minor,
 * generator, bound, schema; words_out[nbytes/4] = byte-order-normalised words;
 * inst_off[*inst_count] = instruction start offsets; *status = SKG_ST_*, and on
 * failure *error holds the exact message.  `workspace` must hold
 * skg_decode_large_workspace_bytes(nbytes / 4). */
uint64_t skg_decode_large_workspace_bytes(uint64_t n_words);
int skg_decode_large(const uint8_t* data, uint64_t nbytes, uint32_t max_opcode, uint32_t* header,
                     uint32_t* inst_off, uint32_t* inst_count, uint32_t* words_out, int32_t* status,
                     skg_error* error, void* workspace, uint64_t workspace_bytes, void* stream);

/* validate_module for ONE large module (config 3) over the whole GPU: the tiled
 * boundary pass, then one grid-stride kernel per phase (first/last-wins id maps
 * by atomics on the instruction index, per-instruction diagnostic sizes, a
 * device-wide scan, the write; skg_big.cuh).  Host-synchronous.
 * Replaces: validate.validate_module (reference validate.py:73-94) for one
 * module of nbytes bytes at `data` (device).  Returns 0: text[0:*text_bytes]
 * holds the diagnostics_text lines and *status = SKG_ST_OK; 1: an exception
 * escapes (*status, *error); 3: *text_bytes > text_cap (call again with a
 * larger arena); 10 + s: the module does not decode (status s, *error = the
 * message: the validator's only diagnostic); 2: ids at/above the header bound
 * (use skg_validate).  `workspace` must hold skg_large_workspace_bytes(nbytes
 * / 4, S) with S = max(header bound, min_table).  min_table (0 = the header
 * bound) widens the direct id tables: a module with ids at or above its header
 * bound (return 2) can be redone with min_table = 2 * nbytes / 4 + 64 instead of
 * falling back to the one-warp path; messages keep the header bound. */
uint64_t skg_large_workspace_bytes(uint64_t n_words, uint32_t bound);
int skg_validate_large(const skg_tables* t, const uint8_t* data, uint64_t nbytes, uint8_t* text,
                       uint64_t text_cap, uint64_t* text_bytes, int32_t* status, skg_error* error,
                       void* workspace, uint64_t workspace_bytes, void* stream, uint32_t min_table);

/* disassemble_module for ONE large module (config 3) over the whole GPU: the
 * phases of skg_disasm as grid-wide kernels (tiled boundary pass, atomic id
 * maps, per-instruction grammar walks, friendly names with device-wide scans
 * and a prefix-max over id space, the text written per 1024-word range at
 * scanned offsets; skg_disasm.cu / skg_big.cuh).  Host-synchronous.
 * Replaces: Disassembler.to_text (reference disasm.py:117-127) for one module
 * of nbytes bytes at `data` (device) with option bits `opts` (SKG_OPT_*).
 * Returns 0: text[0:*text_bytes] and *status = SKG_ST_OK; 1: the exception the
 * reference raises (*status, *error); 3: *text_bytes > text_cap (call again);
 * 10 + s: the module does not decode (status s, *error); 2: ids at/above the
 * header bound (use skg_disasm).  Workspace: skg_large_workspace_bytes. */
int skg_disasm_large(const skg_tables* t, const uint8_t* data, uint64_t nbytes, uint32_t opts, uint8_t* text,
                     uint64_t text_cap, uint64_t* text_bytes, int32_t* status, skg_error* error,
                     void* workspace, uint64_t workspace_bytes, void* stream, uint32_t min_table);

/* tokenize_line for a batch of lines (reference asm.py:51-90).
 * Input: UTF-8 byte arena `text` with int64 per-line offsets/lengths (one
 * logical line each, no line separators inside).  Output, line l with its
 * tokens in slots line_off[l] + k (k < ntok[l]; the arrays are sized like
 * `text`): tok_off = byte offset of the token text -- in `text` for bare
 * tokens, in `esc` (same size as `text`) for string tokens, which are stored
 * with their backslash escapes resolved; tok_len = bytes; tok_col = 1-based
 * code-point column of the token start (the quote for strings); tok_flags bit 0
 * = string token.  kind[l]: 0 blank/comment line (None), 1 instruction, 2
 * instruction with a "%r =" result, 3 unterminated string literal (err_col[l]
 * = column of its opening quote). */
int skg_tokenize(const uint8_t* text, const int64_t* line_off, const int64_t* line_len, uint32_t n_lines,
                 uint64_t* tok_off, uint32_t* tok_len, uint32_t* tok_col, uint8_t* tok_flags, uint8_t* esc,
                 int32_t* kind, int32_t* ntok, uint32_t* err_col, void* stream);

/* encode_module for a batch (reference codec.py:192-196 with encode_header
 * :61-79 and encode_instruction :92-101; the words of ModuleScope.serialize,
 * builder.py:208-224).  header: 5 int64 per module (major, minor,
 * generator_magic & 0xFFFFFFFF, bound, schema & 0xFFFFFFFF); module m owns
 * instructions [inst_base[m], inst_base[m+1]); instruction i has opcode[i] and
 * the operand words ops[op_off[i] : op_off[i+1]] (already masked to 32 bits;
 * op_off has n_inst + 1 entries).  Module m's words start at word
 * 5m + inst_base[m] + op_off[inst_base[m]] of `out`.  err[m] = all ones when
 * the module encodes, else (k << 8 | code) for its first error: code 1 bound 0,
 * 2 bound out of range, 3 version bytes (k = 0), 4 instruction length
 * overflows 16 bits, 5 opcode out of range (k = 1 + instruction index in the
 * module). */
int skg_encode_modules(const int64_t* header, uint32_t n_mod, const int64_t* inst_base, const int64_t* opcode,
                       uint64_t n_inst, const int64_t* op_off, const uint32_t* ops, uint64_t n_ops,
                       uint32_t* out, uint64_t* err, void* stream);

/* encode_string_literal for a batch of UTF-8 strings (reference codec.py:104-114):
 * string s = bytes[off[s] : off[s] + len[s]] packs into len[s] / 4 + 1
 * little-endian words (NUL-terminated, zero padded) at out[word_off[s]...];
 * bad[s] is set to 1 (caller zeroes it) when the string holds a NUL byte
 * (CodecError). */
int skg_pack_strings(const uint8_t* bytes, const int64_t* off, const int64_t* len, const int64_t* word_off,
                     uint32_t n_str, uint64_t n_words, uint32_t* out, int32_t* bad, void* stream);

/* encode_context_dependent_literal for a batch (reference codec.py:132-168).
 * width[k]: bit width; flags[k]: 1 signed, 2 floating, 4 negative integer, 8
 * integer magnitude >= 2^64, 16 width is None (unresolved); val[k]: |integer| or the IEEE-754
 * double bits of the float.  Output words[2k], words[2k+1] (nwords[k] of them)
 * and status[k]: 0 ok, 1 unresolved width, 2 unsupported width, 3 unsupported
 * float width, 4 OverflowError (e format), 5 OverflowError (f format), 6 / 7 the
 * value does not fit a signed / unsigned literal of that width. */
int skg_ctx_literals(const int64_t* width, const uint32_t* flags, const uint64_t* val, uint32_t n,
                     uint32_t* words, int32_t* nwords, int32_t* status, void* stream);

/* Self-test (tests only): repr() of every float32 bit pattern in [start, start +
 * count) as the disassembler renders it, checked on the device against the
 * assembler's independent float() parser -- the text reads back as the same
 * double and no (n-1)-significant-digit neighbour does (shortest round trip);
 * nan / inf / zero spelled as CPython does.  *fails += failures (caller zeroes),
 * *first_fail = min failing bit pattern (caller sets 0xFFFFFFFF). */
int skg_selftest_repr_f32(const skg_tables* t, uint64_t start, uint64_t count, uint64_t* fails,
                          uint32_t* first_fail, void* stream);

/* Counters of the last call on `workspace` (device->host copy, synchronous on
 * `stream`): number of error records wanted, 1 if the text arena overflowed,
 * and the text bytes the batch needs (allocator cursor). */
int skg_last_counts(const void* workspace, uint32_t* n_errors, uint32_t* text_overflow,
                    uint64_t* text_bytes, void* stream);

/* Copy n_words 32-bit words from device memory into page-locked host memory
 * (host_dst from cudaHostAlloc / a pinned tensor) with a kernel on `stream`:
 * the stores travel over PCIe without a copy engine, so a pipeline can read a
 * chunk's counters while a large D2H copy of the previous chunk is in flight
 * (a cudaMemcpyAsync of the counters would queue behind it).  Not a reference
 * interface: plumbing of the host-buffer round-trip session. */
int skg_store_counters(void* host_dst, const void* dev_src, uint32_t n_words, void* stream);

/* Copy n_bytes from device memory into page-locked host memory (host_dst from
 * cudaHostAlloc / a pinned tensor; both 16-byte aligned, else a plain async copy)
 * with a kernel of n_ctas CTAs (0: 64) on `stream`: SM stores over PCIe, no copy
 * engine, so small driver copies of concurrent calls do not queue behind it
 * (skg_disasm_large's text while skg_validate_large runs).  Not a reference
 * interface: plumbing of the single-large-module disassemble + validate call. */
int skg_copy_to_host(void* host_dst, const void* dev_src, uint64_t n_bytes, uint32_t n_ctas, void* stream);

/* Version / build info string. */
const char* skg_version(void);

#ifdef __cplusplus
}
#endif
#endif
