// Instruction-boundary pass for decode_module (reference codec.py:199-231):
// one thread per module (the single-module API and small batches), writing the
// byte-order-normalised words, the header and every instruction's word offset.
#include "skg_module.cuh"

namespace skg {

struct DecodeArgs {
  const uint8_t* data;
  const int64_t* mod_off;
  const int64_t* mod_len;
  uint32_t n_mod;
  uint32_t* header;          // 5 per module
  uint32_t* inst_off;        // at inst_base[m]
  const int64_t* inst_base;
  uint32_t* inst_count;
  uint32_t* words_out;       // normalised words at words_base[m]
  const int64_t* words_base;
  int32_t* status;
  uint32_t* counters;        // [1] error count
  ErrRec* errs;
  uint32_t err_cap;
};

__global__ void decode_kernel(DecodeArgs a) {
  const uint32_t m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= a.n_mod) return;
  const int64_t n = a.mod_len[m];
  const uint8_t* src = a.data + a.mod_off[m];
  ErrSink es{a.errs, a.counters + 1, a.err_cap};
  a.inst_count[m] = 0;
  if (n % 4 != 0 || n < 20) {
    a.status[m] = ST_TRUNCATED;
    if (ErrRec* r = es.alloc()) {
      ErrWriter ew{r};
      put_u64(ew, (uint64_t)n);
      put_cstr(ew, " bytes is not a whole word stream of at least 5 words");
      r->module = (int32_t)m; r->cls = ST_TRUNCATED; r->len = ew.n;
    }
    return;
  }
  const uint32_t W = (uint32_t)(n / 4);
  auto raw = [&](uint32_t k) {
    const uint8_t* p = src + 4ull * k;
    return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
  };
  const uint32_t w0 = raw(0);
  bool swap = false;
  if (w0 != MAGIC) {
    if (bswap32(w0) != MAGIC) {
      a.status[m] = ST_NOTSPIRV;
      if (ErrRec* r = es.alloc()) {
        ErrWriter ew{r};
        put_cstr(ew, "magic word 0x"); put_hex8_upper(ew, w0); put_cstr(ew, " is not SPIR-V");
        r->module = (int32_t)m; r->cls = ST_NOTSPIRV; r->len = ew.n;
      }
      return;
    }
    swap = true;
  }
  uint32_t* out = a.words_out + a.words_base[m];
  for (uint32_t k = 0; k < W; ++k) {
    uint32_t v = raw(k);
    out[k] = swap ? bswap32(v) : v;
  }
  uint32_t* h = a.header + 5ull * m;
  h[0] = (out[1] >> 16) & 0xFF;
  h[1] = (out[1] >> 8) & 0xFF;
  h[2] = out[2];
  h[3] = out[3];
  h[4] = out[4];
  uint32_t* io = a.inst_off + a.inst_base[m];
  uint32_t p = 5, I = 0;
  while (p < W) {
    uint32_t wc = out[p] >> 16;
    int32_t st = wc == 0 ? ST_CORRUPT : (p + wc > W ? ST_TRUNCATED : ST_OK);
    if (st != ST_OK) {
      a.status[m] = st;
      if (ErrRec* r = es.alloc()) {
        ErrWriter ew{r};
        put_cstr(ew, "instruction at word "); put_u64(ew, p);
        put_cstr(ew, st == ST_CORRUPT ? " has word count 0" : " runs past the end of the stream");
        r->module = (int32_t)m; r->cls = st; r->len = ew.n;
      }
      return;
    }
    io[I++] = p;
    p += wc;
  }
  a.inst_count[m] = I;
  a.status[m] = ST_OK;
}

}  // namespace skg
