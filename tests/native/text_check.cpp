// Host build of the assembler's text primitives (test infrastructure only):
// argv[1] = grammar table blob (uint32 LE, tables.py) for the Unicode tables.
// stdin commands, one per line, payload hex-encoded UTF-8:
//   I <base> <hex>   int(s, base)        -> "OK <str(v)|LIMITSTR> <format(v,'#x')>" | "INVALID" | "LIMIT <n>"
//   F <hex>          float(s)            -> "<16 hex digits of the double>" | "INVALID"
//   R <limit> <hex>  repr(s)[:limit]     -> hex of the UTF-8 repr
//   P <hex64>        pack('<e'), pack('<f') -> "<h|OVF> <f|OVF>"
#define SKG_HD
#define SKG_TABLE
#define SKG_NOINLINE
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>
#include "../../paper_2305_09493_b200/csrc/skg_text.cuh"

struct StrSink {
  std::string s;
  void put(uint8_t c) { s.push_back((char)c); }
  void putn(const uint8_t* p, uint32_t n) { s.append((const char*)p, n); }
  void fill(uint8_t c, uint32_t k) { s.append(k, (char)c); }
};

static std::vector<uint8_t> unhex(const char* h) {
  std::vector<uint8_t> out;
  for (size_t i = 0; h[i] && h[i + 1]; i += 2) {
    unsigned v;
    sscanf(h + i, "%2x", &v);
    out.push_back((uint8_t)v);
  }
  return out;
}
static std::string tohex(const std::string& s) {
  std::string o;
  char b[3];
  for (unsigned char c : s) { snprintf(b, 3, "%02x", c); o += b; }
  return o;
}

int main(int argc, char** argv) {
  FILE* f = fopen(argv[1], "rb");
  std::vector<uint32_t> blob;
  uint32_t w;
  while (fread(&w, 4, 1, f) == 1) blob.push_back(w);
  fclose(f);
  const uint32_t* h = blob.data();
  skg::Uni U{h + h[41], h[42], h + h[43], h[44], h + h[45], h[46], h + h[47], h[48]};
  static char line[1 << 22];
  std::vector<uint32_t> scratch(1 << 16);
  while (fgets(line, sizeof line, stdin)) {
    size_t L = strlen(line);
    while (L && (line[L - 1] == '\n' || line[L - 1] == '\r')) line[--L] = 0;
    char* sp = strchr(line, ' ');
    if (line[0] == 'I') {
      unsigned base;
      char* rest = sp + 1;
      sscanf(rest, "%u", &base);
      char* hx = strchr(rest, ' ');
      std::vector<uint8_t> s = unhex(hx ? hx + 1 : "");
      skg::IntVal v = skg::parse_int(s.data(), (uint32_t)s.size(), base, U);
      if (v.status == skg::INT_INVALID) puts("INVALID");
      else if (v.status == skg::INT_LIMIT) printf("LIMIT %u\n", v.ndig);
      else {
        StrSink d, x;
        bool ok = skg::put_int_decimal(d, s.data(), v, U, scratch.data(), (uint32_t)scratch.size() / 2);
        skg::put_int_hex(x, s.data(), v, U, scratch.data(), (uint32_t)scratch.size());
        printf("OK %s %s\n", ok ? d.s.c_str() : "LIMITSTR", x.s.c_str());
      }
    } else if (line[0] == 'F') {
      std::vector<uint8_t> s = unhex(sp ? sp + 1 : "");
      uint64_t bits;
      if (skg::parse_float(s.data(), (uint32_t)s.size(), U, bits) != skg::FLT_OK) puts("INVALID");
      else printf("%016llx\n", (unsigned long long)bits);
    } else if (line[0] == 'R') {
      unsigned lim;
      char* rest = sp + 1;
      sscanf(rest, "%u", &lim);
      char* hx = strchr(rest, ' ');
      std::vector<uint8_t> s = unhex(hx ? hx + 1 : "");
      StrSink o;
      skg::put_py_repr(o, s.data(), (uint32_t)s.size(), U, lim);
      printf("%s\n", tohex(o.s).c_str());
    } else if (line[0] == 'P') {
      unsigned long long b;
      sscanf(sp + 1, "%llx", &b);
      uint32_t a16, a32;
      bool o16 = skg::pack_f16(b, a16), o32 = skg::pack_f32(b, a32);
      if (o16) printf("%04x ", a16); else printf("OVF ");
      if (o32) printf("%08x\n", a32); else printf("OVF\n");
    }
  }
  return 0;
}
