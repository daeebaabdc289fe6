// Host build of the device formatting primitives (test infrastructure only):
// reads hex bit patterns on stdin ("d XXXXXXXXXXXXXXXX", "f XXXXXXXX", "h XXXX"),
// prints the repr the CUDA code would emit, one per line.
#define SKG_HD
#define SKG_TABLE
#define SKG_NOINLINE
#include <cstdio>
#include <cstring>
#include <string>
#include "../../paper_2305_09493_b200/csrc/skg_fmt.cuh"

struct StrSink {
  std::string s;
  void put(uint8_t c) { s.push_back((char)c); }
  void putn(const uint8_t* p, uint32_t n) { s.append((const char*)p, n); }
  void fill(uint8_t c, uint32_t k) { s.append(k, (char)c); }
};

int main() {
  char kind[4];
  unsigned long long v;
  while (scanf("%3s %llx", kind, &v) == 2) {
    uint64_t bits = v;
    if (kind[0] == 'f') bits = skg::f32_to_f64_bits((uint32_t)v);
    if (kind[0] == 'h') bits = skg::f16_to_f64_bits((uint32_t)v);
    StrSink s;
    skg::put_repr_double(s, bits);
    puts(s.s.c_str());
  }
  return 0;
}
