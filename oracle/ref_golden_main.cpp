// oracle/_ref driver — TEST INFRASTRUCTURE ONLY. Compiled against the reference's OWN shipped
// infrastructure sources where they lie (/root/reference/proj/core/include/snop/rng.hpp,
// parallel.hpp, src/binary_io.cpp; never copied into this repo) to emit golden vectors that pin
// the oracle's and the product's restatements of the seeded-input RNG stream (rng.hpp:17-49),
// the deterministic chunk partition (parallel.hpp:17-48) and the FNV-1a-64 file digest
// (binary_io.cpp:12-17,73-83). Output: JSON on stdout.
#include <cstdio>
#include <mutex>
#include <vector>

#include "snop/binary_io.hpp"
#include "snop/parallel.hpp"
#include "snop/rng.hpp"

int main(int argc, char** argv) {
  const char* tmpfile = argc > 1 ? argv[1] : "/tmp/snop_ref_golden.bin";
  std::printf("{\n  \"rng\": [\n");
  const unsigned long long seeds[] = {0ull, 1ull, 42ull, 1234567ull, 0xdeadbeefcafeull};
  for (int s = 0; s < 5; ++s) {
    snop::Rng a(seeds[s]), b(seeds[s]), c(seeds[s]);
    std::printf("    {\"seed\": %llu, \"u64\": [", seeds[s]);
    for (int i = 0; i < 8; ++i) std::printf("%s\"%llu\"", i ? ", " : "", (unsigned long long)a.next_u64());
    std::printf("], \"uniform\": [");
    for (int i = 0; i < 8; ++i) std::printf("%s%.17g", i ? ", " : "", b.uniform());
    std::printf("], \"normal\": [");
    for (int i = 0; i < 7; ++i) std::printf("%s%.17g", i ? ", " : "", c.normal());
    std::printf("]}%s\n", s < 4 ? "," : "");
  }
  std::printf("  ],\n  \"rng_10000th\": ");
  {
    snop::Rng r(5489ull);
    unsigned long long v = 0;
    for (int i = 0; i < 10000; ++i) v = r.next_u64();
    std::printf("\"%llu\",\n", v);
  }
  std::printf("  \"chunks\": [\n");
  const std::size_t cases[][2] = {{10, 3}, {2048, 8}, {7, 7}, {5, 9}, {1000, 64}};
  for (int k = 0; k < 5; ++k) {
    std::vector<std::pair<std::size_t, std::size_t>> got(cases[k][1] > cases[k][0] ? cases[k][0] : cases[k][1]);
    std::mutex m;
    snop::parallel_chunks(cases[k][0], cases[k][1], [&](std::size_t c, std::size_t b, std::size_t e) {
      std::lock_guard<std::mutex> lk(m);
      got[c] = {b, e};
    }, 3);
    std::printf("    {\"n_items\": %zu, \"n_chunks\": %zu, \"bounds\": [", cases[k][0], cases[k][1]);
    for (std::size_t c = 0; c < got.size(); ++c) std::printf("%s[%zu, %zu]", c ? ", " : "", got[c].first, got[c].second);
    std::printf("]}%s\n", k < 4 ? "," : "");
  }
  std::printf("  ],\n");
  {
    snop::BinaryWriter w(tmpfile);
    w.write_u32(7u);
    w.write_f64(1.30621);
    const double arr[3] = {0.5, -2.25, 1e-300};
    w.write_f64_array(std::span<const double>(arr, 3));
    w.write_string("snop");
    const unsigned long long d = w.digest();
    w.finish();
    std::FILE* f = std::fopen(tmpfile, "rb");
    std::printf("  \"binary_io\": {\"digest\": \"%llu\", \"bytes_hex\": \"", d);
    int ch;
    while ((ch = std::fgetc(f)) != EOF) std::printf("%02x", ch);
    std::fclose(f);
    std::printf("\"},\n");
  }
  // Model files written through the reference's own BinaryWriter with the
  // record of paper_2509_01416_b200/csrc/model_io.h; tiny fixed architectures, parameters
  // exactly representable in fp32 (tests/test_model_io.py regenerates them the same way).
  {
    auto hex_of = [&](const char* label, bool last) {
      std::FILE* f = std::fopen(tmpfile, "rb");
      std::printf("  \"%s\": \"", label);
      int ch;
      while ((ch = std::fgetc(f)) != EOF) std::printf("%02x", ch);
      std::fclose(f);
      std::printf("\"%s\n", last ? "" : ",");
    };
    {
      snop::BinaryWriter w(tmpfile);
      w.write_string("SNOP-MODEL");
      w.write_u32(1);
      w.write_string("deeponet");
      w.write_f64(10.0);
      w.write_u64(4);
      w.write_f64(1.0);
      w.write_f64(0.5);
      w.write_u32(1);  // tanh
      const unsigned long long bs[3] = {4, 3, 2}, ts[3] = {1, 3, 2};
      w.write_u32(3);
      for (auto v : bs) w.write_u64(v);
      w.write_u32(3);
      for (auto v : ts) w.write_u64(v);
      w.write_u8(1);
      w.write_f64(0.125);
      const int nbp = 4 * 3 + 3 + 3 * 2 + 2, ntp = 1 * 3 + 3 + 3 * 2 + 2;
      w.write_u64(nbp + ntp);
      for (int i = 0; i < nbp; ++i) w.write_f64((double)(((i % 7) - 3) * 0.125f));
      for (int i = 0; i < ntp; ++i) w.write_f64((double)(((i % 5) - 2) * 0.25f));
      w.finish();
      hex_of("model_deeponet_hex", false);
    }
    {
      snop::BinaryWriter w(tmpfile);
      w.write_string("SNOP-MODEL");
      w.write_u32(1);
      w.write_string("fno");
      w.write_f64(10.0);
      w.write_u64(8);
      w.write_f64(1.0);
      w.write_f64(0.8);
      w.write_u32(2);  // gelu
      const unsigned long long dims[4] = {2, 2, 1, 3};  // width, modes, layers, hidden
      for (auto v : dims) w.write_u64(v);
      const int np = 3 * 2 + 1 * (2 * 2 * 2 * 2 + 2 * 2 + 2) + 3 * 2 + 2 * 3 + 1;
      w.write_u64(np);
      for (int i = 0; i < np; ++i) w.write_f64((double)((float)(((i * 3) % 11) - 5) / 16.0f));
      w.finish();
      hex_of("model_fno_hex", true);
    }
  }
  std::printf("}\n");
  return 0;
}
