// binding_main.cpp — TEST: the INTEGRATION.md binding (gpu_binding.hpp),
// compiled against the unmodified reference headers and library, against the
// reference's own run_sieve on the same sinks.  Exit 0 = every case equal.
//   erato_binding_test            all cases (needs a GPU)
//   erato_binding_test --link     only proves it linked (CPU container)
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <iterator>
#include <string>
#include <unistd.h>

#include "gpu_binding.hpp"

namespace {

struct Collect final : erato::SegmentSink {  // a user sink: bytes + the order of t
  std::vector<uint8_t> bytes;
  std::vector<uint64_t> ts;
  void on_segment(const erato::SegmentBuffer& seg, uint64_t t, const erato::SieveParams& p) override {
    const size_t off = bytes.size();
    bytes.resize(off + p.segment_bytes());
    erato::segment_to_bytes(seg, bytes.data() + off);
    ts.push_back(t);
  }
};

std::string slurp(const std::filesystem::path& p) {
  std::ifstream in(p, std::ios::binary);
  return std::string(std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>());
}

int fails = 0;
void expect(bool ok, const char* what, unsigned l, uint64_t f, uint64_t n) {
  if (!ok) {
    std::printf("FAIL %s (l=%u f=%llu n=%llu)\n", what, l, (unsigned long long)f, (unsigned long long)n);
    ++fails;
  }
}

}  // namespace

int main(int argc, char** argv) {
  if (argc > 1 && std::strcmp(argv[1], "--link") == 0) {
    std::printf("linked: erato_gpu_run_to_sink=%p\n", (void*)&erato_gpu_run_to_sink);
    return 0;
  }
  struct Case { unsigned l; uint64_t f, n; bool test; };
  const Case cases[] = {{10, 2048, 4, false}, {12, 4096, 8, false}, {4, 2048, 4, true}, {20, 523776, 40, false},
                        {22, (uint64_t{1} << 37) - 4096, 40, false}, {13, 5000, 77, false}, {10, 6, 1, false}};
  const auto dir = std::filesystem::temp_directory_path() / ("erato_binding_" + std::to_string(::getpid()));
  for (const Case& c : cases) {
    const auto p = erato::validate_params(c.l, c.f, c.n, c.test);
    erato::NullSink n1, n2;
    const auto g0 = erato::run_sieve_gpu(p, n1), r0 = erato::run_sieve(p, n2);
    expect(g0.prime_count == r0.prime_count, "NullSink count", c.l, c.f, c.n);
    erato::TableSink t1, t2;
    const auto g1 = erato::run_sieve_gpu(p, t1);
    erato::run_sieve(p, t2);
    expect(t1.bytes() == t2.bytes() && g1.prime_count == r0.prime_count, "TableSink bytes", c.l, c.f, c.n);
    erato::PrimeCollectSink c1, c2;
    erato::run_sieve_gpu(p, c1);
    erato::run_sieve(p, c2);
    expect(c1.primes() == c2.primes(), "PrimeCollectSink primes", c.l, c.f, c.n);
    Collect u1;
    erato::run_sieve_gpu(p, u1);
    bool in_order = u1.ts.size() == p.n;
    for (uint64_t t = 0; t < u1.ts.size(); ++t) in_order = in_order && u1.ts[t] == t;
    expect(in_order && u1.bytes == t2.bytes(), "user sink order + bytes", c.l, c.f, c.n);
    {
      std::string a, b;
      {
        erato::FileSink fs(dir / "gpu", p);
        erato::run_sieve_gpu(p, fs);
        a = slurp(fs.path());
      }
      {
        erato::FileSink fs(dir / "ref", p);
        erato::run_sieve(p, fs);
        b = slurp(fs.path());
      }
      expect(!a.empty() && a == b, "FileSink file", c.l, c.f, c.n);
    }
  }
  // errors keep the reference's codes
  try {
    erato::SieveParams bad;
    bad.l = 3;
    bad.f = 1;
    bad.n = 1;
    erato::NullSink ns;
    erato::run_sieve_gpu(bad, ns);
    expect(false, "L_OUT_OF_RANGE thrown", 3, 1, 1);
  } catch (const erato::Error& e) {
    expect(e.code() == erato::errc::l_out_of_range, "L_OUT_OF_RANGE code", 3, 1, 1);
  }
  std::filesystem::remove_all(dir);
  std::printf(fails ? "binding FAILED (%d)\n" : "binding OK: run_sieve_gpu == run_sieve on every sink%.0d\n", fails);
  return fails ? 1 : 0;
}
