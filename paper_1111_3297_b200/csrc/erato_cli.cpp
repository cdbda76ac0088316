// erato_cli.cpp — command-line front end over the C ABI (include/erato_gpu.h),
// with the flags, output lines and exit codes of the reference CLI
// (/root/reference/proj/tools/erato.cpp:65-176):
//
//   erato-gpu sieve  --log-seg 21 --midpoint-exp 12 --segments 512 --count-only
//   erato-gpu sieve  --log-seg 10 --first 2048 --segments 4 --out-dir /tmp
//   erato-gpu verify --log-seg 12 --first 4096 --segments 8
//   erato-gpu bench  --exps 12,13,14 --csv bench.csv
//   erato-gpu sieve  --log-seg 22 --first 137438949376 --segments 8192 --gpus 8
//
// --gpus N / --devices D0,D1,..: range shards over several GPUs (one host
// thread each, counts summed with one ncclAllReduce; erato_gpu_multi_*).
//
// Exit codes: 0 success, 1 parameter error, 2 runtime error.  Extension:
// --allow-overlap admits f = 0 / u^2 <= v (SURVEY.md §8c convention).
// `verify` checks the GPU table against an independent Miller-Rabin test
// (every bit for tables up to 2^22 bits, a seeded sample above).
#include <algorithm>
#include <chrono>
#include <cerrno>
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "../../include/erato_gpu.h"

namespace {

struct Flags {
  std::string cmd;
  unsigned l = 21;
  bool have_f = false, have_e = false, have_n = false;
  uint64_t f = 0;
  unsigned e = 0;
  uint64_t n = 1;
  bool test_mode = false, count_only = false, allow_overlap = false;
  std::string out_dir;
  uint64_t max_base_pairs = uint64_t{1} << 27;
  std::vector<unsigned> exps;
  std::string csv, machine = "unknown";
  unsigned reps = 3;
  std::vector<int> devices;  // --gpus / --devices (empty: one GPU, device 0)
};

[[noreturn]] void usage(const char* msg) {
  std::fprintf(stderr,
               "error: %s\n"
               "usage: erato-gpu sieve|verify --log-seg L (--first F | --midpoint-exp E) --segments N\n"
               "                 [--test-mode] [--allow-overlap] [--out-dir D] [--count-only] [--max-base-pairs P]\n"
               "                 [--gpus N | --devices D0,D1,..]\n"
               "       erato-gpu bench --exps E1,E2,.. [--log-seg L] [--csv PATH] [--reps R] [--machine M]\n",
               msg);
  std::exit(1);
}

bool parse_u64(const char* s, uint64_t& out) {
  if (!s || !*s) return false;
  char* end = nullptr;
  errno = 0;
  const unsigned long long v = std::strtoull(s, &end, 10);
  if (errno || *end || s[0] == '-') return false;
  out = v;
  return true;
}

Flags parse(int argc, char** argv) {
  Flags fl;
  if (argc < 2) usage("a subcommand is required");
  fl.cmd = argv[1];
  if (fl.cmd != "sieve" && fl.cmd != "verify" && fl.cmd != "bench") usage("unknown subcommand");
  const char* tmp = std::getenv("TMPDIR");  // std::filesystem::temp_directory_path (erato.cpp:92)
  fl.out_dir = tmp && *tmp ? tmp : "/tmp";
  for (int i = 2; i < argc; ++i) {
    const std::string a = argv[i];
    auto val = [&](void) -> const char* {
      if (i + 1 >= argc) usage(("missing value for " + a).c_str());
      return argv[++i];
    };
    uint64_t x = 0;
    if (a == "--log-seg" || a == "-l") {
      if (!parse_u64(val(), x)) usage("bad --log-seg");
      fl.l = (unsigned)std::min<uint64_t>(x, 1000);
    } else if (a == "--first" || a == "-f") {
      if (!parse_u64(val(), fl.f)) usage("bad --first");
      fl.have_f = true;
    } else if (a == "--midpoint-exp" || a == "-e") {
      if (!parse_u64(val(), x)) usage("bad --midpoint-exp");
      fl.e = (unsigned)std::min<uint64_t>(x, 1000);
      fl.have_e = true;
    } else if (a == "--segments" || a == "-n") {
      if (!parse_u64(val(), fl.n)) usage("bad --segments");
      fl.have_n = true;
    } else if (a == "--test-mode") {
      fl.test_mode = true;
    } else if (a == "--allow-overlap") {
      fl.allow_overlap = true;
    } else if (a == "--count-only") {
      fl.count_only = true;
    } else if (a == "--out-dir") {
      fl.out_dir = val();
    } else if (a == "--max-base-pairs") {
      if (!parse_u64(val(), fl.max_base_pairs)) usage("bad --max-base-pairs");
    } else if (a == "--exps") {
      std::string s = val();
      size_t p = 0;
      while (p <= s.size()) {
        const size_t q = s.find(',', p);
        const std::string tok = s.substr(p, q == std::string::npos ? std::string::npos : q - p);
        if (!parse_u64(tok.c_str(), x)) usage("bad --exps");
        fl.exps.push_back((unsigned)x);
        if (q == std::string::npos) break;
        p = q + 1;
      }
    } else if (a == "--csv") {
      fl.csv = val();
    } else if (a == "--reps") {
      if (!parse_u64(val(), x)) usage("bad --reps");
      fl.reps = (unsigned)std::max<uint64_t>(1, x);
    } else if (a == "--machine") {
      fl.machine = val();
    } else if (a == "--gpus") {
      if (!parse_u64(val(), x) || x < 1 || x > 4096) usage("bad --gpus");
      fl.devices.clear();
      for (uint64_t g = 0; g < x; ++g) fl.devices.push_back((int)g);
    } else if (a == "--devices") {
      std::string s = val();
      fl.devices.clear();
      size_t p = 0;
      while (p <= s.size()) {
        const size_t q = s.find(',', p);
        const std::string tok = s.substr(p, q == std::string::npos ? std::string::npos : q - p);
        if (!parse_u64(tok.c_str(), x) || x > 4096) usage("bad --devices");
        fl.devices.push_back((int)x);
        if (q == std::string::npos) break;
        p = q + 1;
      }
    } else if (a == "--kernels") {
      val();  // no GPU counterpart (no multi-backend dispatch)
    } else {
      usage(("unknown option " + a).c_str());
    }
  }
  if (fl.cmd == "bench") {
    if (fl.exps.empty()) usage("--exps is required");
  } else {
    if (!fl.have_n) usage("--segments is required");
    if (fl.have_f && fl.have_e) usage("--first excludes --midpoint-exp");
  }
  return fl;
}

int exit_code(int rc) {  // is_param_error, erato.cpp:21-33
  if (rc >= ERATO_GPU_L_OUT_OF_RANGE && rc <= ERATO_GPU_INDEX_OUT_OF_RANGE) return 1;
  return 2;
}

int report(int rc) {
  std::fprintf(stderr, "error: %s\n", erato_gpu_last_error());
  return exit_code(rc);
}

uint64_t mulmod(uint64_t a, uint64_t b, uint64_t m) { return (uint64_t)((unsigned __int128)a * b % m); }

bool miller_rabin(uint64_t n) {  // bases 2..37: exact for 64-bit (tests/support.hpp:28-54)
  if (n < 2) return false;
  static const uint64_t bases[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  for (uint64_t p : bases) {
    if (n == p) return true;
    if (n % p == 0) return false;
  }
  uint64_t d = n - 1;
  unsigned s = 0;
  while ((d & 1) == 0) {
    d >>= 1;
    ++s;
  }
  for (uint64_t a : bases) {
    uint64_t x = 1, b = a % n, e = d;
    while (e) {
      if (e & 1) x = mulmod(x, b, n);
      b = mulmod(b, b, n);
      e >>= 1;
    }
    if (x == 1 || x == n - 1) continue;
    bool comp = true;
    for (unsigned r = 1; r < s; ++r) {
      x = mulmod(x, x, n);
      if (x == n - 1) {
        comp = false;
        break;
      }
    }
    if (comp) return false;
  }
  return true;
}

void print_stats(const erato_gpu_stats& st) {  // print_stats, erato.cpp:75-83
  std::printf("primes    %" PRIu64 "\n", st.prime_count);
  std::printf("segments  %" PRIu64 "\n", st.segments);
  std::printf("init      %.3fs\n", st.init_s);
  std::printf("masks     %.3fs\n", st.masks_s);
  std::printf("medium    %.3fs\n", st.small_s > st.masks_s ? st.small_s - st.masks_s : 0.0);
  std::printf("large     %.3fs\n", st.large_s);
  std::printf("output    %.3fs\n", st.output_s);
}

}  // namespace

int main(int argc, char** argv) {
  const Flags fl = parse(argc, argv);
  const unsigned flags = (fl.test_mode ? ERATO_GPU_TEST_MODE : 0u) | (fl.allow_overlap ? ERATO_GPU_ALLOW_OVERLAP : 0u);
  if (fl.cmd == "bench") {  // bench_run, src/bench.cpp:20-50
    erato_gpu_ctx* ctx = nullptr;
    if (int rc = erato_gpu_create(0, &ctx)) return report(rc);
    std::FILE* csv = fl.csv.empty() ? nullptr : std::fopen(fl.csv.c_str(), "w");
    if (!fl.csv.empty() && !csv) {
      std::fprintf(stderr, "error: IO_ERROR: cannot open %s\n", fl.csv.c_str());
      return 2;
    }
    if (csv) std::fprintf(csv, "e,seconds,l\n");
    std::printf("machine %s, l=%u, interval 2^30 bits\n", fl.machine.c_str(), fl.l);
    for (unsigned e : fl.exps) {
      if (fl.l > 30) {
        std::printf("e=%-3u failed: L_OUT_OF_RANGE\n", e);
        continue;
      }
      const uint64_t n = uint64_t{1} << (30 - fl.l);
      uint64_t f = 0, cnt = 0;
      if (erato_gpu_f_from_midpoint(e, fl.l, n, flags, &f) != 0) {
        std::printf("e=%-3u failed: %s\n", e, erato_gpu_last_error());
        continue;
      }
      auto timed = [&] {
        const auto t0 = std::chrono::steady_clock::now();
        const int rc = erato_gpu_count(ctx, fl.l, f, n, flags, &cnt, nullptr);
        return rc ? -1.0 : std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      };
      timed();  // warm-up
      std::vector<double> ts;
      for (unsigned r = 0; r < fl.reps; ++r) ts.push_back(timed());
      std::sort(ts.begin(), ts.end());
      const double med = ts[ts.size() / 2];
      if (med < 0) {
        std::printf("e=%-3u failed: %s\n", e, erato_gpu_last_error());
        continue;
      }
      std::printf("e=%-3u %8.6fs\n", e, med);
      if (csv) std::fprintf(csv, "%u,%.6f,%u\n", e, med, fl.l);
    }
    if (csv) std::fclose(csv);
    erato_gpu_destroy(ctx);
    return 0;
  }
  // sieve / verify: ParamFlags::resolve (erato.cpp:53-62)
  uint64_t f = fl.f;
  if (fl.have_e) {
    if (int rc = erato_gpu_f_from_midpoint(fl.e, fl.l, fl.n, flags, &f)) return report(rc);
  } else if (!fl.have_f) {
    std::fprintf(stderr, "error: F_ZERO_OR_OVERLAP: need --first or --midpoint-exp\n");
    return 1;
  }
  uint64_t u = 0, v = 0;
  if (int rc = erato_gpu_validate(fl.l, f, fl.n, flags, &u, &v)) return report(rc);
  erato_gpu_stats st{};
  int rc = 0;
  // per-phase device times for print_stats (masks / medium / large)
  const unsigned run_flags = flags | ERATO_GPU_PHASE_TIMING;
  if (fl.cmd == "sieve" && fl.devices.size() > 1) {  // range shards over several GPUs
    erato_gpu_multi* m = nullptr;
    if ((rc = erato_gpu_multi_create((int)fl.devices.size(), fl.devices.data(), &m))) return report(rc);
    uint64_t cnt = 0;
    if (fl.count_only) {
      rc = erato_gpu_multi_count(m, fl.l, f, fl.n, run_flags, &cnt, &st);
      if (!rc) print_stats(st);
    } else {
      char path[4096];
      rc = erato_gpu_multi_write_table(m, fl.out_dir.c_str(), fl.l, f, fl.n, run_flags, path, sizeof(path), &cnt, &st);
      if (!rc) {
        print_stats(st);
        std::printf("table     %s (%" PRIu64 " bytes)\n", path, (fl.n << fl.l) / 8);
      }
    }
    erato_gpu_multi_destroy(m);
    if (rc) return report(rc);
    return 0;
  }
  erato_gpu_ctx* ctx = nullptr;
  if ((rc = erato_gpu_create(fl.devices.empty() ? 0 : fl.devices[0], &ctx))) return report(rc);
  erato_gpu_set_max_base_pairs(ctx, fl.max_base_pairs);
  if (fl.cmd == "sieve") {
    if (fl.count_only) {
      uint64_t cnt = 0;
      rc = erato_gpu_count(ctx, fl.l, f, fl.n, run_flags, &cnt, &st);
      if (!rc) print_stats(st);
    } else {
      char path[4096];
      rc = erato_gpu_write_table(ctx, fl.out_dir.c_str(), fl.l, f, fl.n, f, fl.n, run_flags, path, sizeof(path), &st);
      if (!rc) {
        print_stats(st);
        std::printf("table     %s (%" PRIu64 " bytes)\n", path, (fl.n << fl.l) / 8);
      }
    }
  } else {  // verify
    const uint64_t bits = fl.n << fl.l;
    std::vector<uint8_t> table(bits / 8);
    rc = erato_gpu_sieve_to_host(ctx, fl.l, f, fl.n, flags, table.data(), table.size(), &st);
    if (!rc) {
      std::mt19937_64 rng(1234);
      const bool all = bits <= (uint64_t{1} << 22);
      const uint64_t checks = all ? bits : 1 << 20;
      uint64_t bad = 0;
      for (uint64_t k = 0; k < checks; ++k) {
        const uint64_t j = all ? k : rng() % bits;
        const uint64_t num = u + 2 * j;
        const bool composite = (table[j >> 3] >> (j & 7)) & 1;
        const bool expect_comp = num == 1 ? false : !miller_rabin(num);
        if (composite != expect_comp) ++bad;
      }
      if (bad == 0) {
        std::printf("PASS  [%" PRIu64 ", %" PRIu64 "] %s (%zu bytes, %" PRIu64 " bits checked by Miller-Rabin)\n", u,
                    v, all ? "matches" : "sample matches", table.size(), checks);
      } else {
        std::printf("FAIL  %" PRIu64 " of %" PRIu64 " checked bits differ\n", bad, checks);
        erato_gpu_destroy(ctx);
        return 2;
      }
    }
  }
  erato_gpu_destroy(ctx);
  if (rc) return report(rc);
  return 0;
}
