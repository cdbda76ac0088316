// gpu_binding.hpp — the erato-side binding of the B200 sieve, as a maintainer
// would add it to the reference.  Compiled and run by the
// tests against the reference's own headers and run_sieve
// (tests/integration/binding_main.cpp, oracle/Makefile target `binding`).
//
// erato::run_sieve_gpu has the contract of erato::run_sieve
// (/root/reference/proj/include/erato/driver.hpp:91, src/driver.cpp:83-120):
// segments reach the sink in order t = 0..n-1 through a SegmentBuffer that is
// valid only during on_segment, then finish(); NullSink stays on the device
// (only the count comes back).  Errors come back as erato::Error with the
// reference's errc (the C ABI returns errc ordinal + 1).
#pragma once
#include <algorithm>
#include <cstring>
#include <exception>
#include <vector>

#include "erato/driver.hpp"
#include "erato_gpu.h"

namespace erato {
namespace gpu_detail {

inline void check(int rc) {
  if (rc == 0) return;
  // 1..10: erato::errc ordinals + 1 (params.hpp:18-29); the rest are GPU runtime errors
  throw Error(rc <= 10 ? errc(rc - 1) : errc::io_error, erato_gpu_last_error());
}

inline erato_gpu_ctx* context() {
  static erato_gpu_ctx* ctx = [] {
    erato_gpu_ctx* c = nullptr;
    check(erato_gpu_create(0, &c));
    return c;
  }();
  return ctx;
}

// Re-cuts the ordered wave slices of erato_gpu_run_to_sink into the
// reference's segments.  Exceptions thrown by the sink must not cross the C
// ABI: they are kept and rethrown after the run.
struct SegmentFeed {
  SegmentSink* sink;
  const SieveParams* p;
  SegmentBuffer seg;
  std::vector<uint8_t> carry;
  uint64_t t = 0;
  std::exception_ptr error;
};

inline int feed(void* user, const uint8_t* bytes, uint64_t, uint64_t nbytes) {
  auto* f = static_cast<SegmentFeed*>(user);
  try {
    const uint64_t sb = f->p->segment_bytes();
    while (nbytes) {
      const uint64_t take = std::min<uint64_t>(nbytes, sb - f->carry.size());
      f->carry.insert(f->carry.end(), bytes, bytes + take);
      bytes += take;
      nbytes -= take;
      if (f->carry.size() == sb) {
        f->seg.clear(f->t);
        std::memcpy(f->seg.words(), f->carry.data(), sb);  // LSB-first bytes == little-endian words
        f->sink->on_segment(f->seg, f->t, *f->p);
        ++f->t;
        f->carry.clear();
      }
    }
    return 0;
  } catch (...) {
    f->error = std::current_exception();
    return 1;
  }
}

}  // namespace gpu_detail

inline RunStats run_sieve_gpu(const SieveParams& p, SegmentSink& sink, const RunOptions& opt = {}) {
  erato_gpu_ctx* ctx = gpu_detail::context();
  gpu_detail::check(erato_gpu_set_max_base_pairs(ctx, opt.max_base_pairs));  // RunOptions::max_base_pairs
  const unsigned flags = p.l < kMinLogSeg ? ERATO_GPU_TEST_MODE : 0u;      // params validated in test mode
  erato_gpu_stats st{};
  if (dynamic_cast<NullSink*>(&sink)) {
    uint64_t count = 0;
    gpu_detail::check(erato_gpu_count(ctx, p.l, p.f, p.n, flags, &count, &st));
  } else {  // every other sink sees the reference's segments, in order
    gpu_detail::SegmentFeed f{&sink, &p, SegmentBuffer(p.l), {}, 0, nullptr};
    const int rc = erato_gpu_run_to_sink(ctx, p.l, p.f, p.n, flags, gpu_detail::feed, &f, &st);
    if (f.error) std::rethrow_exception(f.error);
    gpu_detail::check(rc);
  }
  sink.finish(p);
  RunStats rs;
  rs.prime_count = st.prime_count;
  rs.segments = p.n;
  rs.init_s = st.init_s;
  rs.masks_s = st.masks_s;
  rs.medium_s = st.small_s - st.masks_s;
  rs.large_s = st.large_s;
  rs.output_s = st.output_s;
  return rs;
}

}  // namespace erato
