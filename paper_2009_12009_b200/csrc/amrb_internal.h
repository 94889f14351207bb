// Internal helpers shared by the libamrb translation units.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/amrb.h"

namespace amrb {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void set_last_error(const std::string& msg);

// Run fn, translating exceptions into a status code + thread-local message.
template <class F>
int guarded(F&& fn) {
  try {
    fn();
    return AMRB_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("out of host memory");
    return AMRB_ENOMEM;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return AMRB_EINVAL;
  }
}

// One congruent copy: src cells [lo, hi] of box `src` land at [lo, hi] + shift
// of box `dst`.  3-D padded.
struct Record {
  int src, dst;
  int lo[3], hi[3];
  int shift[3];
  int64_t cells() const {
    return (int64_t)(hi[0] - lo[0] + 1) * (hi[1] - lo[1] + 1) * (hi[2] - lo[2] + 1);
  }
};

struct Plan {
  int dim = 3;
  std::vector<Record> recs;
  int64_t cells() const;
};

}  // namespace amrb
