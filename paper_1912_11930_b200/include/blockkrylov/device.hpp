// blockkrylov/device.hpp — the process-wide device context behind the
// drop-in API.  The reference is a CPU library with no context object; here
// every hot-path call runs on one lazily created bkg_ctx (device from
// $BKG_DEVICE, default 0; numerics from $BKG_NUMERICS = fast|exact).
#pragma once

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "bkg.h"
#include "blockkrylov/errors.hpp"

namespace blockkrylov {
namespace gpu {

enum class Numerics { fast = BKG_NUMERICS_FAST, exact = BKG_NUMERICS_EXACT };

namespace detail {
struct Holder {
  bkg_ctx* ctx = nullptr;
  std::mutex mu;
  ~Holder() {
    if (ctx) bkg_ctx_destroy(ctx);
  }
};
inline Holder& holder() {
  static Holder h;
  return h;
}
}  // namespace detail

/// The shared context (created on first use).
inline bkg_ctx* context() {
  auto& h = detail::holder();
  std::lock_guard<std::mutex> lock(h.mu);
  if (!h.ctx) {
    const char* dev = std::getenv("BKG_DEVICE");
    blockkrylov::detail::check(bkg_ctx_create(dev ? std::atoi(dev) : 0, &h.ctx));
    const char* num = std::getenv("BKG_NUMERICS");
    if (num && std::strcmp(num, "exact") == 0)
      blockkrylov::detail::check(bkg_ctx_set_numerics(h.ctx, BKG_NUMERICS_EXACT));
  }
  return h.ctx;
}

/// exact: bit-identical to the reference CPU build; fast: fused kernels.
inline void set_numerics(Numerics n) {
  blockkrylov::detail::check(bkg_ctx_set_numerics(context(), static_cast<int>(n)));
}

inline Numerics numerics() {
  int v = 0;
  blockkrylov::detail::check(bkg_ctx_get_numerics(context(), &v));
  return static_cast<Numerics>(v);
}

}  // namespace gpu
}  // namespace blockkrylov
