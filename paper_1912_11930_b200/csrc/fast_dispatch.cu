// fast_dispatch.cu — (k, p) -> tuned kernel table.
#include "fast_table.cuh"

namespace bkg {

bool fast_lookup(int k, int p, bool global, FastTable* t) {
  switch (k) {
    case 4: return fast_lookup_k<4>(p, global, t);
    case 8: return fast_lookup_k<8>(p, global, t);
    case 16: return fast_lookup_k<16>(p, global, t);
    case 32: return fast_lookup_k<32>(p, global, t);
    case 64: return fast_lookup_k<64>(p, global, t);
    case 128: return fast_lookup_k<128>(p, global, t);
    default: return false;
  }
}

}  // namespace bkg
