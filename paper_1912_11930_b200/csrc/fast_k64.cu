// fast_k64.cu — tuned fused kernels for k = 64 lanes (generated layout, see fast_table.cuh).
#include "fast_table.cuh"

namespace bkg {

template <>
bool fast_lookup_k<64>(int p, bool global, FastTable* t) {
  switch (p) {
    case 1: return fill_p<64, 1>(global, t);
    case 2: return fill_p<64, 2>(global, t);
    case 4: return fill_p<64, 4>(global, t);
    case 8: return fill_p<64, 8>(global, t);
    case 16: return fill_p<64, 16>(global, t);
    default: return false;
  }
}

}  // namespace bkg
