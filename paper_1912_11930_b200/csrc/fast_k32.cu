// fast_k32.cu — tuned fused kernels for k = 32 lanes (generated layout, see fast_table.cuh).
#include "fast_table.cuh"

namespace bkg {

template <>
bool fast_lookup_k<32>(int p, bool global, FastTable* t) {
  switch (p) {
    case 1: return fill_p<32, 1>(global, t);
    case 2: return fill_p<32, 2>(global, t);
    case 4: return fill_p<32, 4>(global, t);
    case 8: return fill_p<32, 8>(global, t);
    case 16: return fill_p<32, 16>(global, t);
    default: return false;
  }
}

}  // namespace bkg
