// fast_k8.cu — tuned fused kernels for k = 8 lanes (generated layout, see fast_table.cuh).
#include "fast_table.cuh"

namespace bkg {

template <>
bool fast_lookup_k<8>(int p, bool global, FastTable* t) {
  switch (p) {
    case 1: return fill_p<8, 1>(global, t);
    case 2: return fill_p<8, 2>(global, t);
    case 4: return fill_p<8, 4>(global, t);
    case 8: return fill_p<8, 8>(global, t);
    default: return false;
  }
}

}  // namespace bkg
