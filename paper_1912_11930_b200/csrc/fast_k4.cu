// fast_k4.cu — tuned fused kernels for k = 4 lanes (generated layout, see fast_table.cuh).
#include "fast_table.cuh"

namespace bkg {

template <>
bool fast_lookup_k<4>(int p, bool global, FastTable* t) {
  switch (p) {
    case 1: return fill_p<4, 1>(global, t);
    case 2: return fill_p<4, 2>(global, t);
    case 4: return fill_p<4, 4>(global, t);
    default: return false;
  }
}

}  // namespace bkg
