// fast_k128.cu — tuned fused kernels for k = 128 lanes (the paper's experiment width) (generated layout, see fast_table.cuh).
#include "fast_table.cuh"

namespace bkg {

template <>
bool fast_lookup_k<128>(int p, bool global, FastTable* t) {
  switch (p) {
    case 1: return fill_p<128, 1>(global, t);
    case 2: return fill_p<128, 2>(global, t);
    case 4: return fill_p<128, 4>(global, t);
    case 8: return fill_p<128, 8>(global, t);
    case 16: return fill_p<128, 16>(global, t);
    default: return false;
  }
}

}  // namespace bkg
