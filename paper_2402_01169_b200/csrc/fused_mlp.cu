// fused_mlp.cu — instantiations of the one-kernel MLP (fused_mlp.cuh).  Compiled
// once per -DFUSED_PART=k (parallel build), each object holding the 16 variants whose
// flags have (flags >> 4) == k: k = 0..3 (flags 0..63: GELU, hidden zero point, FC1 bias,
// fp64 LN, small-K conversion, taps); the host picks one by flags.
#include <utility>

#include "fused_mlp.cuh"

#ifndef FUSED_PART
#error "compile with -DFUSED_PART=<0..3>"
#endif

namespace swinmlp {

using FusedFn = void (*)(CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, FusedArgs);

namespace {   // internal linkage: each part's table is its own (no COMDAT folding across parts)
template <int... Is>
FusedFn pick_fused(int f, std::integer_sequence<int, Is...>) {
    static const FusedFn table[] = {fused_mlp_kernel<FUSED_PART * 16 + Is>...};
    return table[f & 15];
}
}  // namespace

#define FUSED_PART_FN2(k) fused_kernel_part##k
#define FUSED_PART_FN(k) FUSED_PART_FN2(k)
FusedFn FUSED_PART_FN(FUSED_PART)(int flags) { return pick_fused(flags, std::make_integer_sequence<int, 16>{}); }

}  // namespace swinmlp
