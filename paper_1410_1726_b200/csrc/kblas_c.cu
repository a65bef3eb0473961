// kblas_c.cu — single-complex precision: the C entry points of include/kblas_b200.h
// for this precision and every kernel instantiation they need.  One
// translation unit per precision so the library builds in parallel.
#include "kblas_entry_macros.cuh"

using namespace kb;
using namespace kbi;

namespace kbi {
KBI_ENTRY_TEMPLATES(, float2)
}  // namespace kbi

extern "C" {

KB_GEMV(c, cuFloatComplex)
KB_SYMV(chemv, cuFloatComplex, true)
KB_SYMV(csymv, cuFloatComplex, false)

}  // extern "C"
