// kblas_z.cu — double-complex precision: the C entry points of include/kblas_b200.h
// for this precision and every kernel instantiation they need.  One
// translation unit per precision so the library builds in parallel.
#include "kblas_entry_macros.cuh"

using namespace kb;
using namespace kbi;

namespace kbi {
KBI_ENTRY_TEMPLATES(, double2)
}  // namespace kbi

extern "C" {

KB_GEMV(z, cuDoubleComplex)
KB_SYMV(zhemv, cuDoubleComplex, true)
KB_SYMV(zsymv, cuDoubleComplex, false)

}  // extern "C"
