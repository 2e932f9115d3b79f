// apply_3_2.cu -- instantiations of the apply kernels for d = 3, p = 2: one
// translation unit per (d, p) so nvcc compiles the straight-line bodies in parallel.
#include "apply_impl.cuh"

namespace dogip {

cudaError_t launch_apply_3_2(const ApplyArgs& a) { return launch_form<3, 2>(a); }

bool ref_info_3_2(int form, int store, RefInfo& r) {
    if (form == 0 && store == 0) { fill_info<3, 2, 0, 0>(r); return true; }
    if (form == 1 && store == 0) { fill_info<3, 2, 1, 0>(r); return true; }
    if (form == 1 && store == 1) { fill_info<3, 2, 1, 1>(r); return true; }
    if (form == 0 && store == 5) { fill_info<3, 2, 0, 5>(r); return true; }
    return false;
}

}  // namespace dogip
