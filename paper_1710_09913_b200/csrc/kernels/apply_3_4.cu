// apply_3_4.cu -- instantiations of the apply kernels for d = 3, p = 4: one
// translation unit per (d, p) so nvcc compiles the straight-line bodies in parallel.
#include "apply_impl.cuh"

namespace dogip {

cudaError_t launch_apply_3_4(const ApplyArgs& a) { return launch_form<3, 4>(a); }

bool ref_info_3_4(int form, int store, RefInfo& r) {
    if (form == 0 && store == 0) { fill_info<3, 4, 0, 0>(r); return true; }
    if (form == 1 && store == 0) { fill_info<3, 4, 1, 0>(r); return true; }
    if (form == 1 && store == 1) { fill_info<3, 4, 1, 1>(r); return true; }
    if (form == 0 && store == 5) { fill_info<3, 4, 0, 5>(r); return true; }
    if (full_sym_body<3, 4>() && form == 0 && store == 6) { fill_info<3, 4, 0, 6>(r); return true; }   // FULL, symmetry-adapted body
    return false;
}

}  // namespace dogip
