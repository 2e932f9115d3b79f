// apply.cu -- dispatch of the apply kernels (kernels/apply_impl.cuh, instantiated per
// (d, p) in apply_<d>_<p>.cu) and the host-side reference-element constants.
#include <cuda_runtime.h>

#include "apply.cuh"

namespace dogip {

cudaError_t launch_apply_2_1(const ApplyArgs& a);
bool ref_info_2_1(int form, int store, RefInfo& r);
cudaError_t launch_apply_2_2(const ApplyArgs& a);
bool ref_info_2_2(int form, int store, RefInfo& r);
cudaError_t launch_apply_2_3(const ApplyArgs& a);
bool ref_info_2_3(int form, int store, RefInfo& r);
cudaError_t launch_apply_2_4(const ApplyArgs& a);
bool ref_info_2_4(int form, int store, RefInfo& r);
cudaError_t launch_apply_3_1(const ApplyArgs& a);
bool ref_info_3_1(int form, int store, RefInfo& r);
cudaError_t launch_apply_3_2(const ApplyArgs& a);
bool ref_info_3_2(int form, int store, RefInfo& r);
cudaError_t launch_apply_3_3(const ApplyArgs& a);
bool ref_info_3_3(int form, int store, RefInfo& r);
cudaError_t launch_apply_3_4(const ApplyArgs& a);
bool ref_info_3_4(int form, int store, RefInfo& r);

std::atomic<long long> g_launches{0};

cudaError_t launch_apply(const ApplyArgs& a) {
#define DOGIP_CASE(D, P) \
    if (a.d == D && a.p == P) return launch_apply_##D##_##P(a);
    DOGIP_CASE(2, 1) DOGIP_CASE(2, 2) DOGIP_CASE(2, 3) DOGIP_CASE(2, 4)
    DOGIP_CASE(3, 1) DOGIP_CASE(3, 2) DOGIP_CASE(3, 3) DOGIP_CASE(3, 4)
#undef DOGIP_CASE
    return cudaErrorInvalidValue;
}

bool ref_info(int d, int p, int form, int store, RefInfo& r) {
#define DOGIP_CASE(D, P) \
    if (d == D && p == P) return ref_info_##D##_##P(form, store, r);
    DOGIP_CASE(2, 1) DOGIP_CASE(2, 2) DOGIP_CASE(2, 3) DOGIP_CASE(2, 4)
    DOGIP_CASE(3, 1) DOGIP_CASE(3, 2) DOGIP_CASE(3, 3) DOGIP_CASE(3, 4)
#undef DOGIP_CASE
    return false;
}

}  // namespace dogip
