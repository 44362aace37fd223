// nfs_tc.cu -- tcgen05 tensor-core operator path (placeholder until the kernel lands).
#include "nfs_tc.cuh"

namespace nfs {

struct TcPlan {};
static thread_local std::string g_tc_err;

TcPlan* tc_create(int64_t, int64_t, int, int, int, std::string* why) {
  if (why) *why = "tcgen05 path not built in this revision";
  return nullptr;
}
void tc_destroy(TcPlan* t) { delete t; }
const char* tc_describe(TcPlan*) { return ""; }
const char* tc_last_error() { return g_tc_err.c_str(); }
int tc_set_tables(TcPlan*, const void*, const void*, cudaStream_t) { return 1; }
int tc_set_sens(TcPlan*, const void*, int, cudaStream_t) { return 1; }
int tc_forward(TcPlan*, const double2*, void*, const int*, cudaStream_t) { return 1; }
int tc_adjoint(TcPlan*, const void*, double2*, const int*, cudaStream_t) { return 1; }
int tc_forward_parts(TcPlan*, const double2*, void*, const int*, cudaStream_t, int) { return 1; }
int tc_adjoint_parts(TcPlan*, const void*, double2*, const int*, cudaStream_t, int) { return 1; }
int tc_launches_per_apply(TcPlan*) { return 0; }

}  // namespace nfs
