// SA / DBS incremental pixel search (algorithms.py:208-467) — placeholder
// entry points; the persistent search kernel lands in the next milestone.
#include "runtime.cuh"

using namespace cgh;

extern "C" {

int cgh_sa_run(const cgh_problem*, const cgh_sa_params*, const double*, const uint8_t*, const double*, void*, int64_t*,
               double*, int64_t, cgh_report*, const cgh_callbacks*) {
    return fail(CGH_ERR_UNSUPPORTED, "SA not built yet");
}
int cgh_dbs_run(const cgh_problem*, const cgh_dbs_params*, const double*, const uint8_t*, const double*, void*, int64_t*,
                double*, int64_t, cgh_report*, const cgh_callbacks*) {
    return fail(CGH_ERR_UNSUPPORTED, "DBS not built yet");
}
int cgh_delta_error(int32_t, const double*, const double*, const double*, const double*, const int32_t*, const int32_t*,
                    int64_t, int32_t, int32_t, double, double, double*) {
    return fail(CGH_ERR_UNSUPPORTED, "not built yet");
}
int cgh_commit_update(int32_t, double*, const double*, const double*, const int32_t*, const int32_t*, int64_t, int32_t,
                      int32_t, double, double) {
    return fail(CGH_ERR_UNSUPPORTED, "not built yet");
}
int cgh_best_delta(int32_t, const double*, const double*, const double*, const double*, const int32_t*, const int32_t*,
                   int64_t, int32_t, int32_t, const double*, int64_t, int64_t*, double*) {
    return fail(CGH_ERR_UNSUPPORTED, "not built yet");
}
}
