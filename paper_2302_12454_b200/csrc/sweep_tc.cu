// sweep_tc.cu -- fused tcgen05 sweep engine (work in progress: not yet
// enabled; tc_supported() returns false until the kernel passes parity).
#include "sweep_tc.h"

namespace ssqa_engine {

bool tc_supported(int, int) { return false; }
int tc_run(ssqa_batch_s*, const ScanArgs&) { return SSQA_EUNSUP; }
int tc_sweep(ssqa_batch_s*, double, double) { return SSQA_EUNSUP; }
const char* tc_last_error() { return "tcgen05 engine not available"; }

}  // namespace ssqa_engine
