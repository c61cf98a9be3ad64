// ab2_pipeline.cu -- out-of-core run (Alg. 2, scheduler.hpp:72-168) as a multi-stream pipeline.
#include "ab2_internal.h"

extern "C" int aires_b200_run(const aires_b200_matrix* a, const aires_b200_matrix* b,
                              const aires_b200_run_config* cfg, aires_b200_output* c,
                              aires_b200_run_report* report) {
  (void)a; (void)b; (void)cfg; (void)c; (void)report;
  return AIRES_B200_UNSUPPORTED_FORMAT;
}
