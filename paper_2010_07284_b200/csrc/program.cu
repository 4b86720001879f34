// program.cu -- placeholder; the device-resident DAG executor lands next.
#include "slcs_internal.h"
extern "C" {
int slcs_program_create(slcs_ctx*, int, const char* const*, const double*, const char* const*,
                        const int*, const int*, slcs_program**) { return SLCS_ERR_RUN; }
int slcs_program_destroy(slcs_program*) { return SLCS_OK; }
int slcs_program_bind(slcs_program*, const char*, const slcs_image*) { return SLCS_ERR_RUN; }
int slcs_program_run(slcs_program*, int) { return SLCS_ERR_RUN; }
int slcs_program_result(slcs_program*, int, int*, slcs_image**, double*) { return SLCS_ERR_RUN; }
int slcs_program_launches(slcs_program*, int*) { return SLCS_ERR_RUN; }
const char* slcs_program_plan(slcs_program*) { return ""; }
}
