// TEST INFRASTRUCTURE: links the reference's own callers of
// kvadmit::run_simulation (the acceptance gate, acceptance.cpp:70-80, and the
// kva_* scenario ABI through execute_run, experiment.cpp:159-182) against the
// B200 engine. The adapter itself is the product header
// include/kvadmit_gpu.hpp; this translation unit only instantiates its
// --wrap entry point (oracle/Makefile: acceptance_gpu, libkvadmit_gpu.so).
#define KVGPU_DEFINE_RUN_SIMULATION_WRAP
#include "kvadmit_gpu.hpp"
