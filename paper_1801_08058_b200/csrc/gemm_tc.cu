// tcgen05 tensor-core Dot (3xTF32) -- placeholder until the kernel lands.
#include <cuda_runtime.h>
#include "gfb200.h"
extern "C" const void* gfb_tc_kernel_ptr(int kind) { (void)kind; return nullptr; }
