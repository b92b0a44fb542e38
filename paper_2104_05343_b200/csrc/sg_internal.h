// Shared host-side helpers of libsg (error slot, device queries).
#pragma once
#include <cuda_runtime.h>

namespace sg {
int set_error(int code, const char* msg);
void clear_error();
void count_launch();  // every kernel this library launches (bench gpu_launches)
}  // namespace sg

extern "C" int sg_device_sm_count(void);
