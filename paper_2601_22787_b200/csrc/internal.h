// internal.h — host-side helpers shared between translation units of libentquant (not
// part of the C ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/entquant.h"

namespace eq {
// ‖W‖₁ of n bf16 values in f64, deterministic two-stage reduction; part: scratch of
// l1_scratch_bytes(n) bytes; out: one device double.
uint64_t l1_scratch_bytes(int64_t n);
eq_status l1_device(const uint16_t* W, int64_t n, double* out, void* part, cudaStream_t st);
}  // namespace eq
