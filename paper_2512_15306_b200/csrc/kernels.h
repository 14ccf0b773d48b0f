// Internal include: the public C-ABI (include/qtrain_b200.h) plus the
// epilogue enum shared by the GEMM kernels.
#pragma once
#include "../../include/qtrain_b200.h"
