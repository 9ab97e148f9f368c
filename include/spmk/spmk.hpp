// spmk/spmk.hpp — umbrella include, drop-in for
// /root/reference/proj/include/spmk/spmk.hpp:1-11 (hot-path headers only:
// csr, kernels, selector, error, io; plus the resident-handle API).
#pragma once

#include "spmk/csr.hpp"
#include "spmk/device.hpp"
#include "spmk/error.hpp"
#include "spmk/io.hpp"
#include "spmk/kernels.hpp"
#include "spmk/selector.hpp"
