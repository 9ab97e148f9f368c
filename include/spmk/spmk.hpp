// spmk/spmk.hpp — umbrella include, drop-in for
// /root/reference/proj/include/spmk/spmk.hpp:1-11: bench, corpus
// (NamedMatrix, make_dense), csr, error, io, kernels, rmat, selector, plus the
// resident-handle API (device.hpp).  reduction.hpp's lane model stays test
// infrastructure (oracle/).
#pragma once

#include "spmk/bench.hpp"
#include "spmk/corpus.hpp"
#include "spmk/csr.hpp"
#include "spmk/device.hpp"
#include "spmk/error.hpp"
#include "spmk/io.hpp"
#include "spmk/kernels.hpp"
#include "spmk/rmat.hpp"
#include "spmk/selector.hpp"
