// nqueens/nqueens.hpp — umbrella header of the drop-in API (reference nqueens.hpp).
// Link with libnqb200.so (paper_2511_12009_b200/libnqb200.so): counting runs on the
// sm_100a kernels; frontier generation, partitions and log formatting run on the host.
#pragma once

#include "nqueens/bitboard.hpp"
#include "nqueens/errors.hpp"
#include "nqueens/runner.hpp"
#include "nqueens/scheduler.hpp"
#include "nqueens/solver.hpp"
#include "nqueens/stack_config.hpp"
#include "nqueens/subproblems.hpp"
