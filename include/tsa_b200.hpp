// tsa_b200.hpp -- C++ drop-in for the reference operator API on B200.
//
// The reference (`tsa` library, /root/reference/proj) declares its operators in
// tsa/token_coverage.hpp and tsa/attention.hpp.  paper_2602_03216_b200/cpp/
// tsa_b200_adapter.cpp DEFINES those same functions -- same namespace, names,
// signatures, error types and messages -- on top of the C ABI in tsa_b200.h:
//
//   tsa::score_tokens            token_coverage.hpp:32  -> tsa_score (f32 reference-order)
//   tsa::aggregate_scores        token_coverage.hpp:36  -> tsa_aggregate_scores + tsa_check
//   tsa::coverage_budget         token_coverage.hpp:42  -> tsa_coverage_budget
//   tsa::fixed_budget            token_coverage.hpp:45  -> host arithmetic (as the reference)
//   tsa::select_tokens           token_coverage.hpp:50  -> tsa_select
//   tsa::dense_causal_attention  attention.hpp:31       -> tsa_dense_attention
//   tsa::token_sparse_attention  attention.hpp:44       -> tsa_token_sparse_attention
//                                                          (custom `inner`: tsa_gather ->
//                                                           inner per head -> tsa_scatter_rows)
//
// So a reference build switches to the GPU by linking tsa_b200_adapter.o and
// libtsa_b200.so in place of token_coverage.o and the two operator
// definitions of attention.o (masked_sparse_oracle, the reference's ground
// truth, stays on the CPU).  INTEGRATION.md shows the CMake change; the
// reference's own test_attention / test_coverage suites are built this way
// and run on the B200 (tests/test_reference_suites.py).
//
// Extra knobs (not in the reference API):
#pragma once

#include "tsa_b200.h"

namespace tsa {
namespace b200 {

// CUDA device the adapter uses (default 0).
void set_device(int device);

// Scoring arithmetic for f32 inputs: TSA_SCORING_REFERENCE (default; the
// reference's f32 operation order) -- see tsa_b200.h.
void set_scoring(int scoring);

}  // namespace b200
}  // namespace tsa
