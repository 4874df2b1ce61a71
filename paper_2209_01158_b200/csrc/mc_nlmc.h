// mc_nlmc.h — what the NLMC builder (mc_nlmc.cu) reads from a fine context (mc_api.cu).
// Not part of the public ABI.
#pragma once
#include <cstdint>
#include <vector>

#include "../../include/mc.h"

namespace mc {

// The fine operator of a context split as A = D + Q + W, in the
// caller's numbering, continua concatenated (global fine DOF g = off[alpha] + i).
struct FineSystem {
  int L = 0;
  int device = 0;                            // the context's CUDA device
  int nx = 0, ny = 0;                        // the grid every MC_GRID2D continuum lives on
  std::vector<int64_t> off;                  // [L + 1]
  std::vector<int32_t> kind;                 // [L] 0 grid, 1 graph
  std::vector<int32_t> cont, host;           // per fine DOF: continuum, host grid cell
  std::vector<double> meas, mass, F, u0;     // |cell|, c|cell|, F (Dirichlet + wells + f|cell|), p^0
  std::vector<double> ddiag, wdiag;          // non-edge diagonal of D (Dirichlet faces); wells
  std::vector<int32_t> ei, ej;               // D: two-point connections within a continuum
  std::vector<double> et;
  std::vector<int32_t> qi, qj;               // Q: transfer entries between continua
  std::vector<double> qs;
};

// Fill fs from a set-up, not yet finalised context.  host[alpha]: graph continua's host
// grid cells (caller numbering, host or device pointers).
mc_status export_fine(mc_ctx* c, const int32_t* const* host, FineSystem& fs);
// Record an error message on the context (mc_error_string).
mc_status ctx_error(mc_ctx* c, mc_status st, const char* msg);

}  // namespace mc
