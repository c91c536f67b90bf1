// Measured token-budget selection: fit the reference's timing
// constants to observed batch timings — here, B200 forward times — so that
// compute_token_budget and the SLO derivation run on this hardware's clock.
//
// Restates servesim::calibrate (reference proj/src/calibrate.cpp:121-193,
// declared costmodel.hpp:71-102): a weighted (1/observed^2) least-squares fit
// of (fixed, per-token, quad, kv-read, decode-per-kv), linear once the
// saturation point is fixed, swept over saturation = 1..max and the smallest
// relative SSE kept. Terms no anchor exercises are pinned to zero; an anchor
// set that cannot identify the rest is rejected, naming the parameter.
#pragma once

#include <stdexcept>
#include <string>
#include <vector>

#include "costmodel.hpp"

namespace ss {

struct CalibrationError : std::runtime_error {  // costmodel.hpp:74-76
    using std::runtime_error::runtime_error;
};

struct Anchor {  // CalibrationAnchor, costmodel.hpp:78-81
    Batch batch;
    double observed_ms = 0.0;
};

struct CalibrationOptions {  // costmodel.hpp:91-95
    int tile_size = 256;
    double tile_penalty_frac = 0.32;
    int max_saturation_tokens = 2048;
};

struct Calibration {  // CalibrationResult, costmodel.hpp:83-89
    CostParams params;
    std::vector<double> predicted_ms;
    std::vector<double> relative_error;
    double max_relative_error = 0.0;
    std::vector<std::string> zeroed_terms;
};

Calibration calibrate(const std::vector<Anchor>& anchors, const CalibrationOptions& opts = {});

}  // namespace ss
