// msplat C++ drop-in -- loss report and combine (reference API:
// proj/core/include/msplat/losses.hpp).  The per-frame loss evaluation and
// seed assembly run on the device (evaluate_frame_losses, trainer.hpp).
#pragma once

#include "msplat/types.hpp"

#include <array>

namespace msplat {

struct ScalarLoss {
    Scalar value = 0;
    GridF grad;  // same shape as the differentiated input
};

struct LossReport {
    Scalar l1 = 0, ssim = 0, depth = 0, normal = 0, seg = 0, k = 0;
    Scalar combined = 0;
    // |L_l1| / |L_x| magnitude-normalization ratios, frozen per iteration.
    Scalar ratio_ssim = 0, ratio_normal = 0, ratio_depth = 0, ratio_seg = 0, ratio_k = 0;
    // Effective gradient-seed scales (zero when a term is disabled or vanishes).
    Scalar seed_l1 = 0, seed_ssim = 0, seed_depth = 0, seed_normal = 0, seed_seg = 0, seed_k = 0;
};

/// Magnitude-normalized total loss. lambdas = (l1, ssim, normal, depth, seg, k).
LossReport combine(Scalar l1, Scalar ssim, Scalar normal, Scalar depth, Scalar seg, Scalar k,
                   const std::array<Scalar, 6>& lambdas);

}  // namespace msplat
