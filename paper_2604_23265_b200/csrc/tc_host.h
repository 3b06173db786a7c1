// Host helpers for the tensor-core kernels (NOT part of the ABI): TMA tensor-map encoding via the
// driver entry point (no link-time libcuda dependency) and the 3xTF32 operand split.
#pragma once

#include <cuda.h>
#include <stdint.h>

#include <vector>

namespace rte {
namespace tc {

// 4-D map over an NHWC fp32 tensor [B][H][W][C] (dims C, W, H, B), SWIZZLE_128B, box
// (32 channels, box_w, box_h, 1) with traversal stride `es` along W and H (1 or 2); the
// out-of-bounds fill is zero (implements the convolutions' zero padding).
CUtensorMap make_map_act(const float* base, int C, int W, int H, int B, int box_w, int box_h, int es);
// 5-D map over a pre-split activation [B][2][H][W][C] (plane 0 hi, plane 1 lo), dims
// (C, W, H, plane, B), same boxes as make_map_act with a plane extent of 1.
CUtensorMap make_map_act_split(const float* base, int C, int W, int H, int B, int box_w, int box_h, int es);
// L2-prefetch map (no swizzle, no shared-memory destination) over NHWC [B][H][W][C], box (box_c, box_w, box_h, 1).
CUtensorMap make_map_prefetch(const float* base, int C, int W, int H, int B, int box_c, int box_w, int box_h);
// 2-D map over a row-major fp32 matrix [rows][K] (K contiguous), SWIZZLE_128B, box (32, box_rows).
CUtensorMap make_map_kmajor(const float* base, int K, int rows, int box_rows);

// Host 3xTF32 split (round-to-nearest, ties away -- the same rule as cvt.rna.tf32.f32).
float tf32_rna_host(float v);
void split_host(const std::vector<float>& w, std::vector<float>& hi, std::vector<float>& lo);

// RTE_TC_DBG perf-experiment switches (see Geom::dbg); 0 unless the variable is set.
int tc_debug_flags();

// Opt a kernel into `bytes` of dynamic shared memory (once per kernel pointer).
void ensure_smem(const void* kernel, int bytes);

}  // namespace tc
}  // namespace rte
