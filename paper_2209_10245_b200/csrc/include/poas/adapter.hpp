#pragma once
// Adapt: whole rows per unit, xpu row alignment (k % align == 0 required,
// the 16-byte TMA row-pitch rule for 16-bit operands), re-homing of the
// shaved rows, and the squareness-maximising (k', q) tiling inside each
// unit's profiled ops window (reference: proj/include/poas/adapter.hpp).

#include <cstdint>
#include <string>
#include <vector>

#include "poas/device_model.hpp"
#include "poas/optimizer.hpp"

namespace poas {

// m' x k' block of A times the k' x n block of B (n is never split).
struct Tile {
  std::int64_t m = 0;
  std::int64_t k = 0;
  std::int64_t n = 0;
};

struct TileDecision {
  std::int64_t k_prime = 0;
  std::vector<Tile> tiles;  // strip-major: for each k'-strip, its q m-parts
  double sq = 0.0;          // sum of min(m,k)/max(m,k) * m*k*n
};

struct PlannedDevice {
  std::string device_id;
  std::int64_t rows = 0;
  OpsCount ops = 0;
  TileDecision tiling;
  bool window_fallback = false;
};

struct TilePlan {
  MatrixDims dims;
  std::vector<PlannedDevice> devices;  // machine order
};

std::int64_t ops_to_rows(OpsCount c, const MatrixDims& dims);
std::int64_t align_rows(std::int64_t rows, const DeviceProfile& dev, const MatrixDims& dims);
void reassign_shaved(std::vector<std::int64_t>& rows, std::int64_t shaved,
                     const MachineProfile& machine, const WorkloadSplit& split);
TileDecision tile_device(const DeviceProfile& dev, std::int64_t rows, const MatrixDims& dims);
TilePlan build_tile_plan(const MachineProfile& machine, const MatrixDims& dims,
                         const WorkloadSplit& split);

}  // namespace poas
