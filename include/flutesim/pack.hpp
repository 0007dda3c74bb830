// flute-b200 — offline weight restructuring.
//
// Two layouts live here:
//
//  * The reference-canonical layout (reference: proj/include/flutesim/pack.hpp:
//    20-85, pack.cpp:48-173): fragment-major permutation plus little-endian
//    bit-slice packing, 3-bit split into a 2-bit and a 1-bit plane.  Kept
//    bit-exact for interchange (FLTE files, the reference API and its tests).
//
//  * The sm_100a device layout (new): the exact per-lane register order the
//    swapped m16n8k16 tensor-core MMA consumes, so the kernel unpacks with one
//    PRMT per weight pair.  See DESIGN.md §3 for the byte-level definition.
//    DevicePacked is bijective with the index matrix (unpack_device inverts it)
//    and converts from/to the canonical layout without touching the indices.
#pragma once

#include <cstddef>
#include <cstdint>
#include <vector>

#include "flutesim/quantize.hpp"

namespace flutesim {

struct LayoutDescriptor {
  int tile_m = 16;
  int tile_n = 64;
  int tile_k = 64;
  int frag_m = 16;
  int frag_n = 8;
  int frag_k = 16;

  void validate() const;

  int frags_per_tile_k() const { return tile_k / frag_k; }
  int frags_per_tile_n() const { return tile_n / frag_n; }
  long tile_elems() const { return static_cast<long>(tile_k) * tile_n; }
  long frag_elems() const { return static_cast<long>(frag_k) * frag_n; }
};

std::size_t packed_pos(const LayoutDescriptor& layout, int k, int n, int i, int j);
void unpacked_coords(const LayoutDescriptor& layout, int k, int n, std::size_t pos, int& i,
                     int& j);

struct BitSlice {
  int bits = 0;
  std::vector<std::uint32_t> words;
};

struct PackedWeights {
  std::vector<BitSlice> slices;  // high-to-low plane
  LayoutDescriptor layout;
  int bits = 0;
  int k = 0;
  int n = 0;

  long tiles_k() const { return k / layout.tile_k; }
  long tiles_n() const { return n / layout.tile_n; }
  long tile_count() const { return tiles_k() * tiles_n(); }
  long frags_per_tile() const {
    return static_cast<long>(layout.frags_per_tile_k()) * layout.frags_per_tile_n();
  }
};

PackedWeights reorder_and_split(const QuantizedMatrix& q, const LayoutDescriptor& layout);
std::uint8_t combine_slices(std::uint8_t hi, std::uint8_t lo);
std::vector<std::uint8_t> unpack_fragment(const PackedWeights& pw, long tile_idx, long frag_idx);
std::vector<std::uint8_t> unpack_matrix(const PackedWeights& pw);

// ---------------------------------------------------------------------------
// sm_100a device layout
// ---------------------------------------------------------------------------

// Geometry of one Stream-K work unit on the device: 64 output columns x 128 k.
inline constexpr int kUnitN = 64;
inline constexpr int kUnitK = 128;

struct DeviceGeometry {
  int k = 0, n = 0, bits = 0, group = 0;
  int kp = 0, np = 0;  // padded to kUnitK / kUnitN
  int tiles_k() const { return kp / kUnitK; }
  int tiles_n() const { return np / kUnitN; }
  long units() const { return static_cast<long>(tiles_k()) * tiles_n(); }
  std::size_t unit_bytes() const { return static_cast<std::size_t>(kUnitN) * kUnitK * bits / 8; }
  std::size_t weight_bytes() const { return unit_bytes() * static_cast<std::size_t>(units()); }
  int groups_padded() const { return kp / group; }
  std::size_t scale_bytes() const {
    return static_cast<std::size_t>(tiles_n()) * groups_padded() * kUnitN * 2;
  }
};

DeviceGeometry device_geometry(int k, int n, int bits, int group);

// Host-side packing into device order.  Padding rows/columns (k up to kp, n
// up to np) get the table's zero index 2^(b-1)-1 and scale 0, so they add
// exact zeros.
std::vector<std::uint8_t> pack_device(const std::vector<std::uint8_t>& indices, int k, int n,
                                      int bits, int group);
std::vector<std::uint8_t> pack_device_from_canonical(const PackedWeights& pw, int group);
std::vector<std::uint8_t> unpack_device(const std::vector<std::uint8_t>& dev, int k, int n,
                                        int bits, int group);
// [n][k/g] binary16 scales -> device scale blocks.
std::vector<std::uint16_t> scales_to_device(const std::vector<Half>& scales, int k, int n,
                                            int group);

}  // namespace flutesim
