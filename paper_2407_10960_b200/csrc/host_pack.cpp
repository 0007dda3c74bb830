// flute-b200 — offline restructuring: the reference-canonical packer
// (bit-exact with reorder_and_split, pack.cpp:48-173) and the sm_100a device
// layout the GPU kernel streams.
//
// Device layout.  The weight stream is a sequence of Stream-K
// units u = nt * tiles_k + kt (n-tile major, k inner — the reference's unit
// order), each covering 64 output columns x 128 k.  Inside a unit, the eight
// consumer warps w own one 16-deep k step each; every lane owns, per 16x16
// "atom" j (columns 16j..16j+15), the eight weights the swapped
// mma.m16n8k16 A-fragment needs (rows = n, cols = k, g = lane/4, t = lane%4):
//     reg p=0: n=g,   k=2t,2t+1     reg p=1: n=g+8, k=2t,2t+1
//     reg p=2: n=g,   k=2t+8,+9     reg p=3: n=g+8, k=2t+8,+9
// Each (n, k, k+1) pair is stored as one vLUT index, first (even k) in the high
// bits, pair q = 4j + p of the lane:
//   4-bit: byte p of word j = idx_k << 4 | idx_k1 (a lane's 4 atoms are one
//          16-byte LDS);
//   2-bit: word j>>1, byte p, nibble j&1 = idx_k << 2 | idx_k1 (8 B per lane);
//   3-bit: six-bit pair index D = (hi_k << 2 | hi_k1) << 2 | (lo_k << 1 | lo_k1)
//          (2-bit plane hi, 1-bit plane lo; the device vLUT is permuted to this
//          index) in three lane words A, B (8 B per lane, the unit's first
//          2 KiB) and C (4 B per lane, last 1 KiB): byte p of A / B / C holds
//          D of atom 0 / 1 / 2 in bits 0..5 and bits 0-1 / 2-3 / 4-5 of atom
//          3's D in bits 6..7 (dequant.cuh atom_index_bytes<3>).
// These are exactly the byte vectors dequant.cuh's atom_index_bytes expects.
#include <algorithm>
#include <cstring>
#include <string>

#include "flutesim/errors.hpp"
#include "flutesim/pack.hpp"

namespace flutesim {
namespace {

void require_divisible(int value, int divisor, const char* what) {
  if (divisor <= 0 || value % divisor != 0) {
    throw ConfigError(std::string(what) + ": " + std::to_string(value) + " not divisible by " +
                      std::to_string(divisor));
  }
}

inline std::uint32_t read_field(const BitSlice& s, std::size_t pos) {
  const std::size_t bit = pos * static_cast<std::size_t>(s.bits);
  return (s.words[bit >> 5] >> (bit & 31u)) & ((1u << s.bits) - 1u);
}

inline void write_field(BitSlice& s, std::size_t pos, std::uint32_t v) {
  const std::size_t bit = pos * static_cast<std::size_t>(s.bits);
  s.words[bit >> 5] |= v << (bit & 31u);
}

int round_up(int v, int m) { return (v + m - 1) / m * m; }

}  // namespace

// ---------------------------------------------------------------------------
// Canonical layout
// ---------------------------------------------------------------------------

void LayoutDescriptor::validate() const {
  if (tile_m <= 0 || tile_n <= 0 || tile_k <= 0 || frag_m <= 0 || frag_n <= 0 || frag_k <= 0) {
    throw ConfigError("layout: tile/fragment dims must be positive");
  }
  require_divisible(tile_m, frag_m, "layout: tile_m by frag_m");
  require_divisible(tile_n, frag_n, "layout: tile_n by frag_n");
  require_divisible(tile_k, frag_k, "layout: tile_k by frag_k");
  if (frag_k % 2 != 0) throw ConfigError("layout: frag_k must be even for paired dequantization");
  if (tile_elems() % 32 != 0) throw ConfigError("layout: a weight tile must cover whole 32-bit words");
}

std::size_t packed_pos(const LayoutDescriptor& L, int k, int n, int i, int j) {
  (void)n;
  const long tiles_k = k / L.tile_k;
  const long tile = static_cast<long>(j / L.tile_n) * tiles_k + i / L.tile_k;
  const int ki = i % L.tile_k, nj = j % L.tile_n;
  const long frag = static_cast<long>(ki / L.frag_k) * L.frags_per_tile_n() + nj / L.frag_n;
  const long within = static_cast<long>(ki % L.frag_k) * L.frag_n + nj % L.frag_n;
  return static_cast<std::size_t>(tile * L.tile_elems() + frag * L.frag_elems() + within);
}

void unpacked_coords(const LayoutDescriptor& L, int k, int n, std::size_t pos, int& i, int& j) {
  (void)n;
  const long tiles_k = k / L.tile_k;
  const long p = static_cast<long>(pos);
  const long tile = p / L.tile_elems();
  const long frag = (p % L.tile_elems()) / L.frag_elems();
  const long w = p % L.frag_elems();
  i = static_cast<int>((tile % tiles_k) * L.tile_k + (frag / L.frags_per_tile_n()) * L.frag_k +
                       w / L.frag_n);
  j = static_cast<int>((tile / tiles_k) * L.tile_n + (frag % L.frags_per_tile_n()) * L.frag_n +
                       w % L.frag_n);
}

PackedWeights reorder_and_split(const QuantizedMatrix& q, const LayoutDescriptor& layout) {
  layout.validate();
  require_divisible(q.k, layout.tile_k, "pack: k by tile_k");
  require_divisible(q.n, layout.tile_n, "pack: n by tile_n");
  PackedWeights pw;
  pw.layout = layout;
  pw.bits = q.cfg.bits;
  pw.k = q.k;
  pw.n = q.n;
  if (pw.bits == 3) {
    pw.slices = {BitSlice{2, {}}, BitSlice{1, {}}};
  } else {
    pw.slices = {BitSlice{pw.bits, {}}};
  }
  const std::size_t total = static_cast<std::size_t>(q.k) * q.n;
  for (BitSlice& s : pw.slices) s.words.assign((total * s.bits + 31) / 32, 0u);
  for (int i = 0; i < q.k; ++i) {
    for (int j = 0; j < q.n; ++j) {
      const std::uint32_t v = q.indices[static_cast<std::size_t>(i) * q.n + j];
      const std::size_t pos = packed_pos(layout, q.k, q.n, i, j);
      if (pw.bits == 3) {
        write_field(pw.slices[0], pos, v >> 1);
        write_field(pw.slices[1], pos, v & 1u);
      } else {
        write_field(pw.slices[0], pos, v);
      }
    }
  }
  return pw;
}

std::uint8_t combine_slices(std::uint8_t hi, std::uint8_t lo) {
  if (hi >= 4 || lo >= 2) throw InternalError("combine_slices: slice value out of range");
  return static_cast<std::uint8_t>((hi << 1) | lo);
}

std::vector<std::uint8_t> unpack_fragment(const PackedWeights& pw, long tile_idx, long frag_idx) {
  if (tile_idx < 0 || tile_idx >= pw.tile_count()) {
    throw InputError("unpack_fragment: tile index " + std::to_string(tile_idx) + " out of range");
  }
  if (frag_idx < 0 || frag_idx >= pw.frags_per_tile()) {
    throw InputError("unpack_fragment: fragment index " + std::to_string(frag_idx) +
                     " out of range");
  }
  const long fe = pw.layout.frag_elems();
  const std::size_t base =
      static_cast<std::size_t>(tile_idx * pw.layout.tile_elems() + frag_idx * fe);
  std::vector<std::uint8_t> out(static_cast<std::size_t>(fe));
  for (long t = 0; t < fe; ++t) {
    out[t] = pw.bits == 3
                 ? combine_slices(static_cast<std::uint8_t>(read_field(pw.slices[0], base + t)),
                                  static_cast<std::uint8_t>(read_field(pw.slices[1], base + t)))
                 : static_cast<std::uint8_t>(read_field(pw.slices[0], base + t));
  }
  return out;
}

std::vector<std::uint8_t> unpack_matrix(const PackedWeights& pw) {
  std::vector<std::uint8_t> out(static_cast<std::size_t>(pw.k) * pw.n);
  const std::size_t total = out.size();
  for (std::size_t pos = 0; pos < total; ++pos) {
    int i = 0, j = 0;
    unpacked_coords(pw.layout, pw.k, pw.n, pos, i, j);
    const std::uint32_t v =
        pw.bits == 3 ? combine_slices(static_cast<std::uint8_t>(read_field(pw.slices[0], pos)),
                                      static_cast<std::uint8_t>(read_field(pw.slices[1], pos)))
                     : read_field(pw.slices[0], pos);
    out[static_cast<std::size_t>(i) * pw.n + j] = static_cast<std::uint8_t>(v);
  }
  return out;
}

// ---------------------------------------------------------------------------
// Device layout
// ---------------------------------------------------------------------------

DeviceGeometry device_geometry(int k, int n, int bits, int group) {
  QuantConfig{bits, group}.validate(k);
  if (k < 1 || n < 1) throw ConfigError("device layout: k and n must be positive");
  if (k % 16 != 0 || n % 16 != 0) {
    throw ConfigError("device layout: k and n must be multiples of 16 (the MMA atom)");
  }
  DeviceGeometry g;
  g.k = k;
  g.n = n;
  g.bits = bits;
  g.group = group;
  g.kp = round_up(k, kUnitK);
  g.np = round_up(n, kUnitN);
  if (g.kp % group != 0) throw ConfigError("device layout: padded k not divisible by group");
  return g;
}

namespace {

// Visits every (unit, warp, lane, atom, reg) slot of the device stream and the
// (n, k) coordinate of the pair's first weight.
template <class F>
void for_each_pair_slot(const DeviceGeometry& g, F&& f) {
  const long units = g.units();
#pragma omp parallel for schedule(static)
  for (long u = 0; u < units; ++u) {
    const int nt = static_cast<int>(u / g.tiles_k());
    const int kt = static_cast<int>(u % g.tiles_k());
    for (int w = 0; w < 8; ++w) {
      for (int lane = 0; lane < 32; ++lane) {
        const int gr = lane >> 2, t = lane & 3;
        for (int j = 0; j < 4; ++j) {
          for (int p = 0; p < 4; ++p) {
            const int col = nt * kUnitN + 16 * j + gr + 8 * (p & 1);
            const int row = kt * kUnitK + 16 * w + 2 * t + 8 * (p >> 1);
            f(u, w, lane, j, p, row, col);
          }
        }
      }
    }
  }
}

}  // namespace

std::vector<std::uint8_t> pack_device(const std::vector<std::uint8_t>& indices, int k, int n,
                                      int bits, int group) {
  const DeviceGeometry g = device_geometry(k, n, bits, group);
  if (indices.size() != static_cast<std::size_t>(k) * n) {
    throw InputError("pack_device: expected k*n indices");
  }
  const std::uint8_t zero = static_cast<std::uint8_t>((1u << (bits - 1)) - 1u);
  const std::uint32_t limit = 1u << bits;
  for (const std::uint8_t v : indices) {
    if (v >= limit) throw InputError("pack_device: index out of range for bit width");
  }
  auto at = [&](int row, int col) -> std::uint32_t {
    return (row < k && col < n) ? indices[static_cast<std::size_t>(row) * n + col] : zero;
  };
  std::vector<std::uint8_t> out(g.weight_bytes(), 0);
  const std::size_t ub = g.unit_bytes();
  for_each_pair_slot(g, [&](long u, int w, int lane, int j, int p, int row, int col) {
    std::uint8_t* unit = out.data() + static_cast<std::size_t>(u) * ub;
    const std::uint32_t a = at(row, col), b = at(row + 1, col);
    const int slot = w * 32 + lane;
    if (bits == 4) {
      unit[slot * 16 + j * 4 + p] = static_cast<std::uint8_t>((a << 4) | b);
    } else if (bits == 2) {
      // word j>>1 of the lane, byte p, low nibble for even j, high for odd j
      unit[slot * 8 + (j >> 1) * 4 + p] |= static_cast<std::uint8_t>(((a << 2) | b) << (4 * (j & 1)));
    } else {  // 3-bit: lane words A, B (8 B / lane) then C (4 B / lane)
      const std::uint32_t d = ((((a >> 1) << 2) | (b >> 1)) << 2) | ((a & 1u) << 1) | (b & 1u);
      auto word_byte = [&](int wi) -> std::uint8_t& {
        return wi < 2 ? unit[slot * 8 + wi * 4 + p] : unit[2048 + slot * 4 + p];
      };
      if (j < 3) {
        word_byte(j) |= static_cast<std::uint8_t>(d);
      } else {
        for (int wi = 0; wi < 3; ++wi) word_byte(wi) |= static_cast<std::uint8_t>(((d >> (2 * wi)) & 3u) << 6);
      }
    }
  });
  return out;
}

std::vector<std::uint8_t> pack_device_from_canonical(const PackedWeights& pw, int group) {
  return pack_device(unpack_matrix(pw), pw.k, pw.n, pw.bits, group);
}

std::vector<std::uint8_t> unpack_device(const std::vector<std::uint8_t>& dev, int k, int n,
                                        int bits, int group) {
  const DeviceGeometry g = device_geometry(k, n, bits, group);
  if (dev.size() != g.weight_bytes()) throw InputError("unpack_device: size mismatch");
  std::vector<std::uint8_t> out(static_cast<std::size_t>(k) * n, 0);
  const std::size_t ub = g.unit_bytes();
  for_each_pair_slot(g, [&](long u, int w, int lane, int j, int p, int row, int col) {
    if (row >= k || col >= n) return;
    const std::uint8_t* unit = dev.data() + static_cast<std::size_t>(u) * ub;
    const int slot = w * 32 + lane;
    std::uint32_t a = 0, b = 0;
    if (bits == 4) {
      const std::uint32_t v = unit[slot * 16 + j * 4 + p];
      a = v >> 4;
      b = v & 15u;
    } else if (bits == 2) {
      const std::uint32_t nib = (unit[slot * 8 + (j >> 1) * 4 + p] >> (4 * (j & 1))) & 15u;
      a = nib >> 2;
      b = nib & 3u;
    } else {
      auto word_byte = [&](int wi) -> std::uint32_t {
        return wi < 2 ? unit[slot * 8 + wi * 4 + p] : unit[2048 + slot * 4 + p];
      };
      std::uint32_t d = 0;
      if (j < 3) {
        d = word_byte(j) & 63u;
      } else {
        for (int wi = 0; wi < 3; ++wi) d |= (word_byte(wi) >> 6) << (2 * wi);
      }
      const std::uint32_t hi = d >> 2, lo = d & 3u;  // hi = (a >> 1) << 2 | b >> 1
      a = ((hi >> 2) << 1) | (lo >> 1);
      b = ((hi & 3u) << 1) | (lo & 1u);
    }
    out[static_cast<std::size_t>(row) * n + col] = static_cast<std::uint8_t>(a);
    out[static_cast<std::size_t>(row + 1) * n + col] = static_cast<std::uint8_t>(b);
  });
  return out;
}

std::vector<std::uint16_t> scales_to_device(const std::vector<Half>& scales, int k, int n,
                                            int group) {
  const DeviceGeometry g = device_geometry(k, n, 4, group);
  const int gpc = k / group;
  if (scales.size() != static_cast<std::size_t>(gpc) * n) {
    throw InputError("scales_to_device: expected (k/group)*n scales");
  }
  const int gp = g.groups_padded();
  std::vector<std::uint16_t> out(static_cast<std::size_t>(g.tiles_n()) * gp * kUnitN, 0);
  for (int nt = 0; nt < g.tiles_n(); ++nt) {
    for (int G = 0; G < gp; ++G) {
      std::uint16_t* blk = out.data() + (static_cast<std::size_t>(nt) * gp + G) * kUnitN;
      for (int gr = 0; gr < 8; ++gr) {
        for (int j = 0; j < 4; ++j) {
          for (int h = 0; h < 2; ++h) {
            const int col = nt * kUnitN + 16 * j + gr + 8 * h;
            blk[gr * 8 + j * 2 + h] =
                (col < n && G < gpc) ? scales[static_cast<std::size_t>(col) * gpc + G].bits : 0;
          }
        }
      }
    }
  }
  return out;
}

}  // namespace flutesim
