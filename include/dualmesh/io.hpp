// io.hpp -- the SPEC cli_io file formats:
// the on-disk formats either side of the path.
//
// MeshFile (text): "dualmesh v1", "dim D", "nodes N" + N coordinate lines,
// "elements M" + M connectivity lines (1-based), optional "boundary K" + K
// boundary-element lines (1-based, outward).  '#' starts a comment; blanks
// and tabs separate tokens.  A missing boundary section is derived
// (derive_boundary_faces).  Coordinates are written with 17 significant
// digits, so read(write(m)) == m bit for bit.
//
// MetricsFile (JSON): {"format": "dualmesh-metrics v1", "dim", "provenance":
// {"nav_algo", "vol_algo", "mesh_checksum", "n_nodes", "n_edges"}, "edges"
// (1-based pairs), "navs" (per-edge D-vectors), "volumes"}; 17 significant
// digits, deterministic bytes (no clock; the checksum is FNV-1a 64 over the
// mesh arrays).
#ifndef DUALMESH_IO_HPP
#define DUALMESH_IO_HPP

#include <cstdint>
#include <string>

#include "dualmesh/mesh.hpp"
#include "dualmesh/metrics.hpp"

namespace dualmesh {

// Parse errors throw std::runtime_error("<path>:<line>: <what>") -- syntax,
// count mismatch, invalid index.
Mesh read_mesh(const std::string& path);
void write_mesh(const Mesh& mesh, const std::string& path);

// FNV-1a 64 over dim, the coordinate bytes, element ids and boundary ids.
std::uint64_t mesh_checksum(const Mesh& mesh);

void write_metrics(const std::string& path, const Mesh& mesh, const EdgeList& edges,
                   const LumpedNavField& navs, const DualVolumeField& volumes, NavAlgo nav_algo,
                   VolAlgo vol_algo);

}  // namespace dualmesh

#endif  // DUALMESH_IO_HPP
