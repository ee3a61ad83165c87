// io.cpp -- SPEC cli_io MeshFile / MetricsFile as host C++.
//
// Host-only: these entry points touch no device (they load and run on a
// machine without a GPU).  The formats are described in include/dualmesh/io.hpp.
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "dm_capi.h"
#include "dualmesh/io.hpp"

namespace {

struct ParseError {
  long line;
  std::string what;
};

struct Parsed {
  int dim = 0;
  std::vector<double> coords;
  std::vector<int32_t> elements, boundary;
  bool has_boundary = false;
};

// Splits s into whitespace-separated tokens (after stripping a '#' comment).
void tokens(std::string_view s, std::vector<std::string_view>& out) {
  out.clear();
  const size_t hash = s.find('#');
  if (hash != std::string_view::npos) s = s.substr(0, hash);
  size_t i = 0;
  while (i < s.size()) {
    while (i < s.size() && (s[i] == ' ' || s[i] == '\t' || s[i] == '\r')) ++i;
    size_t j = i;
    while (j < s.size() && s[j] != ' ' && s[j] != '\t' && s[j] != '\r') ++j;
    if (j > i) out.push_back(s.substr(i, j - i));
    i = j;
  }
}

bool to_i64(std::string_view t, long long& v) {
  auto r = std::from_chars(t.data(), t.data() + t.size(), v);
  return r.ec == std::errc() && r.ptr == t.data() + t.size();
}
bool to_f64(std::string_view t, double& v) {
  auto r = std::from_chars(t.data(), t.data() + t.size(), v);
  return r.ec == std::errc() && r.ptr == t.data() + t.size();
}

Parsed parse_mesh(const std::string& text) {
  Parsed P;
  std::vector<std::string_view> tk;
  std::string_view all(text);
  size_t pos = 0;
  long line = 0;
  // next non-empty line's tokens; false at EOF
  auto next = [&]() -> bool {
    while (pos < all.size()) {
      size_t e = all.find('\n', pos);
      if (e == std::string_view::npos) e = all.size();
      const std::string_view ln = all.substr(pos, e - pos);
      pos = e + 1;
      ++line;
      tokens(ln, tk);
      if (!tk.empty()) return true;
    }
    return false;
  };
  auto keyword = [&](const char* name, long long& count) {
    if (!next()) throw ParseError{line, std::string("missing \"") + name + "\" section"};
    if (tk.size() != 2 || tk[0] != name || !to_i64(tk[1], count) || count < 0)
      throw ParseError{line, std::string("expected \"") + name + " <count>\""};
  };
  if (!next() || tk.size() != 2 || tk[0] != "dualmesh" || tk[1] != "v1")
    throw ParseError{line, "expected header \"dualmesh v1\""};
  long long dim = 0;
  keyword("dim", dim);
  if (dim != 2 && dim != 3) throw ParseError{line, "dim must be 2 or 3"};
  P.dim = static_cast<int>(dim);
  long long nv = 0;
  keyword("nodes", nv);
  if (nv >= (1ll << 31)) throw ParseError{line, "node ids are 32-bit"};
  // grown line by line: a declared count is only trusted as far as the
  // remaining input could hold it (every value takes >= 2 bytes), so a huge
  // count over a short file reports the count mismatch, not bad_alloc
  auto cap = [&](long long values) {
    return static_cast<size_t>(std::min<long long>(values, (all.size() - std::min(pos, all.size())) / 2 + 1));
  };
  P.coords.reserve(cap(dim * nv));
  // the next data line of a section; a missing one (end of file or a
  // keyword line) is a count mismatch reported at that line
  auto data_line = [&](const char* section, long long want, long long got) {
    double probe;
    if (!next() || !to_f64(tk[0], probe))
      throw ParseError{line, "count mismatch: " + std::to_string(want) + " " + section +
                                 " lines declared, " + std::to_string(got) + " found"};
  };
  for (long long v = 0; v < nv; ++v) {
    data_line("node", nv, v);
    if (static_cast<long long>(tk.size()) != dim)
      throw ParseError{line, "expected " + std::to_string(dim) + " coordinates"};
    for (int d = 0; d < dim; ++d) {
      double xv;
      if (!to_f64(tk[d], xv)) throw ParseError{line, "bad number \"" + std::string(tk[d]) + "\""};
      P.coords.push_back(xv);
    }
  }
  auto ids = [&](const char* section, long long count, int per, std::vector<int32_t>& out) {
    out.clear();
    out.reserve(cap(count * per));
    for (long long r = 0; r < count; ++r) {
      data_line(section, count, r);
      if (static_cast<int>(tk.size()) != per)
        throw ParseError{line, "expected " + std::to_string(per) + " node ids"};
      for (int a = 0; a < per; ++a) {
        long long id;
        if (!to_i64(tk[a], id)) throw ParseError{line, "bad id \"" + std::string(tk[a]) + "\""};
        if (id < 1 || id > nv)
          throw ParseError{line, "invalid index " + std::to_string(id) + " (nodes are 1.." +
                                     std::to_string(nv) + ")"};
        out.push_back(static_cast<int32_t>(id - 1));
      }
    }
  };
  long long ne = 0;
  keyword("elements", ne);
  ids("element", ne, P.dim + 1, P.elements);
  if (next()) {
    long long nb = 0;
    if (tk.size() != 2 || tk[0] != "boundary" || !to_i64(tk[1], nb) || nb < 0)
      throw ParseError{line, "expected \"boundary <count>\" or end of file"};
    P.has_boundary = true;
    ids("boundary", nb, P.dim, P.boundary);
    if (next()) throw ParseError{line, "unexpected content after the boundary section"};
  }
  return P;
}

std::string slurp(const char* path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw std::runtime_error(std::string(path) + ": cannot open");
  std::ostringstream s;
  s << f.rdbuf();
  return s.str();
}

void put_f64(std::string& out, double v) {
  if (!std::isfinite(v)) {
    out += "null";
    return;
  }
  char b[40];
  auto r = std::to_chars(b, b + sizeof(b), v, std::chars_format::general, 17);
  out.append(b, r.ptr);
}
void put_i64(std::string& out, long long v) {
  char b[24];
  auto r = std::to_chars(b, b + sizeof(b), v);
  out.append(b, r.ptr);
}

void write_file(const char* path, const std::string& s) {
  FILE* f = std::fopen(path, "wb");
  if (!f) throw std::runtime_error(std::string(path) + ": cannot open for writing");
  const size_t w = std::fwrite(s.data(), 1, s.size(), f);
  const int c = std::fclose(f);
  if (w != s.size() || c != 0) throw std::runtime_error(std::string(path) + ": write failed");
}

std::string mesh_text(int dim, const double* x, int64_t nv, const int32_t* el, int64_t ne,
                      const int32_t* bnd, int64_t nb) {
  std::string o;
  o.reserve(static_cast<size_t>(nv * dim * 24 + ne * (dim + 1) * 9 + nb * dim * 9 + 64));
  o += "dualmesh v1\ndim ";
  put_i64(o, dim);
  o += "\nnodes ";
  put_i64(o, nv);
  o += '\n';
  for (int64_t v = 0; v < nv; ++v) {
    for (int d = 0; d < dim; ++d) {
      if (d) o += ' ';
      put_f64(o, x[dim * v + d]);
    }
    o += '\n';
  }
  o += "elements ";
  put_i64(o, ne);
  o += '\n';
  for (int64_t e = 0; e < ne; ++e) {
    for (int a = 0; a <= dim; ++a) {
      if (a) o += ' ';
      put_i64(o, static_cast<long long>(el[(dim + 1) * e + a]) + 1);
    }
    o += '\n';
  }
  {  // always written, so an empty boundary stays empty (no derivation on read)
    o += "boundary ";
    put_i64(o, nb);
    o += '\n';
    for (int64_t b = 0; b < nb; ++b) {
      for (int a = 0; a < dim; ++a) {
        if (a) o += ' ';
        put_i64(o, static_cast<long long>(bnd[dim * b + a]) + 1);
      }
      o += '\n';
    }
  }
  return o;
}

uint64_t fnv(uint64_t h, const void* p, size_t n) {
  const unsigned char* c = static_cast<const unsigned char*>(p);
  for (size_t i = 0; i < n; ++i) {
    h ^= c[i];
    h *= 0x100000001B3ull;
  }
  return h;
}

void set_err(char* err, int64_t len, const std::string& msg) {
  if (!err || len <= 0) return;
  const size_t n = std::min<size_t>(msg.size(), static_cast<size_t>(len - 1));
  std::memcpy(err, msg.data(), n);
  err[n] = '\0';
}

const char* nav_name(int a) { return a == DM_NAV_DUALFREE ? "dualfree" : "traditional"; }
const char* vol_name(int a) { return a == DM_VOL_EDGE ? "edge" : "element"; }

}  // namespace

// ------------------------------------------------------------------ C-ABI
extern "C" {

int dm_mesh_file_read(const char* path, int* dim, int64_t* n_nodes, int64_t* n_elements,
                      int64_t* n_boundary, int* has_boundary, double* coords, int32_t* elements,
                      int32_t* boundary, char* err, int64_t err_len) {
  if (!path) return DM_ERR_INVALID_ARG;
  try {
    const Parsed P = parse_mesh(slurp(path));
    const int64_t nv = static_cast<int64_t>(P.coords.size()) / P.dim;
    const int64_t ne = static_cast<int64_t>(P.elements.size()) / (P.dim + 1);
    const int64_t nb = static_cast<int64_t>(P.boundary.size()) / P.dim;
    if (dim) *dim = P.dim;
    if (n_nodes) *n_nodes = nv;
    if (n_elements) *n_elements = ne;
    if (n_boundary) *n_boundary = nb;
    if (has_boundary) *has_boundary = P.has_boundary ? 1 : 0;
    if (coords) std::memcpy(coords, P.coords.data(), P.coords.size() * sizeof(double));
    if (elements) std::memcpy(elements, P.elements.data(), P.elements.size() * sizeof(int32_t));
    if (boundary) std::memcpy(boundary, P.boundary.data(), P.boundary.size() * sizeof(int32_t));
    set_err(err, err_len, "");
    return DM_OK;
  } catch (const ParseError& e) {
    set_err(err, err_len, std::string(path) + ":" + std::to_string(e.line) + ": " + e.what);
    return DM_ERR_INVALID_ARG;
  } catch (const std::exception& e) {
    set_err(err, err_len, e.what());
    return DM_ERR_INVALID_ARG;
  }
}

int dm_mesh_file_write(const char* path, int dim, const double* coords, int64_t n_nodes,
                       const int32_t* elements, int64_t n_elements, const int32_t* boundary,
                       int64_t n_boundary) {
  if (!path || (dim != 2 && dim != 3) || n_nodes < 0 || n_elements < 0 || n_boundary < 0)
    return DM_ERR_INVALID_ARG;
  try {
    write_file(path, mesh_text(dim, coords, n_nodes, elements, n_elements, boundary, n_boundary));
    return DM_OK;
  } catch (const std::exception&) {
    return DM_ERR_INVALID_ARG;
  }
}

uint64_t dm_mesh_checksum(int dim, const double* coords, int64_t n_nodes, const int32_t* elements,
                          int64_t n_elements, const int32_t* boundary, int64_t n_boundary) {
  uint64_t h = 0xCBF29CE484222325ull;
  const int32_t d32 = dim;
  h = fnv(h, &d32, sizeof(d32));
  h = fnv(h, &n_nodes, sizeof(n_nodes));
  if (coords) h = fnv(h, coords, sizeof(double) * dim * n_nodes);
  h = fnv(h, &n_elements, sizeof(n_elements));
  if (elements) h = fnv(h, elements, sizeof(int32_t) * (dim + 1) * n_elements);
  h = fnv(h, &n_boundary, sizeof(n_boundary));
  if (boundary) h = fnv(h, boundary, sizeof(int32_t) * dim * n_boundary);
  return h;
}

int dm_metrics_file_write(const char* path, int dim, const int32_t* edges, int64_t n_edges,
                          const double* navs, const double* volumes, int64_t n_nodes,
                          int nav_algo, int vol_algo, uint64_t mesh_checksum) {
  if (!path || (dim != 2 && dim != 3) || n_edges < 0 || n_nodes < 0 ||
      (n_edges && (!edges || !navs)) || (n_nodes && !volumes))
    return DM_ERR_INVALID_ARG;
  try {
    std::string o;
    o.reserve(static_cast<size_t>(n_edges * (dim * 25 + 24) + n_nodes * 26 + 512));
    char ck[32];
    std::snprintf(ck, sizeof(ck), "fnv1a64:%016llx", static_cast<unsigned long long>(mesh_checksum));
    o += "{\n \"format\": \"dualmesh-metrics v1\",\n \"dim\": ";
    put_i64(o, dim);
    o += ",\n \"provenance\": {\"nav_algo\": \"";
    o += nav_name(nav_algo);
    o += "\", \"vol_algo\": \"";
    o += vol_name(vol_algo);
    o += "\", \"mesh_checksum\": \"";
    o += ck;
    o += "\", \"n_nodes\": ";
    put_i64(o, n_nodes);
    o += ", \"n_edges\": ";
    put_i64(o, n_edges);
    o += "},\n \"edges\": [";
    for (int64_t e = 0; e < n_edges; ++e) {
      o += e ? ",\n  [" : "\n  [";
      put_i64(o, static_cast<long long>(edges[2 * e]) + 1);
      o += ", ";
      put_i64(o, static_cast<long long>(edges[2 * e + 1]) + 1);
      o += ']';
    }
    o += "\n ],\n \"navs\": [";
    for (int64_t e = 0; e < n_edges; ++e) {
      o += e ? ",\n  [" : "\n  [";
      for (int d = 0; d < dim; ++d) {
        if (d) o += ", ";
        put_f64(o, navs[dim * e + d]);
      }
      o += ']';
    }
    o += "\n ],\n \"volumes\": [";
    for (int64_t v = 0; v < n_nodes; ++v) {
      o += v ? ",\n  " : "\n  ";
      put_f64(o, volumes[v]);
    }
    o += "\n ]\n}\n";
    write_file(path, o);
    return DM_OK;
  } catch (const std::exception&) {
    return DM_ERR_INVALID_ARG;
  }
}

}  // extern "C"

// ------------------------------------------------------------------ C++ API
namespace dualmesh {

Mesh read_mesh(const std::string& path) {
  Parsed P;
  try {
    P = parse_mesh(slurp(path.c_str()));
  } catch (const ParseError& e) {
    throw std::runtime_error(path + ":" + std::to_string(e.line) + ": " + e.what);
  }
  Mesh m;
  m.dim = P.dim;
  m.coords = std::move(P.coords);
  m.elements.assign(P.elements.begin(), P.elements.end());
  m.boundary.assign(P.boundary.begin(), P.boundary.end());
  // a missing boundary section triggers derivation
  if (!P.has_boundary && !m.elements.empty()) m.boundary = derive_boundary_faces(m);
  return m;
}

void write_mesh(const Mesh& mesh, const std::string& path) {
  static_assert(sizeof(Index) == sizeof(int32_t), "mesh ids are 32-bit");
  write_file(path.c_str(),
             mesh_text(mesh.dim, mesh.coords.data(), static_cast<int64_t>(mesh.num_nodes()),
                       reinterpret_cast<const int32_t*>(mesh.elements.data()),
                       static_cast<int64_t>(mesh.num_elements()),
                       reinterpret_cast<const int32_t*>(mesh.boundary.data()),
                       static_cast<int64_t>(mesh.num_boundary())));
}

std::uint64_t mesh_checksum(const Mesh& mesh) {
  return dm_mesh_checksum(mesh.dim, mesh.coords.data(), static_cast<int64_t>(mesh.num_nodes()),
                          reinterpret_cast<const int32_t*>(mesh.elements.data()),
                          static_cast<int64_t>(mesh.num_elements()),
                          reinterpret_cast<const int32_t*>(mesh.boundary.data()),
                          static_cast<int64_t>(mesh.num_boundary()));
}

void write_metrics(const std::string& path, const Mesh& mesh, const EdgeList& edges,
                   const LumpedNavField& navs, const DualVolumeField& volumes, NavAlgo nav_algo,
                   VolAlgo vol_algo) {
  const int64_t ne = static_cast<int64_t>(edges.edges.size());
  if (navs.navs.size() != static_cast<size_t>(mesh.dim * ne) ||
      volumes.volumes.size() != mesh.num_nodes())
    throw std::invalid_argument("field/mesh mismatch");
  std::vector<int32_t> flat(static_cast<size_t>(2 * ne));
  for (int64_t e = 0; e < ne; ++e) {
    flat[2 * e] = edges.edges[e][0];
    flat[2 * e + 1] = edges.edges[e][1];
  }
  if (dm_metrics_file_write(path.c_str(), mesh.dim, flat.data(), ne, navs.navs.data(),
                            volumes.volumes.data(), static_cast<int64_t>(mesh.num_nodes()),
                            static_cast<int>(nav_algo), static_cast<int>(vol_algo),
                            mesh_checksum(mesh)) != DM_OK)
    throw std::runtime_error(path + ": write failed");
}

}  // namespace dualmesh
