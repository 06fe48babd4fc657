// graph_io.cpp -- the reference's on-disk graph format, host side:
//
//   edges.bin        raw Edge records (u32 src, rel, dst; 12 B, little endian)
//   graph_meta.json  {"num_edges", "num_nodes", "num_relations"}
//
// write_graph / read_graph (graph.cpp:152-192).  The JSON text is byte-for-
// byte what the reference's nlohmann dump(2) + "\n" writes (keys sorted,
// two-space indent), so either side reads the other's files
// (tests/test_graph_io.py checks both directions against the compiled
// reference).  Errors are std::runtime_error as in the reference.
#include <cerrno>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <sys/stat.h>

#include "abi.hpp"

namespace {

std::string join(const char* dir, const char* name) {
  std::string p(dir);
  if (!p.empty() && p.back() != '/') p += '/';
  return p + name;
}

void make_dirs(const std::string& dir) {  // std::filesystem::create_directories
  std::string cur;
  for (size_t i = 0; i <= dir.size(); ++i) {
    if (i == dir.size() || dir[i] == '/') {
      if (!cur.empty() && mkdir(cur.c_str(), 0777) != 0 && errno != EEXIST)
        throw std::runtime_error("cannot create directory " + cur);
    }
    if (i < dir.size()) cur += dir[i];
  }
}

// value of "key": <unsigned integer> in a flat JSON object (nlohmann's output
// or any equivalent whitespace); json::at throws when a key is missing
uint64_t json_u64(const std::string& text, const char* key) {
  const std::string q = std::string("\"") + key + "\"";
  size_t at = text.find(q);
  if (at == std::string::npos) throw std::runtime_error(std::string("graph_meta.json: key '") + key + "' not found");
  at = text.find(':', at + q.size());
  if (at == std::string::npos) throw std::runtime_error("graph_meta.json: malformed");
  ++at;
  while (at < text.size() && (text[at] == ' ' || text[at] == '\t' || text[at] == '\n' || text[at] == '\r')) ++at;
  if (at >= text.size() || text[at] < '0' || text[at] > '9')
    throw std::runtime_error(std::string("graph_meta.json: '") + key + "' is not an unsigned integer");
  uint64_t v = 0;
  while (at < text.size() && text[at] >= '0' && text[at] <= '9') v = v * 10 + uint64_t(text[at++] - '0');
  return v;
}

}  // namespace

extern "C" {

int lgd_write_graph(const char* dir, const uint32_t* edges, uint64_t num_edges, uint64_t num_nodes,
                    uint64_t num_relations) {
  return lgd::guarded([&] {
    if (!dir) throw std::invalid_argument("null directory");
    if (num_edges && !edges) throw std::invalid_argument("null edge array");
    make_dirs(dir);
    const std::string bin = join(dir, "edges.bin");
    FILE* f = std::fopen(bin.c_str(), "wb");
    if (!f) throw std::runtime_error("cannot write " + bin);
    const size_t n = num_edges ? std::fwrite(edges, 12, num_edges, f) : 0;
    const bool ok = std::fclose(f) == 0 && n == num_edges;
    if (!ok) throw std::runtime_error("short write to edges.bin");
    const std::string meta = join(dir, "graph_meta.json");
    FILE* m = std::fopen(meta.c_str(), "w");
    if (!m) throw std::runtime_error("cannot write graph_meta.json");
    std::fprintf(m, "{\n  \"num_edges\": %llu,\n  \"num_nodes\": %llu,\n  \"num_relations\": %llu\n}\n",
                 (unsigned long long)num_edges, (unsigned long long)num_nodes,
                 (unsigned long long)num_relations);
    if (std::fclose(m) != 0) throw std::runtime_error("cannot write graph_meta.json");
  });
}

int lgd_read_graph_meta(const char* dir, uint64_t* num_edges, uint64_t* num_nodes,
                        uint64_t* num_relations) {
  return lgd::guarded([&] {
    if (!dir) throw std::invalid_argument("null directory");
    const std::string meta = join(dir, "graph_meta.json");
    FILE* m = std::fopen(meta.c_str(), "r");
    if (!m) throw std::runtime_error(std::string("missing graph_meta.json in ") + dir);
    std::string text;
    char buf[4096];
    size_t got;
    while ((got = std::fread(buf, 1, sizeof buf, m)) > 0) text.append(buf, got);
    std::fclose(m);
    const uint64_t V = json_u64(text, "num_nodes"), R = json_u64(text, "num_relations");
    const uint64_t E = json_u64(text, "num_edges");
    if (num_nodes) *num_nodes = V;
    if (num_relations) *num_relations = R;
    if (num_edges) *num_edges = E;
  });
}

int lgd_read_graph(const char* dir, uint32_t* edges_out, uint64_t num_edges) {
  return lgd::guarded([&] {
    if (!dir) throw std::invalid_argument("null directory");
    if (num_edges && !edges_out) throw std::invalid_argument("null edge array");
    const std::string bin = join(dir, "edges.bin");
    FILE* f = std::fopen(bin.c_str(), "rb");
    if (!f) throw std::runtime_error(std::string("missing edges.bin in ") + dir);
    const size_t n = num_edges ? std::fread(edges_out, 12, num_edges, f) : 0;
    std::fclose(f);
    if (n != num_edges) throw std::runtime_error("edges.bin shorter than metadata claims");
  });
}

}  // extern "C"
