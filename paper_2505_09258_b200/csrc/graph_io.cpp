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

// ------------------------------------------------------------------ ingest
// ingest (graph.cpp:39-118): TSV edge list, 2 (pairs) or 3 (triples) decimal
// columns separated by tabs / spaces, '#'-first lines and blank lines
// skipped, '\r\n' accepted.  Chunks of lines are parsed by host threads; the
// first malformed line in file order raises the reference's ParseError text.
// remap_ids: dense ids in first-appearance order (src, rel, dst per line),
// done in file order after the parallel parse.
#include <algorithm>
#include <charconv>
#include <thread>
#include <unordered_map>
#include <vector>

namespace {

struct ParseChunk {
  const char* begin;
  const char* end;
  std::vector<uint64_t> cols;  // want_cols per edge
  uint64_t lines = 0;
  uint64_t err_line = 0;       // 1-based within the chunk, 0 = none
  std::string err;
};

bool parse_u64(const char* b, const char* e, uint64_t& out) {
  if (b == e) return false;
  auto [p, ec] = std::from_chars(b, e, out);
  return ec == std::errc{} && p == e;
}

void parse_chunk(ParseChunk& c, int want) {
  const char* p = c.begin;
  while (p < c.end) {
    const char* nl = static_cast<const char*>(std::memchr(p, '\n', c.end - p));
    const char* le = nl ? nl : c.end;
    ++c.lines;
    const char* q = p;
    const char* qe = le;
    if (qe > q && qe[-1] == '\r') --qe;
    p = nl ? nl + 1 : c.end;
    if (q == qe || *q == '#') continue;
    const char* fb[4];
    const char* fe[4];
    int nf = 0;
    while (q < qe) {
      while (q < qe && (*q == '\t' || *q == ' ')) ++q;
      if (q >= qe) break;
      const char* s = q;
      while (q < qe && *q != '\t' && *q != ' ') ++q;
      if (nf < 4) {
        fb[nf] = s;
        fe[nf] = q;
      }
      ++nf;
    }
    if (nf == 0) continue;
    if (nf != want) {
      c.err_line = c.lines;
      c.err = ": expected " + std::to_string(want) + " columns, got " + std::to_string(nf);
      return;
    }
    for (int f = 0; f < nf; ++f) {
      uint64_t v;
      if (!parse_u64(fb[f], fe[f], v)) {
        c.err_line = c.lines;
        c.err = ": malformed integer field '" + std::string(fb[f], fe[f]) + "'";
        return;
      }
      c.cols.push_back(v);
    }
  }
}

}  // namespace

extern "C" {

int lgd_ingest_tsv(const char* path, int triples, int remap_ids, int threads, uint32_t** edges_out,
                   uint64_t* num_edges, uint64_t* num_nodes, uint64_t* num_relations) {
  return lgd::guarded([&] {
    if (!path || !edges_out || !num_edges) throw std::invalid_argument("null argument");
    *edges_out = nullptr;
    FILE* f = std::fopen(path, "rb");
    if (!f) throw std::runtime_error(std::string("cannot open edge file: ") + path);
    std::string text;
    {
      std::fseek(f, 0, SEEK_END);
      const long sz = std::ftell(f);
      std::fseek(f, 0, SEEK_SET);
      text.resize(sz > 0 ? (size_t)sz : 0);
      const size_t got = sz > 0 ? std::fread(&text[0], 1, (size_t)sz, f) : 0;
      std::fclose(f);
      text.resize(got);
    }
    const int want = triples ? 3 : 2;
    int T = threads > 0 ? threads : (int)std::max(1u, std::thread::hardware_concurrency());
    T = (int)std::min<size_t>(T, std::max<size_t>(1, text.size() / (64 << 10)));  // >= 64 KB each
    std::vector<ParseChunk> chunks(T);
    const char* b = text.data();
    const char* e = b + text.size();
    for (int t = 0; t < T; ++t) {  // cut at line starts
      const char* cb = t == 0 ? b : chunks[t - 1].end;
      const char* ce = t == T - 1 ? e : b + text.size() * (t + 1) / T;
      if (ce < cb) ce = cb;
      if (t < T - 1) {
        const char* nl = static_cast<const char*>(std::memchr(ce, '\n', e - ce));
        ce = nl ? nl + 1 : e;
      }
      chunks[t].begin = cb;
      chunks[t].end = ce;
    }
    std::vector<std::thread> pool;
    for (int t = 1; t < T; ++t) pool.emplace_back(parse_chunk, std::ref(chunks[t]), want);
    parse_chunk(chunks[0], want);
    for (auto& th : pool) th.join();
    uint64_t lines_before = 0, E = 0;
    for (const auto& c : chunks) {
      if (c.err_line)
        throw std::runtime_error("line " + std::to_string(lines_before + c.err_line) + c.err);
      lines_before += c.lines;
      E += c.cols.size() / want;
    }
    if (E == 0) throw std::runtime_error(std::string("edge file has no edges: ") + path);
    uint32_t* out = static_cast<uint32_t*>(std::malloc(E * 12));
    if (!out) throw std::runtime_error("out of host memory");
    uint64_t max_node = 0, max_rel = 0, k = 0;
    std::unordered_map<uint64_t, uint32_t> nmap, rmap;
    auto node = [&](uint64_t raw) -> uint32_t {
      if (!remap_ids) {
        max_node = std::max(max_node, raw);
        return static_cast<uint32_t>(raw);
      }
      return nmap.emplace(raw, static_cast<uint32_t>(nmap.size())).first->second;
    };
    auto rel = [&](uint64_t raw) -> uint32_t {
      if (!remap_ids) {
        max_rel = std::max(max_rel, raw);
        return static_cast<uint32_t>(raw);
      }
      return rmap.emplace(raw, static_cast<uint32_t>(rmap.size())).first->second;
    };
    for (const auto& c : chunks)
      for (size_t i = 0; i < c.cols.size(); i += want, ++k) {
        if (triples) {
          out[3 * k] = node(c.cols[i]);
          out[3 * k + 1] = rel(c.cols[i + 1]);
          out[3 * k + 2] = node(c.cols[i + 2]);
        } else {
          out[3 * k] = node(c.cols[i]);
          out[3 * k + 1] = LGD_NO_RELATION;
          out[3 * k + 2] = node(c.cols[i + 1]);
        }
      }
    *edges_out = out;
    *num_edges = E;
    if (num_nodes) *num_nodes = remap_ids ? nmap.size() : max_node + 1;
    if (num_relations) *num_relations = remap_ids ? rmap.size() : (triples ? max_rel + 1 : 0);
  });
}

void lgd_free_edges(uint32_t* edges) { std::free(edges); }

}  // extern "C"
