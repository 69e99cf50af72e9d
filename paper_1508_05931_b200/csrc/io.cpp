// Ingest: host loaders for the hull path's input.
//
// * plain XY text and the OBJ vertex subset restate the reference's loaders
//   (datagen.hpp:111-174: load_points, load_obj_projected) with the same
//   parser (std::from_chars), the same skipped lines and the same errors
//   (ParseError with its line number, IoError, EmptyInput), mapped to status
//   codes; the message is kept per thread (gscan_io_error);
// * a binary SoA file ("GSCANSOA", uint64 n, n x-doubles, n y-doubles,
//   little-endian) is the layout the device path consumes, read straight into
//   caller buffers (pinned host memory for the overlapped H2D of
//   gscan_hull_f64) with no parsing.
#include <algorithm>
#include <cerrno>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <string>
#include <system_error>
#include <vector>

#include "../../include/gscan.h"

namespace {

thread_local std::string g_io_err;

int io_fail(int code, const std::string& msg) {
  g_io_err = msg;
  return code;
}

const char* skip_ws(const char* p, const char* end) {
  while (p != end && (*p == ' ' || *p == '\t' || *p == '\r')) ++p;
  return p;
}

bool parse_double(const char*& p, const char* end, double& out) {
  const auto res = std::from_chars(p, end, out);
  if (res.ec != std::errc{}) return false;
  p = res.ptr;
  return true;
}

// load_points (datagen.hpp:111-134) / load_obj_projected (:145-168)
int parse_text(const std::string& path, bool obj, std::vector<double>& xs, std::vector<double>& ys) {
  std::ifstream in(path);
  if (!in) return io_fail(GSCAN_E_IO, "cannot open " + path);
  std::string line;
  size_t line_no = 0;
  while (std::getline(in, line)) {
    ++line_no;
    const char* p = line.data();
    const char* end = line.data() + line.size();
    p = skip_ws(p, end);
    double x, y;
    if (!obj) {
      if (p == end || *p == '#') continue;
      if (!parse_double(p, end, x)) return io_fail(GSCAN_E_PARSE, "bad x coordinate at line " + std::to_string(line_no));
      p = skip_ws(p, end);
      if (!parse_double(p, end, y)) return io_fail(GSCAN_E_PARSE, "bad y coordinate at line " + std::to_string(line_no));
      p = skip_ws(p, end);
      if (p != end) return io_fail(GSCAN_E_PARSE, "trailing characters at line " + std::to_string(line_no));
      if (!std::isfinite(x) || !std::isfinite(y))
        return io_fail(GSCAN_E_PARSE, "non-finite coordinate at line " + std::to_string(line_no));
    } else {
      if (p == end || p[0] != 'v') continue;
      if (p + 1 != end && p[1] != ' ' && p[1] != '\t') continue;
      p = skip_ws(p + 1, end);
      if (!parse_double(p, end, x)) return io_fail(GSCAN_E_PARSE, "bad vertex x at line " + std::to_string(line_no));
      p = skip_ws(p, end);
      if (!parse_double(p, end, y)) return io_fail(GSCAN_E_PARSE, "bad vertex y at line " + std::to_string(line_no));
      if (!std::isfinite(x) || !std::isfinite(y))
        return io_fail(GSCAN_E_PARSE, "non-finite vertex coordinate at line " + std::to_string(line_no));
    }
    xs.push_back(x);
    ys.push_back(y);
  }
  if (in.bad()) return io_fail(GSCAN_E_IO, "read error on " + path);
  if (xs.empty()) return io_fail(GSCAN_E_EMPTY_INPUT, (obj ? "no vertex lines in " : "no points in ") + path);
  return GSCAN_OK;
}

constexpr char kSoaMagic[8] = {'G', 'S', 'C', 'A', 'N', 'S', 'O', 'A'};

int soa_header(FILE* f, const char* path, uint64_t* n) {
  char magic[8];
  if (fread(magic, 1, 8, f) != 8 || memcmp(magic, kSoaMagic, 8) != 0)
    return io_fail(GSCAN_E_PARSE, std::string("not a GSCANSOA file: ") + path);
  if (fread(n, 8, 1, f) != 1) return io_fail(GSCAN_E_PARSE, std::string("truncated header: ") + path);
  return GSCAN_OK;
}

}  // namespace

extern "C" {

const char* gscan_io_error(void) { return g_io_err.c_str(); }

void gscan_free(void* p) { free(p); }

int gscan_load(const char* path, int format, double** xs, double** ys, uint64_t* n) {
  if (!path || !xs || !ys || !n) return io_fail(GSCAN_E_INVALID, "null argument");
  *xs = *ys = nullptr;
  *n = 0;
  if (format == GSCAN_FMT_SOA) {
    uint64_t m = 0;
    int rc = gscan_soa_count(path, &m);
    if (rc) return rc;
    double* a = (double*)malloc(std::max<uint64_t>(m, 1) * 8);
    double* b = (double*)malloc(std::max<uint64_t>(m, 1) * 8);
    if (!a || !b) { free(a); free(b); return io_fail(GSCAN_E_IO, "out of host memory"); }
    rc = gscan_soa_read(path, a, b, m);
    if (rc) { free(a); free(b); return rc; }
    *xs = a; *ys = b; *n = m;
    return GSCAN_OK;
  }
  if (format != GSCAN_FMT_XY && format != GSCAN_FMT_OBJ) return io_fail(GSCAN_E_INVALID, "unknown format");
  std::vector<double> vx, vy;
  const int rc = parse_text(path, format == GSCAN_FMT_OBJ, vx, vy);
  if (rc) return rc;
  double* a = (double*)malloc(vx.size() * 8);
  double* b = (double*)malloc(vy.size() * 8);
  if (!a || !b) { free(a); free(b); return io_fail(GSCAN_E_IO, "out of host memory"); }
  memcpy(a, vx.data(), vx.size() * 8);
  memcpy(b, vy.data(), vy.size() * 8);
  *xs = a; *ys = b; *n = vx.size();
  return GSCAN_OK;
}

int gscan_soa_count(const char* path, uint64_t* n) {
  if (!path || !n) return io_fail(GSCAN_E_INVALID, "null argument");
  FILE* f = fopen(path, "rb");
  if (!f) return io_fail(GSCAN_E_IO, std::string("cannot open ") + path);
  const int rc = soa_header(f, path, n);
  fclose(f);
  if (!rc && *n == 0) return io_fail(GSCAN_E_EMPTY_INPUT, std::string("no points in ") + path);
  return rc;
}

int gscan_soa_read(const char* path, double* xs, double* ys, uint64_t n) {
  if (!path || ((!xs || !ys) && n)) return io_fail(GSCAN_E_INVALID, "null argument");
  FILE* f = fopen(path, "rb");
  if (!f) return io_fail(GSCAN_E_IO, std::string("cannot open ") + path);
  uint64_t m = 0;
  int rc = soa_header(f, path, &m);
  if (!rc && m != n) rc = io_fail(GSCAN_E_INVALID, "point count differs from the file's");
  if (!rc && (fread(xs, 8, n, f) != n || fread(ys, 8, n, f) != n))
    rc = io_fail(GSCAN_E_PARSE, std::string("truncated data: ") + path);
  fclose(f);
  return rc;
}

int gscan_save_soa(const char* path, const double* xs, const double* ys, uint64_t n) {
  if (!path || ((!xs || !ys) && n)) return io_fail(GSCAN_E_INVALID, "null argument");
  FILE* f = fopen(path, "wb");
  if (!f) return io_fail(GSCAN_E_IO, std::string("cannot create ") + path);
  bool ok = fwrite(kSoaMagic, 1, 8, f) == 8 && fwrite(&n, 8, 1, f) == 1 &&
            fwrite(xs, 8, n, f) == n && fwrite(ys, 8, n, f) == n;
  ok = (fclose(f) == 0) && ok;
  return ok ? GSCAN_OK : io_fail(GSCAN_E_IO, std::string("write error on ") + path);
}

}  // extern "C"
