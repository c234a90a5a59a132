// quake_apply — the reference CLI's `apply` subcommand on the GPU path.
//
//   quake_apply [apply] --op softmax|gelu|logistic|exp --input IN --output OUT
//               [--kernel exact|quake|quake2] [--format csv|raw] [--cols N]
//               [--temperature T] [--bias on|off|auto] [--coeffs continuity|minimax]
//               [--devices 0,1,...]
//
// Same options, defaults and exit codes as the reference (tools/quake_cli.cpp:
// 246-296, 350-449: 0 ok, 2 usage / parse / invalid argument, 3 I/O), with the
// buffer formats of quake_b200/io.hpp. The operators are the drop-in quake::
// functions (include/quake_b200/quake.hpp), i.e. the sm_100a kernels;
// `--devices` shards rows / elements over several GPUs (qk_set_devices).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <optional>
#include <string>
#include <vector>

#include "quake_b200/io.hpp"
#include "quake_b200/quake.hpp"

namespace {

constexpr int kExitOk = 0;
constexpr int kExitUsage = 2;
constexpr int kExitIo = 3;

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct Args {
  std::string op;
  std::string kernel = "quake";
  std::string input;
  std::string output;
  std::string format = "csv";
  std::string bias = "auto";
  std::string coeffs = "continuity";
  std::string devices;
  size_t cols = 0;  // 0 = one row spanning the whole buffer
  float temperature = 1.0f;
};

quake::KernelChoice parse_kernel(const std::string& s) {
  if (s == "exact") return quake::KernelChoice::Exact;
  if (s == "quake") return quake::KernelChoice::Quake;
  if (s == "quake2") return quake::KernelChoice::Quake2;
  throw UsageError("unknown kernel: " + s);
}

std::optional<bool> parse_bias(const std::string& s) {
  if (s.empty() || s == "auto") return std::nullopt;
  if (s == "on") return true;
  if (s == "off") return false;
  throw UsageError("--bias must be on, off, or auto");
}

quake::QuadCoeffs parse_quad(const std::string& s) {
  if (s == "continuity") return quake::QuadCoeffs::continuity();
  if (s == "minimax") return quake::QuadCoeffs::minimax();
  throw UsageError("--coeffs must be continuity or minimax");
}

quake::io::BufferFormat parse_format(const std::string& s) {
  if (s == "csv") return quake::io::BufferFormat::Csv;
  if (s == "raw") return quake::io::BufferFormat::Raw;
  throw UsageError("--format must be csv or raw");
}

Args parse_args(int argc, char** argv) {
  Args a;
  int i = 1;
  if (i < argc && std::strcmp(argv[i], "apply") == 0) ++i;
  auto value = [&](const char* flag) -> std::string {
    if (i + 1 >= argc) throw UsageError(std::string(flag) + " needs a value");
    return argv[++i];
  };
  for (; i < argc; ++i) {
    const std::string f = argv[i];
    if (f == "--op") a.op = value("--op");
    else if (f == "--kernel") a.kernel = value("--kernel");
    else if (f == "--input") a.input = value("--input");
    else if (f == "--output") a.output = value("--output");
    else if (f == "--format") a.format = value("--format");
    else if (f == "--bias") a.bias = value("--bias");
    else if (f == "--coeffs") a.coeffs = value("--coeffs");
    else if (f == "--devices") a.devices = value("--devices");
    else if (f == "--cols") {
      const std::string v = value("--cols");
      char* end = nullptr;
      const unsigned long long c = std::strtoull(v.c_str(), &end, 10);
      if (end == v.c_str() || *end) throw UsageError("--cols must be a non-negative integer");
      a.cols = static_cast<size_t>(c);
    } else if (f == "--temperature") {
      const std::string v = value("--temperature");
      char* end = nullptr;
      a.temperature = std::strtof(v.c_str(), &end);
      if (end == v.c_str() || *end) throw UsageError("--temperature must be a number");
    } else if (f == "-h" || f == "--help") {
      std::printf(
          "quake_apply --op softmax|gelu|logistic|exp --input IN --output OUT [--kernel "
          "exact|quake|quake2] [--format csv|raw] [--cols N] [--temperature T] [--bias "
          "on|off|auto] [--coeffs continuity|minimax] [--devices 0,1,...]\n");
      std::exit(kExitOk);
    } else {
      throw UsageError("unknown option: " + f);
    }
  }
  if (a.op.empty()) throw UsageError("--op is required");
  if (a.input.empty()) throw UsageError("--input is required");
  if (a.output.empty()) throw UsageError("--output is required");
  return a;
}

void set_devices(const std::string& list) {
  if (list.empty()) return;
  std::vector<int> devs;
  size_t pos = 0;
  while (pos <= list.size()) {
    const size_t comma = list.find(',', pos);
    const std::string tok = list.substr(pos, comma == std::string::npos ? std::string::npos
                                                                         : comma - pos);
    char* end = nullptr;
    const long d = std::strtol(tok.c_str(), &end, 10);
    if (tok.empty() || *end) throw UsageError("--devices must be a comma-separated list");
    devs.push_back(static_cast<int>(d));
    if (comma == std::string::npos) break;
    pos = comma + 1;
  }
  if (qk_set_devices(devs.data(), static_cast<int>(devs.size())) != QK_OK) {
    throw UsageError(std::string("--devices: ") + qk_last_error());
  }
}

int run_apply(const Args& a) {
  // reference order (quake_cli.cpp:259-296): format, kernel, bias, then the
  // input is read; the op is dispatched only afterwards (an unknown op with a
  // missing input is an I/O error, exit 3), and --coeffs is parsed only where
  // it is used (softmax, exp with QuAKE2), so other ops ignore a bad value
  const auto format = parse_format(a.format);
  const auto kernel = parse_kernel(a.kernel);
  const auto bias = parse_bias(a.bias);
  set_devices(a.devices);
  const std::vector<float> in = quake::io::read_buffer(a.input, format);
  std::vector<float> out(in.size());
  if (a.op == "softmax") {
    quake::SoftmaxParams params;
    params.temperature = a.temperature;
    params.centering_bias = bias;
    params.quad = parse_quad(a.coeffs);
    quake::softmax_rows(in, a.cols == 0 ? in.size() : a.cols, params, kernel, out);
  } else if (a.op == "gelu") {
    quake::gelu_buffer(in, out, kernel, bias);
  } else if (a.op == "logistic") {
    quake::logistic_buffer(in, out, kernel, bias);
  } else if (a.op == "exp") {
    if (kernel == quake::KernelChoice::Exact) {
      if (qk_status s = qk_exp_buffer(in.data(), in.size(), out.data(), out.size(), QK_EXACT)) {
        if (qk_is_invalid_argument(s)) throw std::invalid_argument(qk_last_error());
        throw std::runtime_error(qk_last_error());
      }
    } else {
      const quake::AffineCoeffs c =
          quake::natural_exp_coeffs(quake::resolve_centering_bias(kernel, bias));
      const quake::ClampRange r = quake::clamp_for(c);
      if (kernel == quake::KernelChoice::Quake) {
        quake::quake_buffer(in, out, c, r);
      } else {
        quake::quake2_buffer(in, out, c, parse_quad(a.coeffs), r);
      }
    }
  } else {
    throw UsageError("unknown op: " + a.op);
  }
  quake::io::write_buffer(a.output, out, format);
  return kExitOk;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    return run_apply(parse_args(argc, argv));
  } catch (const UsageError& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return kExitUsage;
  } catch (const quake::io::ParseError& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return kExitUsage;
  } catch (const quake::io::IoError& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return kExitIo;
  } catch (const std::invalid_argument& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return kExitUsage;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return kExitUsage;
  }
}
