// `tucomp` command-line driver on the B200 library: the four subcommands of the
// reference CLI (proj/tools/tucomp_main.cpp:276-350: compress, decompress, info,
// sweep) with the same flags, report lines and exit behaviour, built only on the
// public drop-in surface include/tucomp/pipeline.hpp (-> libtucomp_b200.so).
//
// Differences, all deliberate:
//  * no CLI11 (absent from the image): a small table-driven parser accepting
//    `--flag value` and `--flag=value`; usage errors exit 2 (CLI11's codes
//    differ per error kind), runtime errors print "error: <what>" and exit 1
//    exactly as tucomp_main.cpp:345-348;
//  * measure_error (tucomp_main.cpp:121-135) runs on the device
//    (pipeline::measure_sse: ingest + decompress + sse_between there).
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <functional>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "tucomp/pipeline.hpp"

using namespace tucomp;

namespace {

struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// ------------------------------------------------------------------ files
std::vector<std::uint8_t> slurp(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) throw Error("cannot open " + path);
    f.seekg(0, std::ios::end);
    const auto n = static_cast<std::size_t>(f.tellg());
    f.seekg(0);
    std::vector<std::uint8_t> b(n);
    if (n) f.read(reinterpret_cast<char*>(b.data()), static_cast<std::streamsize>(n));
    return b;
}

void spill(const std::string& path, std::span<const std::uint8_t> b) {
    std::ofstream f(path, std::ios::binary);
    if (!f) throw Error("cannot open " + path + " for writing");
    f.write(reinterpret_cast<const char*>(b.data()), static_cast<std::streamsize>(b.size()));
    if (!f) throw Error("write to " + path + " failed");
}

// ------------------------------------------------------------------ lists
std::vector<std::string> split_commas(const std::string& s) {
    std::vector<std::string> v;
    std::string cur;
    std::istringstream in(s);
    while (std::getline(in, cur, ',')) v.push_back(cur);
    return v;
}

Shape to_shape(const std::string& s) {
    Shape sh;
    for (const auto& t : split_commas(s)) sh.push_back(std::stoull(t));
    if (sh.empty()) throw Error("empty shape");
    return sh;
}

ModePermutation to_perm(const std::string& s) {  // 1-based on the command line
    ModePermutation p;
    for (const auto& t : split_commas(s)) {
        const auto v = std::stoull(t);
        if (v == 0) throw Error("mode orders are 1-based");
        p.push_back(v - 1);
    }
    return p;
}

std::vector<double> to_grid(const std::string& s) {
    std::vector<double> g;
    for (const auto& t : split_commas(s)) g.push_back(std::stod(t));
    return g;
}

// ------------------------------------------------------------------ options
struct Options {
    std::string input, output, shape, dtype = "float64";
    double target_re = -1, target_sse = -1, rtmss = errormodel::kDefaultRtmss;
    int threads = 1;
    std::string vectorization = "lex", coder = "ac", storage_order, mode_order;
    std::uint64_t skip_bytes = 0, block_size = 0;
    bool no_split = false, simple = false, f32 = false, machine = false, no_verify = false;
    std::string re_grid, rtmss_grid;
};

struct Spec {
    enum Kind { Str, Dbl, Int, U64, Flag } kind;
    void* dst;
    bool required;
};

class Parser {
public:
    void add(std::initializer_list<const char*> names, Spec s) {
        const int id = static_cast<int>(specs_.size());
        specs_.push_back(s);
        primary_.push_back(*names.begin());
        for (const char* n : names) names_[n] = id;
    }
    void parse(int argc, char** argv, int first) {
        std::vector<bool> seen(specs_.size(), false);
        for (int i = first; i < argc; ++i) {
            std::string a = argv[i], val;
            bool has_val = false;
            if (const auto eq = a.find('='); a.rfind("--", 0) == 0 && eq != std::string::npos) {
                val = a.substr(eq + 1);
                a = a.substr(0, eq);
                has_val = true;
            }
            const auto it = names_.find(a);
            if (it == names_.end()) throw UsageError("unknown argument " + a);
            const Spec& s = specs_[it->second];
            seen[it->second] = true;
            if (s.kind == Spec::Flag) {
                if (has_val) throw UsageError(a + " takes no value");
                *static_cast<bool*>(s.dst) = true;
                continue;
            }
            if (!has_val) {
                if (i + 1 >= argc) throw UsageError(a + " needs a value");
                val = argv[++i];
            }
            try {
                switch (s.kind) {
                    case Spec::Str: *static_cast<std::string*>(s.dst) = val; break;
                    case Spec::Dbl: *static_cast<double*>(s.dst) = std::stod(val); break;
                    case Spec::Int: *static_cast<int*>(s.dst) = std::stoi(val); break;
                    case Spec::U64: *static_cast<std::uint64_t*>(s.dst) = std::stoull(val); break;
                    case Spec::Flag: break;
                }
            } catch (const std::logic_error&) {
                throw UsageError("bad value for " + a + ": " + val);
            }
        }
        for (std::size_t k = 0; k < specs_.size(); ++k)
            if (specs_[k].required && !seen[k]) throw UsageError(primary_[k] + " is required");
    }

private:
    std::vector<Spec> specs_;
    std::vector<std::string> primary_;
    std::map<std::string, int> names_;
};

void input_options(Parser& p, Options& o) {  // tucomp_main.cpp:284-306
    p.add({"-i", "--input"}, {Spec::Str, &o.input, true});
    p.add({"--shape"}, {Spec::Str, &o.shape, true});
    p.add({"--dtype"}, {Spec::Str, &o.dtype, false});
    p.add({"--skip-bytes"}, {Spec::U64, &o.skip_bytes, false});
    p.add({"--rtmss"}, {Spec::Dbl, &o.rtmss, false});
    p.add({"--threads"}, {Spec::Int, &o.threads, false});
    p.add({"--vectorization"}, {Spec::Str, &o.vectorization, false});
    p.add({"--storage-order"}, {Spec::Str, &o.storage_order, false});
    p.add({"--mode-order"}, {Spec::Str, &o.mode_order, false});
    p.add({"--coder"}, {Spec::Str, &o.coder, false});
    p.add({"--block-size"}, {Spec::U64, &o.block_size, false});
    p.add({"--no-split-planes"}, {Spec::Flag, &o.no_split, false});
    p.add({"--simple-factor-weights"}, {Spec::Flag, &o.simple, false});
    p.add({"--internal-float32"}, {Spec::Flag, &o.f32, false});
}

// to_params (tucomp_main.cpp:77-101)
pipeline::Params params_of(const Options& o) {
    pipeline::Params p;
    if (o.target_re >= 0) {
        if (o.target_re == 0)
            throw Error("--target-re 0 requests lossless output; this is a lossy "
                        "compressor, pick a small positive target instead");
        p.target_re = o.target_re;
    }
    if (o.target_sse >= 0) p.target_sse = o.target_sse;
    p.rtmss = o.rtmss;
    p.threads = o.threads;
    const auto m = vectorize::method_from_name(o.vectorization);
    if (!m) throw Error("unknown vectorization method " + o.vectorization);
    p.method = *m;
    const auto c = entropy::coder_from_name(o.coder);
    if (!c) throw Error("unknown coder " + o.coder);
    p.coder = *c;
    if (!o.storage_order.empty()) p.storage_order = to_perm(o.storage_order);
    if (!o.mode_order.empty()) p.mode_order = to_perm(o.mode_order);
    p.split_planes = !o.no_split;
    p.simple_factor_weights = o.simple;
    p.block_size = o.block_size;
    p.internal_float32 = o.f32;
    return p;
}

container::SourceBuffer source_of(const Options& o, std::span<const std::uint8_t> bytes) {
    const auto t = container::dtype_from_name(o.dtype);
    if (!t) throw Error("unknown dtype " + o.dtype);
    container::SourceBuffer s;
    s.bytes = bytes;
    s.dtype = *t;
    s.shape = to_shape(o.shape);
    s.skip_bytes = o.skip_bytes;
    return s;
}

struct Achieved {
    double sse = 0, re = 0;
};

Achieved achieved(const container::SourceBuffer& src, const pipeline::Params& p,
                  std::span<const std::uint8_t> cont, double norm_sq) {
    Achieved a;
    a.sse = pipeline::measure_sse(src, cont, p.internal_float32);
    a.re = norm_sq > 0 ? std::sqrt(a.sse / norm_sq) : 0.0;
    return a;
}

// ------------------------------------------------------------------ subcommands
void report(const pipeline::CompressResult& r, const Achieved& a, bool machine) {  // tucomp_main.cpp:137-170
    const double est = r.estimate.total();
    double fsum = 0;
    for (double f : r.estimate.factor_terms) fsum += f;
    auto& o = std::cout;
    o << "compressed size:     " << r.container.size() << " bytes\n"
      << "compression factor:  " << r.compression_factor() << "\n"
      << "achieved rel. error: " << a.re << " (measured)\n"
      << "achieved SSE:        " << a.sse << "\n"
      << "estimated rel. error:" << (r.norm_sq > 0 ? std::sqrt(est / r.norm_sq) : 0.0) << " (error model)\n"
      << "estimated SSE:       " << est << "\n"
      << "  truncation SSE:    " << r.estimate.truncation_sse << "\n"
      << "  core quant SSE:    " << r.estimate.core_quantization_sse << "\n"
      << "  factor terms SSE:  " << fsum << "\n"
      << "ranks:              ";
    for (auto k : r.ranks) o << " " << k;
    o << "\ntimes (ms): sthosvd " << r.times.sthosvd_ms << ", quantize " << r.times.quantize_ms << ", core encode "
      << r.times.core_encode_ms << ", factors " << r.times.factor_encode_ms << ", serialize " << r.times.serialize_ms
      << ", total " << r.times.total_ms << "\n"
      << "peak alloc estimate: " << r.peak_alloc_estimate << " bytes\n";
    if (r.ingest_precision_loss)
        o << "warning: 64-bit integer input exceeds the 53-bit double mantissa; "
             "values were rounded during ingest\n";
    if (!machine) return;
    o << "report.bytes " << r.container.size() << "\n"
      << "report.factor " << r.compression_factor() << "\n"
      << "report.achieved_re " << a.re << "\n"
      << "report.achieved_sse " << a.sse << "\n"
      << "report.estimate_sse " << est << "\n"
      << "report.comp_ms " << r.times.total_ms << "\n";
}

int run_compress(const Options& o) {  // tucomp_main.cpp:172-182
    if (o.target_re < 0 && o.target_sse < 0) throw Error("one of --target-re / --target-sse is required");
    if (o.target_re >= 0 && o.target_sse >= 0) throw Error("--target-re and --target-sse are mutually exclusive");
    const auto bytes = slurp(o.input);
    const auto src = source_of(o, bytes);
    const auto prm = params_of(o);
    const auto r = pipeline::compress(src, prm);
    Achieved a;
    if (!o.no_verify) a = achieved(src, prm, r.container, r.norm_sq);
    spill(o.output, r.container);
    report(r, a, o.machine);
    return 0;
}

int run_decompress(const Options& o) {  // tucomp_main.cpp:184-194
    const auto bytes = slurp(o.input);
    const auto r = pipeline::decompress(bytes, o.threads);
    spill(o.output, r.bytes);
    std::cout << "wrote " << r.bytes.size() << " bytes (" << container::dtype_name(r.dtype) << ", shape";
    for (auto v : r.shape) std::cout << " " << v;
    std::cout << ") in " << r.total_ms << " ms\n";
    return 0;
}

int run_info(const Options& o) {  // tucomp_main.cpp:196-228
    const auto bytes = slurp(o.input);
    const auto h = container::read_container(bytes).header;
    auto& s = std::cout;
    auto list = [&](const char* label, const std::vector<std::uint64_t>& v, std::uint64_t add) {
        s << label;
        for (auto x : v) s << " " << x + add;
        s << "\n";
    };
    s << "format version:  " << int(container::kFormatVersion) << "\n"
      << "source dtype:    " << container::dtype_name(h.source_dtype) << "\n"
      << "internal:        " << (h.internal_float32 ? "float32" : "float64") << "\n"
      << "order:           " << h.order() << "\n";
    list("mode sizes:     ", h.mode_sizes, 0);
    list("ranks:          ", h.ranks, 0);
    list("processing order:", {h.processing_order.begin(), h.processing_order.end()}, 1);
    list("storage order:   ", {h.storage_order.begin(), h.storage_order.end()}, 1);
    s << "vectorization:   " << vectorize::method_name(h.method) << "\n"
      << "entropy coder:   " << entropy::coder_name(h.coder) << "\n"
      << "block size:      " << h.block_size << "\n"
      << "scale exponent:  " << h.core_scale_exponent << "\n"
      << "rtmss:           " << h.rtmss << "\n"
      << "split planes:    " << (h.split_planes ? "yes" : "no") << "\n"
      << "factor weights:  " << (h.simple_weights ? "slice-norm" : "alpha") << "\n";
    if (h.zero_flag) s << "content:         constant zero\n";
    s << "recorded error:  " << (h.norm_sq > 0 ? std::sqrt(h.estimate_sse / h.norm_sq) : 0.0)
      << " relative (estimate; recorded)\n"
      << "compressed size: " << bytes.size() << " bytes\n";
    const std::uint64_t original = h.element_count() * container::dtype_size(h.source_dtype);
    s << "original size:   " << original << " bytes\n"
      << "factor:          " << double(original) / double(bytes.size()) << "\n";
    return 0;
}

int run_sweep(const Options& o) {  // tucomp_main.cpp:230-272
    const auto bytes = slurp(o.input);
    const auto src = source_of(o, bytes);
    const auto res = to_grid(o.re_grid);
    const auto rts = o.rtmss_grid.empty() ? std::vector<double>{o.rtmss} : to_grid(o.rtmss_grid);
    std::ofstream file;
    std::ostream* out = &std::cout;
    if (!o.output.empty()) {
        file.open(o.output);
        if (!file) throw Error("cannot open " + o.output + " for writing");
        out = &file;
    }
    *out << "target_re,achieved_re,factor,rtmss,comp_ms,decomp_ms\n";
    for (const double rt : rts)
        for (const double re : res) {
            Options cell = o;
            cell.target_re = re;
            cell.target_sse = -1;
            cell.rtmss = rt;
            try {
                const auto prm = params_of(cell);
                const auto r = pipeline::compress(src, prm);
                const auto t0 = std::chrono::steady_clock::now();
                (void)pipeline::decompress(r.container, prm.threads);
                const double dms =
                    std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
                const auto a = achieved(src, prm, r.container, r.norm_sq);
                *out << re << "," << a.re << "," << r.compression_factor() << "," << rt << "," << r.times.total_ms
                     << "," << dms << "\n";
            } catch (const std::exception& e) {
                std::cerr << "sweep cell re=" << re << " rtmss=" << rt << " failed: " << e.what() << "\n";
                *out << re << ",nan,nan," << rt << ",nan,nan\n";
            }
        }
    return 0;
}

const char* kUsage =
    "Tucker-based lossy compressor for dense multidimensional arrays (B200)\n"
    "usage: tucomp <compress|decompress|info|sweep> [options]\n"
    "  compress   -i FILE --shape A,B,.. -o OUT (--target-re X | --target-sse X) [--dtype T]\n"
    "             [--skip-bytes N] [--rtmss X] [--threads N] [--vectorization lex|zigzag|zorder]\n"
    "             [--storage-order 3,1,2] [--mode-order ..] [--coder ac|rans] [--block-size N]\n"
    "             [--no-split-planes] [--simple-factor-weights] [--internal-float32] [--machine] [--no-verify]\n"
    "  decompress -i CONTAINER -o OUT [--threads N]\n"
    "  info       -i CONTAINER\n"
    "  sweep      (compress's input options) --target-re-grid X,Y,.. [--rtmss-grid ..] [-o CSV]\n";

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2 || std::string(argv[1]) == "-h" || std::string(argv[1]) == "--help") {
        (argc < 2 ? std::cerr : std::cout) << kUsage;
        return argc < 2 ? 2 : 0;
    }
    const std::string cmd = argv[1];
    Options o;
    Parser p;
    std::function<int(const Options&)> run;
    if (cmd == "compress") {
        input_options(p, o);
        p.add({"-o", "--output"}, {Spec::Str, &o.output, true});
        p.add({"--target-re"}, {Spec::Dbl, &o.target_re, false});
        p.add({"--target-sse"}, {Spec::Dbl, &o.target_sse, false});
        p.add({"--machine"}, {Spec::Flag, &o.machine, false});
        p.add({"--no-verify"}, {Spec::Flag, &o.no_verify, false});
        run = run_compress;
    } else if (cmd == "decompress") {
        p.add({"-i", "--input"}, {Spec::Str, &o.input, true});
        p.add({"-o", "--output"}, {Spec::Str, &o.output, true});
        p.add({"--threads"}, {Spec::Int, &o.threads, false});
        run = run_decompress;
    } else if (cmd == "info") {
        p.add({"-i", "--input"}, {Spec::Str, &o.input, true});
        run = run_info;
    } else if (cmd == "sweep") {
        input_options(p, o);
        p.add({"-o", "--output"}, {Spec::Str, &o.output, false});
        p.add({"--target-re-grid"}, {Spec::Str, &o.re_grid, true});
        p.add({"--rtmss-grid"}, {Spec::Str, &o.rtmss_grid, false});
        run = run_sweep;
    } else {
        std::cerr << "unknown subcommand " << cmd << "\n" << kUsage;
        return 2;
    }
    try {
        p.parse(argc, argv, 2);
    } catch (const UsageError& e) {
        std::cerr << cmd << ": " << e.what() << "\n" << kUsage;
        return 2;
    }
    try {
        return run(o);
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}
