#include "tucomp/pipeline.hpp"
#include <cmath>
#include <cstdio>
int main() {
  std::vector<double> x(16 * 16 * 16);
  for (std::size_t i = 0; i < x.size(); ++i) x[i] = std::sin(0.1 * i) + 0.01 * std::cos(1.7 * i);
  tucomp::container::SourceBuffer src{std::span<const std::uint8_t>(reinterpret_cast<const std::uint8_t*>(x.data()), x.size()*8), tucomp::container::Dtype::float64, {16, 16, 16}, 0};
  tucomp::pipeline::Params p; p.target_re = 1e-2;
  try { auto r = tucomp::pipeline::compress(src, p); std::printf("bytes %zu\n", r.container.size()); }
  catch (const tucomp::Error& e) { std::printf("error: %s\n", e.what()); }
}
