// Minimal restatement of the Eigen-free helpers of the reference's
// tensor.cpp (is_permutation, identity/inverse permutation, shape_numel,
// row_major_strides, DenseTensor::flat_index) so that the reference's own
// integer translation units link without Eigen.  Test infrastructure only.
#include <numeric>
#include "tucomp/tensor.hpp"

namespace tucomp {
bool is_permutation(const ModePermutation& p) {
    std::vector<char> hit(p.size(), 0);
    for (auto v : p) {
        if (v >= p.size() || hit[v]) return false;
        hit[v] = 1;
    }
    return true;
}
ModePermutation identity_permutation(std::size_t d) {
    ModePermutation p(d);
    std::iota(p.begin(), p.end(), std::size_t{0});
    return p;
}
ModePermutation inverse_permutation(const ModePermutation& p) {
    ModePermutation q(p.size());
    for (std::size_t i = 0; i < p.size(); ++i) q[p[i]] = i;
    return q;
}
std::size_t shape_numel(const Shape& s) {
    std::size_t n = 1;
    for (auto v : s) n *= v;
    return n;
}
std::vector<std::size_t> row_major_strides(const Shape& s) {
    std::vector<std::size_t> st(s.size());
    std::size_t acc = 1;
    for (std::size_t i = s.size(); i-- > 0;) { st[i] = acc; acc *= s[i]; }
    return st;
}
template <class T>
std::size_t DenseTensor<T>::flat_index(std::span<const std::size_t> m) const {
    std::size_t f = 0;
    for (std::size_t i = 0; i < m.size(); ++i) f = f * shape_[i] + m[i];
    return f;
}
template class DenseTensor<float>;
template class DenseTensor<double>;
}  // namespace tucomp
