// TEST INFRASTRUCTURE ONLY (oracle build shim) -- never linked into the product.
//
// The reference (`/root/reference/proj/include/stemtn/tree.hpp:9,17`) uses
// `boost::multiprecision::cpp_int` for exact contraction costs. Boost is not in
// this image, and a 128-bit integer overflows while planning 53-qubit circuits,
// so this is a small exact arbitrary-precision signed integer covering the
// operations the reference headers use: construction from built-in integers,
// + - * (and compound forms), shifts, comparisons, msb() and convert_to<T>().
#pragma once

#include <cstdint>
#include <type_traits>
#include <vector>

namespace boost {
namespace multiprecision {

class cpp_int {
 public:
  cpp_int() = default;
  template <class T, class = std::enable_if_t<std::is_integral_v<T>>>
  cpp_int(T v) {  // NOLINT(google-explicit-constructor): mirrors boost
    unsigned long long mag;
    if constexpr (std::is_signed_v<T>) {
      negative_ = v < 0;
      mag = negative_ ? 0ull - (unsigned long long)(long long)v : (unsigned long long)v;
    } else {
      mag = (unsigned long long)v;
    }
    while (mag) {
      limbs_.push_back(std::uint32_t(mag & 0xffffffffu));
      mag >>= 32;
    }
  }

  template <class T>
  T convert_to() const {
    long double acc = 0;
    for (std::size_t i = limbs_.size(); i-- > 0;) acc = acc * 4294967296.0L + limbs_[i];
    return T(negative_ ? -acc : acc);
  }

  bool is_zero() const { return limbs_.empty(); }
  bool is_negative() const { return negative_; }
  const std::vector<std::uint32_t> &limbs() const { return limbs_; }

  cpp_int &operator+=(const cpp_int &o) {
    if (negative_ == o.negative_) {
      limbs_ = add(limbs_, o.limbs_);
    } else if (compare_mag(limbs_, o.limbs_) >= 0) {
      limbs_ = sub(limbs_, o.limbs_);
    } else {
      limbs_ = sub(o.limbs_, limbs_);
      negative_ = o.negative_;
    }
    normalize();
    return *this;
  }
  cpp_int &operator-=(const cpp_int &o) {
    cpp_int neg = o;
    if (!neg.limbs_.empty()) neg.negative_ = !neg.negative_;
    return *this += neg;
  }
  cpp_int &operator*=(const cpp_int &o) {
    std::vector<std::uint32_t> r(limbs_.size() + o.limbs_.size(), 0);
    for (std::size_t i = 0; i < limbs_.size(); ++i) {
      std::uint64_t carry = 0;
      for (std::size_t j = 0; j < o.limbs_.size(); ++j) {
        std::uint64_t cur = std::uint64_t(limbs_[i]) * o.limbs_[j] + r[i + j] + carry;
        r[i + j] = std::uint32_t(cur);
        carry = cur >> 32;
      }
      std::size_t k = i + o.limbs_.size();
      while (carry) {
        std::uint64_t cur = std::uint64_t(r[k]) + carry;
        r[k++] = std::uint32_t(cur);
        carry = cur >> 32;
      }
    }
    negative_ = negative_ != o.negative_;
    limbs_ = std::move(r);
    normalize();
    return *this;
  }
  cpp_int &operator<<=(unsigned s) {
    if (limbs_.empty()) return *this;
    unsigned whole = s / 32, bits = s % 32;
    std::vector<std::uint32_t> r(limbs_.size() + whole + 1, 0);
    for (std::size_t i = 0; i < limbs_.size(); ++i) {
      std::uint64_t v = std::uint64_t(limbs_[i]) << bits;
      r[i + whole] |= std::uint32_t(v);
      r[i + whole + 1] |= std::uint32_t(v >> 32);
    }
    limbs_ = std::move(r);
    normalize();
    return *this;
  }
  cpp_int &operator>>=(unsigned s) {  // magnitude shift (only used on non-negatives)
    unsigned whole = s / 32, bits = s % 32;
    if (whole >= limbs_.size()) {
      limbs_.clear();
      normalize();
      return *this;
    }
    std::vector<std::uint32_t> r(limbs_.size() - whole, 0);
    for (std::size_t i = 0; i < r.size(); ++i) {
      std::uint64_t v = limbs_[i + whole];
      if (i + whole + 1 < limbs_.size()) v |= std::uint64_t(limbs_[i + whole + 1]) << 32;
      r[i] = std::uint32_t(v >> bits);
    }
    limbs_ = std::move(r);
    normalize();
    return *this;
  }

  // Truncating division; the reference only divides costs by bond dimensions
  // (planner.hpp:471), so the divisor must fit in one 32-bit limb.
  cpp_int &operator/=(const cpp_int &o) {
    if (o.limbs_.size() != 1) __builtin_trap();
    std::uint64_t d = o.limbs_[0], rem = 0;
    for (std::size_t i = limbs_.size(); i-- > 0;) {
      std::uint64_t cur = (rem << 32) | limbs_[i];
      limbs_[i] = std::uint32_t(cur / d);
      rem = cur % d;
    }
    negative_ = negative_ != o.negative_;
    normalize();
    return *this;
  }
  friend cpp_int operator/(cpp_int a, const cpp_int &b) { return a /= b; }
  friend cpp_int operator+(cpp_int a, const cpp_int &b) { return a += b; }
  friend cpp_int operator-(cpp_int a, const cpp_int &b) { return a -= b; }
  friend cpp_int operator*(cpp_int a, const cpp_int &b) { return a *= b; }
  friend cpp_int operator<<(cpp_int a, unsigned s) { return a <<= s; }
  friend cpp_int operator>>(cpp_int a, unsigned s) { return a >>= s; }
  friend bool operator<(const cpp_int &a, const cpp_int &b) { return compare(a, b) < 0; }
  friend bool operator>(const cpp_int &a, const cpp_int &b) { return compare(a, b) > 0; }
  friend bool operator<=(const cpp_int &a, const cpp_int &b) { return compare(a, b) <= 0; }
  friend bool operator>=(const cpp_int &a, const cpp_int &b) { return compare(a, b) >= 0; }
  friend bool operator==(const cpp_int &a, const cpp_int &b) { return compare(a, b) == 0; }
  friend bool operator!=(const cpp_int &a, const cpp_int &b) { return compare(a, b) != 0; }

 private:
  bool negative_ = false;
  std::vector<std::uint32_t> limbs_;  // little-endian magnitude, no leading zero limbs

  void normalize() {
    while (!limbs_.empty() && limbs_.back() == 0) limbs_.pop_back();
    if (limbs_.empty()) negative_ = false;
  }
  static int compare_mag(const std::vector<std::uint32_t> &a, const std::vector<std::uint32_t> &b) {
    if (a.size() != b.size()) return a.size() < b.size() ? -1 : 1;
    for (std::size_t i = a.size(); i-- > 0;)
      if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
    return 0;
  }
  static int compare(const cpp_int &a, const cpp_int &b) {
    if (a.negative_ != b.negative_) return a.negative_ ? -1 : 1;
    int c = compare_mag(a.limbs_, b.limbs_);
    return a.negative_ ? -c : c;
  }
  static std::vector<std::uint32_t> add(const std::vector<std::uint32_t> &a,
                                        const std::vector<std::uint32_t> &b) {
    std::size_t n = a.size() > b.size() ? a.size() : b.size();
    std::vector<std::uint32_t> r(n + 1, 0);
    std::uint64_t carry = 0;
    for (std::size_t i = 0; i < n; ++i) {
      std::uint64_t s = carry + (i < a.size() ? a[i] : 0u) + (i < b.size() ? b[i] : 0u);
      r[i] = std::uint32_t(s);
      carry = s >> 32;
    }
    r[n] = std::uint32_t(carry);
    return r;
  }
  static std::vector<std::uint32_t> sub(const std::vector<std::uint32_t> &a,
                                        const std::vector<std::uint32_t> &b) {  // |a| >= |b|
    std::vector<std::uint32_t> r(a.size(), 0);
    std::int64_t borrow = 0;
    for (std::size_t i = 0; i < a.size(); ++i) {
      std::int64_t d = std::int64_t(a[i]) - (i < b.size() ? std::int64_t(b[i]) : 0) - borrow;
      borrow = d < 0 ? 1 : 0;
      r[i] = std::uint32_t(d + (borrow << 32));
    }
    return r;
  }
};

inline unsigned msb(const cpp_int &x) {
  const auto &l = x.limbs();
  std::size_t top = l.size() - 1;
  return unsigned(32 * top + (31 - __builtin_clz(l[top])));
}

}  // namespace multiprecision
}  // namespace boost
