#!/usr/bin/env python3
"""TEST INFRASTRUCTURE ONLY.

Generates oracle/_ref/newell_quad.cpp: a mechanical __float128 rewrite of the
reference's /root/reference/proj/src/newell.cpp (long double -> __float128,
libm -> libquadmath, L literals -> Q, namespace newell -> newell_quad).  The
output lives only in the git-ignored oracle/_ref/ directory; no reference
source is committed.  It is the "truth" tensor of SURVEY.md §9 E3 against
which the device tensor (near-field Newell + Gauss-Legendre far field) is
validated beyond the reference's own long-double accuracy.
"""
import re
import sys

src, dst = sys.argv[1], sys.argv[2]
text = open(src).read()
text = text.replace('#include "magfd/newell.hpp"',
                    '#include <quadmath.h>\n'
                    'namespace magfd::newell_quad { struct TensorEntry { double xx, yy, zz, xy, xz, yz; }; }')
text = text.replace("namespace magfd::newell {", "namespace magfd::newell_quad {")
text = text.replace("} // namespace magfd::newell", "} // namespace magfd::newell_quad")
text = text.replace("long double", "__float128")
for a, b in (("std::fabs", "fabsq"), ("std::sqrt", "sqrtq"), ("std::log", "logq"),
             ("std::atan2", "atan2q"), ("std::atan", "atanq")):
    text = text.replace(a + "(", b + "(")
text = re.sub(r"(\b\d+\.\d*(?:[eE][-+]?\d+)?|\b\d+)L\b", r"\1Q", text)
text += r'''
#include <atomic>
#include <thread>
#include <vector>
#include <algorithm>
extern "C" void quad_tensor_entry(int di, int dj, int dk, double dx, double dy, double dz,
                                  double out[6]) {
    const auto e = magfd::newell_quad::demagTensorEntry(di, dj, dk, dx, dy, dz);
    out[0] = e.xx; out[1] = e.yy; out[2] = e.zz; out[3] = e.xy; out[4] = e.xz; out[5] = e.yz;
}
extern "C" void quad_tensor_octant(int nx, int ny, int nz, double dx, double dy, double dz,
                                   double* out) {
    const long n = (long)nx * ny * nz;
    std::atomic<long> next{0};
    auto work = [&] {
        for (long c; (c = next.fetch_add(1)) < n;) {
            const int i = (int)(c % nx), j = (int)((c / nx) % ny), k = (int)(c / ((long)nx * ny));
            double e[6];
            quad_tensor_entry(i, j, k, dx, dy, dz, e);
            for (int q = 0; q < 6; ++q) out[q * n + c] = e[q];
        }
    };
    std::vector<std::thread> pool;
    const unsigned nt = std::max(1u, std::thread::hardware_concurrency());
    for (unsigned t = 0; t < nt; ++t) pool.emplace_back(work);
    for (auto& t : pool) t.join();
}
'''
open(dst, "w").write(text)
