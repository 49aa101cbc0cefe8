// Golden-vector helper, compiled ONLY in the build container by make_golden.py
// against the reference headers and oracle/_ref/libssjoin_ref.so: exposes the
// reference's own ssj::build_bitmaps (proj/src/bitmap.cpp:145-158) over a CSR
// collection so its sketch stores can be fingerprinted into tests/golden/.
#include <cstdint>
#include <cstring>
#include <vector>

#include "bitmap.hpp"

extern "C" void ref_build_bitmaps(const uint32_t* tokens, const uint64_t* offsets, size_t n,
                                  int method, int width, int hash, uint64_t* out) {
    std::vector<ssj::RecordSet> recs(n);
    for (size_t r = 0; r < n; ++r) {
        recs[r].id = static_cast<uint32_t>(r);
        recs[r].tokens.assign(tokens + offsets[r], tokens + offsets[r + 1]);
    }
    ssj::BitmapConfig cfg;
    cfg.width = width;
    cfg.hash = hash == 1 ? ssj::HashKind::Multiplicative : ssj::HashKind::Modulo;
    auto store = ssj::build_bitmaps(recs, cfg, static_cast<ssj::BitmapMethod>(method));
    std::memcpy(out, store.data.data(), store.data.size() * sizeof(uint64_t));
}
