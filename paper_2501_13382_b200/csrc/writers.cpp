// writers.cpp -- field output of the GBS stage (host code, part of libbf_gbs.so).
//
// bf_write_field_csv replaces beamfield.harness.write_field_csv (harness.py:197-208):
// header "x,y,z,freq_hz,re_p,im_p,spl_db", rows observer-major / frequency-minor,
// every number formatted like Python's format(x, ".17g") (harness.py:39-40), which is
// C's "%.17g" (both correctly rounded; inf/-inf/nan spelled alike).  The reference
// loops over rows in Python; here row blocks are formatted on all host threads into
// buffers that are written in order, so the file is byte-identical.
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <thread>
#include <vector>

#include "../../include/bf_gbs.h"

namespace bf {
int fail(int status, const char *fmt, ...);
}

namespace {

inline void put_g(std::string &out, double v) {
    char buf[40];
    const int n = snprintf(buf, sizeof(buf), "%.17g", v);
    out.append(buf, (size_t)n);
}

void format_rows(const double *pts, int64_t lo, int64_t hi, const double *freqs, int64_t nf,
                 const double *pressure, const double *spl, std::string &out) {
    out.reserve((size_t)((hi - lo) * nf * 120));
    for (int64_t oi = lo; oi < hi; ++oi)
        for (int64_t fi = 0; fi < nf; ++fi) {
            const int64_t k = oi * nf + fi;
            put_g(out, pts[3 * oi]);
            out.push_back(',');
            put_g(out, pts[3 * oi + 1]);
            out.push_back(',');
            put_g(out, pts[3 * oi + 2]);
            out.push_back(',');
            put_g(out, freqs[fi]);
            out.push_back(',');
            put_g(out, pressure[2 * k]);
            out.push_back(',');
            put_g(out, pressure[2 * k + 1]);
            out.push_back(',');
            put_g(out, spl[k]);
            out.push_back('\n');
        }
}

}  // namespace

extern "C" int bf_write_field_csv(const char *path, const double *points, int64_t n_obs,
                                  const double *freqs, int64_t nf, const double *pressure,
                                  const double *spl, int threads) {
    if (!path || n_obs < 0 || nf < 0 || (n_obs > 0 && nf > 0 && (!points || !freqs || !pressure || !spl)))
        return bf::fail(BF_EINVAL, "bf_write_field_csv: bad arguments");
    FILE *fh = fopen(path, "wb");
    if (!fh) return bf::fail(BF_EIO, "bf_write_field_csv: cannot open %s", path);
    static const char header[] = "x,y,z,freq_hz,re_p,im_p,spl_db\n";
    bool ok = fwrite(header, 1, sizeof(header) - 1, fh) == sizeof(header) - 1;
    if (threads <= 0) threads = (int)std::max(1u, std::thread::hardware_concurrency());
    // blocks of rows, formatted in parallel a window at a time, written in order
    const int64_t block = 16384;
    const int64_t n_blocks = (n_obs + block - 1) / block;
    std::vector<std::string> bufs((size_t)threads);
    for (int64_t b0 = 0; ok && b0 < n_blocks; b0 += threads) {
        const int64_t nb = std::min<int64_t>(threads, n_blocks - b0);
        std::vector<std::thread> pool;
        for (int64_t i = 0; i < nb; ++i) {
            bufs[(size_t)i].clear();
            const int64_t lo = (b0 + i) * block, hi = std::min(n_obs, lo + block);
            pool.emplace_back(format_rows, points, lo, hi, freqs, nf, pressure, spl,
                              std::ref(bufs[(size_t)i]));
        }
        for (auto &t : pool) t.join();
        for (int64_t i = 0; ok && i < nb; ++i)
            ok = fwrite(bufs[(size_t)i].data(), 1, bufs[(size_t)i].size(), fh) ==
                 bufs[(size_t)i].size();
    }
    ok = (fclose(fh) == 0) && ok;
    return ok ? BF_OK : bf::fail(BF_EIO, "bf_write_field_csv: write to %s failed", path);
}
