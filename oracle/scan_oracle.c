/* CPU restatement of the reference candidate scan -- TEST INFRASTRUCTURE ONLY.
 *
 * Restates /root/reference/pkg/src/fracodec/_scan.py:14-63 (scan_candidates):
 * for every range m (OpenMP over ranges, as numba prange at _scan.py:29),
 * walk candidates c = (e*8 + iso)*S + si in order, offset o = rint(rmean)
 * (proposed, _scan.py:33) or clip(rint(rmean - s*dmean), 0, 255) (baseline,
 * _scan.py:38-43), exact int64 SSD of clip(q + o, 0, 255) against the range
 * with the result-neutral early exit (_scan.py:48-57), and keep the first
 * strict minimum (_scan.py:58-60).  rint() under the default rounding mode
 * is IEEE round-half-to-even like numba's round() on floats.  Compiled with
 * -ffp-contract=off so s*dmean is rounded before the subtraction.
 */
#include <math.h>
#include <stdint.h>
#ifdef _OPENMP
#include <omp.h>
#endif

void oracle_scan_candidates(int64_t M, int32_t n, const int16_t* ranges, const double* rmeans,
                            const int16_t* q, int64_t E, const double* dmeans, int32_t S,
                            const double* svals, int32_t baseline, int64_t* out_err,
                            int64_t* out_idx, int32_t threads) {
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#endif
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t m = 0; m < M; ++m) {
        const int16_t* r = ranges + m * (int64_t)n;
        int64_t best = (int64_t)1 << 62;
        int64_t bestc = -1;
        const int o_prop = (int)rint(rmeans[m]);
        int64_t c = 0;
        for (int64_t e = 0; e < E; ++e) {
            for (int iso = 0; iso < 8; ++iso) {
                for (int si = 0; si < S; ++si, ++c) {
                    int o;
                    if (baseline) {
                        volatile double prod = svals[si] * dmeans[e];
                        o = (int)rint(rmeans[m] - prod);
                        if (o < 0) o = 0;
                        else if (o > 255) o = 255;
                    } else {
                        o = o_prop;
                    }
                    const int16_t* row = q + c * (int64_t)n;
                    int64_t err = 0;
                    for (int k = 0; k < n; ++k) {
                        int v = row[k] + o;
                        v = v < 0 ? 0 : (v > 255 ? 255 : v);
                        int d = v - r[k];
                        err += (int64_t)d * d;
                        if (err > best) break;
                    }
                    if (err < best) {
                        best = err;
                        bestc = c;
                    }
                }
            }
        }
        out_err[m] = best;
        out_idx[m] = bestc;
    }
}
