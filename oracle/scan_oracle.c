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

/* The same scan over the BASE operand qbase[e*S + si][k] = rint(s*(d - dmean))
 * (or rint(s*d) in baseline mode) with the isometry applied on the fly:
 * q[(e*8 + iso)*S + si][k] = qbase[e*S + si][isomap[iso*n + k]], which is
 * exactly how build_candidate_set fills the reference's operand
 * (matcher.py:143-159: apply_isometry of the rounded base tile).  Same
 * candidate order, offsets and first strict minimum as above; the operand is
 * 8x smaller, so full-size pools (c5: 4.13M domains) fit in host memory.
 *
 * The SSD of candidate (e, iso, si) is summed over base pixels j against the
 * range permuted by the inverse map, r[inv(j)]: the same exact integer, in a
 * different order.  The early exit (_scan.py:48-57) is tested every 16
 * pixels; it only ever drops candidates whose partial sum already exceeds
 * the best, so it is result-neutral wherever it is tested.  Test
 * infrastructure only. */
void oracle_scan_candidates_base(int64_t M, int32_t n, const int16_t* ranges, const double* rmeans,
                                 const int16_t* qbase, int64_t E, const double* dmeans, int32_t S,
                                 const double* svals, int32_t baseline, const int32_t* isomap,
                                 int64_t* out_err, int64_t* out_idx, int32_t threads) {
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#endif
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t m = 0; m < M; ++m) {
        const int16_t* r = ranges + m * (int64_t)n;
        int32_t rp[8][1024];
        for (int iso = 0; iso < 8; ++iso)
            for (int k = 0; k < n; ++k) rp[iso][isomap[iso * n + k]] = r[k];
        int64_t best = (int64_t)1 << 62;
        int64_t bestc = -1;
        const int o_prop = (int)rint(rmeans[m]);
        int64_t c = 0;
        for (int64_t e = 0; e < E; ++e) {
            for (int iso = 0; iso < 8; ++iso) {
                const int32_t* rr = rp[iso];
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
                    const int16_t* base = qbase + (e * S + si) * (int64_t)n;
                    int64_t err = 0;
                    for (int k0 = 0; k0 < n; k0 += 16) {
                        const int kn = n - k0 < 16 ? n - k0 : 16;
                        int32_t part = 0;
                        for (int k = 0; k < kn; ++k) {
                            int v = base[k0 + k] + o;
                            v = v < 0 ? 0 : (v > 255 ? 255 : v);
                            const int d = v - rr[k0 + k];
                            part += d * d;
                        }
                        err += part;
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
