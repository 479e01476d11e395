/* CPU ORACLE (test infrastructure only) — plain-C restatement of the
 * reference's bit-exact cut diagonal, lrqbench problem.py:139-149:
 *
 *   acc = 0; for each edge (i<j) in lexicographic order: acc += w * bit
 *
 * with bit = ((z >> i) ^ (z >> j)) & 1.  w * bit is exact (bit in {0,1}), so
 * the only roundings are the sequential additions, in edge order.  Compiled
 * with -ffp-contract=off -fno-fast-math so nothing is re-associated.
 * Callers: tests/ (checker) only.  See oracle/__init__.py.
 */
#include <stdint.h>

void oracle_cut_values(int n, const double *w, const uint64_t *z, int64_t count,
                       double *out)
{
    for (int64_t k = 0; k < count; ++k) {
        uint64_t x = z[k];
        double acc = 0.0;
        int e = 0;
        for (int i = 0; i < n; ++i)
            for (int j = i + 1; j < n; ++j, ++e) {
                uint64_t bit = ((x >> i) ^ (x >> j)) & 1u;
                acc = acc + w[e] * (double)bit;
            }
        out[k] = acc;
    }
}
