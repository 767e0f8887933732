// dropin_check.cpp -- the shim's id_auto dual and idkit::sketch_rid seen from
// the reference's side: linked like acceptance_b200 (reference sources except
// id.cpp / qr.cpp, plus integration/idkit_b200_shim.cpp), it checks with the
// reference's own Matrix helpers that
//   * id_auto on a tall matrix returns transposed = true and
//     approx == transpose(matmul(select_columns(transpose(a), cols), z)) bit for bit
//     (id.cpp:85-92; test_id.cpp:57-68's exact equality, dual form),
//   * id_auto on a wide matrix returns approx == matmul(select_columns(a, cols), z),
//   * idkit::sketch_rid (integration/idkit_b200_ext.hpp) obeys the same contract,
//     picks k distinct columns and reproduces them exactly (Z[:, cols] = I).
// Prints one line per case and exits non-zero on the first failure.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <set>

#include "idkit/datasets.hpp"
#include "idkit/id.hpp"
#include "idkit/matrix.hpp"
#include "idkit_b200_ext.hpp"

using namespace idkit;

static int fail(const char* what) {
    std::printf("FAIL %s\n", what);
    return 1;
}

// exact_identity: Z[:, cols] = I exactly for the interpolative forms (optim_id,
// sketch_rid); optim_rid's normal-equation Z (id.cpp:68-72) meets it to rounding.
static int check(const Matrix& a, const IdResult& r, std::size_t k, bool want_t, const char* name,
                 bool exact_identity = true) {
    if (r.transposed != want_t) return fail(name);
    const Matrix m = want_t ? transpose(a) : a;
    if (r.cols.size() != k || r.z.rows() != k || r.z.cols() != m.cols()) return fail(name);
    std::set<std::size_t> uniq(r.cols.begin(), r.cols.end());
    if (uniq.size() != k) return fail(name);
    const Matrix prod = matmul(select_columns(m, r.cols), r.z);
    const Matrix approx = want_t ? transpose(prod) : prod;
    if (!(frobenius_distance(approx, r.approx) == 0.0)) return fail(name);
    for (std::size_t j = 0; j < k; ++j)
        for (std::size_t i = 0; i < k; ++i)
            if (exact_identity ? r.z(i, r.cols[j]) != (i == j ? 1.0 : 0.0)
                               : std::fabs(r.z(i, r.cols[j]) - (i == j ? 1.0 : 0.0)) > 1e-8)
                return fail(name);
    const double err = frobenius_distance(a, r.approx) / frobenius_norm(a);
    std::printf("PASS %-28s transposed=%d rel_error=%.6g\n", name, r.transposed ? 1 : 0, err);
    return 0;
}

int main() {
    const Matrix tall = generate(GeneratorKind::uniform, 300, 70, 11);
    const Matrix wide = generate(GeneratorKind::gaussian, 60, 240, 12);
    int bad = 0;
    bad |= check(tall, id_auto(tall, 9, IdMethod::deterministic, 0, 0.2), 9, true, "id_auto det (dual)");
    bad |= check(tall, id_auto(tall, 9, IdMethod::randomized, 5, 0.5), 9, true, "id_auto randomized (dual)", false);
    bad |= check(wide, id_auto(wide, 12, IdMethod::deterministic, 0, 0.2), 12, false, "id_auto det");
    bad |= check(wide, id_auto(wide, 12, IdMethod::randomized, 5, 0.5), 12, false, "id_auto randomized", false);
    bad |= check(wide, sketch_rid(wide, 12, 6, 99), 12, false, "sketch_rid");
    bad |= check(tall, sketch_rid(tall, 9, 4, 99), 9, true, "sketch_rid (dual)");
    return bad;
}
