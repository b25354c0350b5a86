/* capi_example.c -- a plain C caller of libodyssey_b200.so through the reference-facing
 * ABI (include/odyssey_b200.h), the way the reference's own C++ callers use odyssey.h.
 * It replays the reference's test_capi.cpp:121-165 (FAST GEMM through the C API vs
 * matmul_f32 of the dequantized operands, <= 1e-4 relative; counter formulas) and runs
 * every comparison engine (odyssey.h:36-42) plus the error conventions (odyssey.h:1-10).
 *
 *   gcc -O2 -std=c11 -Iinclude tests/c_caller/capi_example.c \
 *       -Lpaper_2311_09550_b200 -lodyssey_b200 -Wl,-rpath,$PWD/paper_2311_09550_b200 -lm
 *   ./capi_example [--link-only]
 *
 * Exit 0 = all checks passed.  --link-only exercises only the GPU-free calls (tensor
 * handles, NULL-argument errors), for machines without a B200. */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "odyssey_b200.h"

static int failures = 0;
#define CHECK(cond)                                                                  \
    do {                                                                             \
        if (!(cond)) {                                                               \
            fprintf(stderr, "CHECK failed at %s:%d: %s (%s)\n", __FILE__, __LINE__, #cond, \
                    ody_last_error() ? ody_last_error() : "");                       \
            ++failures;                                                              \
        }                                                                            \
    } while (0)

static ody_tensor* make_tensor(size_t rows, size_t cols, const float* v) {
    ody_tensor* t = NULL;
    CHECK(ody_tensor_create(rows, cols, v, &t) == ODY_OK);
    return t;
}

int main(int argc, char** argv) {
    const int link_only = argc > 1 && strcmp(argv[1], "--link-only") == 0;
    /* error conventions: NULL arguments -> EINVAL with a thread-local message */
    CHECK(ody_tensor_create(1, 1, NULL, NULL) == ODY_EINVAL);
    CHECK(ody_last_error() != NULL && strlen(ody_last_error()) > 0);
    const float bad[2] = {1.0f, NAN};
    ody_tensor* t = NULL;
    CHECK(ody_tensor_create(1, 2, bad, &t) == ODY_EINVAL); /* DenseTensor rejects NaN (tensor.cpp:21-27) */
    const float good[6] = {1, 2, 3, 4, 5, 6};
    t = make_tensor(2, 3, good);
    size_t r = 0, c = 0;
    const float* d = NULL;
    CHECK(ody_tensor_dims(t, &r, &c) == ODY_OK && r == 2 && c == 3);
    CHECK(ody_tensor_data(t, &d) == ODY_OK && d[5] == 6.0f);
    ody_tensor_free(t);
    ody_set_threads(8); /* the host pool of the ABI's host copies */
    /* extension: a column slice [:, 1:3] of the 2 x 3 matrix, no intermediate copy */
    CHECK(ody_tensor_create_strided(2, 2, 3, good + 1, &t) == ODY_OK);
    CHECK(ody_tensor_data(t, &d) == ODY_OK && d[0] == 2.0f && d[1] == 3.0f && d[2] == 5.0f && d[3] == 6.0f);
    ody_tensor_free(t);
    const float bad_outside[6] = {NAN, 2, 3, NAN, 5, 6}; /* NaN only in the skipped column */
    CHECK(ody_tensor_create_strided(2, 2, 3, bad_outside + 1, &t) == ODY_OK);
    ody_tensor_free(t);
    CHECK(ody_tensor_create_strided(2, 2, 3, bad_outside, &t) == ODY_EINVAL);
    ody_set_threads(0);
    if (link_only) {
        printf(failures ? "FAILED\n" : "capi_example (link-only): ok\n");
        return failures ? 1 : 0;
    }

    /* ref test_capi.cpp:121-165 */
    enum { M = 3, N = 4, K = 8 };
    float av[M * K], wv[N * K];
    for (size_t i = 0; i < M * K; ++i) av[i] = 0.125f * (float)((int)(i * 7 % 23) - 11);
    for (size_t i = 0; i < N * K; ++i) wv[i] = 0.03f * (float)((int)(i * 5 % 17) - 8);
    ody_tensor* a = make_tensor(M, K, av);
    ody_tensor* w = make_tensor(N, K, wv);
    ody_qtensor *a_q = NULL, *w_q = NULL;
    CHECK(ody_quantize_activations(a, &a_q) == ODY_OK);
    CHECK(ody_quantize_weights(w, 4, ODY_PER_CHANNEL, 0, NULL, NULL, &w_q) == ODY_OK);
    ody_gemm_counters cnt;
    memset(&cnt, 0, sizeof(cnt));
    ody_tensor* out = NULL;
    CHECK(ody_gemm(ODY_ENGINE_FAST, NULL, a_q, w_q, &cnt, &out) == ODY_OK);
    CHECK(cnt.int8_mac_ops == (uint64_t)M * N * K && cnt.dequant_events == (uint64_t)M * N);
    ody_tensor *a_dq = NULL, *w_dq = NULL, *ref = NULL;
    CHECK(ody_dequantize(a_q, &a_dq) == ODY_OK);
    CHECK(ody_dequantize(w_q, &w_dq) == ODY_OK);
    CHECK(ody_matmul_f32(a_dq, w_dq, &ref) == ODY_OK);
    const float *got = NULL, *want = NULL;
    CHECK(ody_tensor_data(out, &got) == ODY_OK && ody_tensor_data(ref, &want) == ODY_OK);
    for (size_t i = 0; got && want && i < M * N; ++i)
        CHECK(fabsf(got[i] - want[i]) <= 1e-4f * fmaxf(1.0f, fabsf(want[i])));

    /* every engine through the same ABI; FAST == ASYMMETRIC bit for bit (test_gemm.cpp:129-149) */
    ody_qtensor *w8 = NULL, *wg = NULL;
    CHECK(ody_quantize_weights(w, 8, ODY_PER_CHANNEL, 128, NULL, NULL, &w8) == ODY_OK);
    CHECK(ody_quantize_weights(w, 4, ODY_PER_GROUP, 4, NULL, NULL, &wg) == ODY_OK);
    ody_tensor *o_asym = NULL, *o_fine = NULL, *o_w8 = NULL, *o_w4a16 = NULL;
    CHECK(ody_gemm(ODY_ENGINE_ASYMMETRIC, NULL, a_q, w_q, &cnt, &o_asym) == ODY_OK);
    CHECK(cnt.zero_point_sub_ops == (uint64_t)N * K);
    CHECK(ody_gemm(ODY_ENGINE_FINEGRAINED, NULL, a_q, wg, &cnt, &o_fine) == ODY_OK);
    CHECK(cnt.dequant_events == (uint64_t)M * N * (K / 4));
    CHECK(ody_gemm(ODY_ENGINE_W8A8, NULL, a_q, w8, &cnt, &o_w8) == ODY_OK);
    CHECK(ody_gemm(ODY_ENGINE_W4A16, a, NULL, wg, &cnt, &o_w4a16) == ODY_OK);
    CHECK(cnt.dequant_events == (uint64_t)M * N * K);
    const float* ga = NULL;
    CHECK(ody_tensor_data(o_asym, &ga) == ODY_OK);
    for (size_t i = 0; ga && got && i < M * N; ++i) CHECK(memcmp(&ga[i], &got[i], 4) == 0);
    /* reference validation: W8A8 needs 8-bit weights, the engine enum is range-checked */
    ody_tensor* o_bad = NULL;
    CHECK(ody_gemm(ODY_ENGINE_W8A8, NULL, a_q, w_q, NULL, &o_bad) == ODY_EINVAL);
    CHECK(ody_gemm((ody_engine)9, NULL, a_q, w_q, NULL, &o_bad) == ODY_EINVAL);

    ody_tensor_free(o_asym);
    ody_tensor_free(o_fine);
    ody_tensor_free(o_w8);
    ody_tensor_free(o_w4a16);
    ody_qtensor_free(w8);
    ody_qtensor_free(wg);
    ody_tensor_free(ref);
    ody_tensor_free(a_dq);
    ody_tensor_free(w_dq);
    ody_tensor_free(out);
    ody_qtensor_free(a_q);
    ody_qtensor_free(w_q);
    ody_tensor_free(a);
    ody_tensor_free(w);
    printf(failures ? "FAILED (%d)\n" : "capi_example: ok\n", failures);
    return failures ? 1 : 0;
}
