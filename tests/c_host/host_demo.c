/* A plain-C host of the C ABI (include/dz_b200.h): no Python, no torch. Exercises the host-side
 * entry points a C/C++ serving process calls before touching the GPU: the plan (group_by_delta,
 * inference.py:106-123), the unknown-slot error (inference.py:135-137), the mixed plan, and the
 * DZDL container walk + zlib inflate (formats.py:102-169) on a file the reference wrote.
 * Usage: host_demo <dzdl file>. Prints one line per check; exit code 0 = all good. */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "dz_b200.h"

#define CHECK(c)                                        \
  do {                                                  \
    if (!(c)) {                                         \
      fprintf(stderr, "FAILED %s:%d %s\n", __FILE__, __LINE__, #c); \
      return 1;                                         \
    }                                                   \
  } while (0)

int main(int argc, char** argv) {
  printf("%s\n", dz_version());
  /* plan: ids [2,0,2,1] -> stable order [1,3,0,2], base job + one job per slot */
  int32_t slots[4] = {2, 0, 2, 1}, kinds[3] = {DZ_KIND_SPARSE4, DZ_KIND_SPARSE4, DZ_KIND_SPARSE4};
  int32_t order[4], n_jobs = 0;
  dz_job jobs[16];
  CHECK(dz_plan(slots, 4, kinds, 3, 1, order, jobs, dz_plan_max_jobs(4), &n_jobs, 8) == DZ_OK);
  CHECK(n_jobs == 4 && order[0] == 1 && order[1] == 3 && order[2] == 0 && order[3] == 2);
  CHECK(jobs[0].slot == -1 && jobs[0].tok_count == 4 && jobs[3].slot == 2 && jobs[3].tok_count == 2);
  printf("plan ok: %d jobs\n", n_jobs);
  int32_t bad[2] = {0, 7};
  CHECK(dz_plan(bad, 2, kinds, 3, 1, order, jobs, 16, &n_jobs, 8) == DZ_E_UNKNOWN);
  printf("unknown slot -> %s\n", dz_strerror(DZ_E_UNKNOWN));
  /* mixed plan: 300 tokens on slot 0 -> two prefill jobs of equal 16-aligned size (160 + 140) */
  int32_t T = 300 + 5, *s2 = malloc(sizeof(int32_t) * T), *perm = malloc(sizeof(int32_t) * T);
  int32_t *ord2 = malloc(sizeof(int32_t) * T), n_pf = 0, t_pf = 0;
  dz_job* jobs2 = malloc(sizeof(dz_job) * dz_plan_max_jobs(T));
  for (int i = 0; i < T; i++) s2[i] = i < 300 ? 0 : 1;
  CHECK(dz_plan_mixed(s2, T, kinds, 3, 1, 192, perm, ord2, jobs2, dz_plan_max_jobs(T), &n_jobs, &n_pf, &t_pf, 8) ==
        DZ_OK);
  CHECK(t_pf == 300 && n_pf == 2 && jobs2[0].tok_count == 160 && jobs2[1].tok_count == 140);
  printf("mixed plan ok: %d prefill rows, %d jobs\n", t_pf, n_jobs);
  /* DZDL walk */
  if (argc > 1) {
    FILE* f = fopen(argv[1], "rb");
    CHECK(f != NULL);
    fseek(f, 0, SEEK_END);
    long len = ftell(f);
    fseek(f, 0, SEEK_SET);
    uint8_t* buf = malloc(len);
    CHECK(fread(buf, 1, len, f) == (size_t)len);
    fclose(f);
    dz_dzdl_info info;
    int64_t off = -1;
    CHECK(dz_dzdl_parse_header(buf, len, &info, &off) == DZ_OK);
    /* the header is JSON; "layer_count": N */
    const char* lc = strstr((const char*)buf + info.header_off, "\"layer_count\": ");
    CHECK(lc != NULL);
    int n_layers = atoi(lc + 15);
    dz_dzdl_layer layers[8];
    CHECK(n_layers > 0 && n_layers <= 8);
    CHECK(dz_dzdl_parse_layers(buf, len, info.layers_off, n_layers, layers, &off) == DZ_OK);
    for (int i = 0; i < n_layers; i++) {
      int64_t words = layers[i].payload_len / 4;
      if (info.lossless) {
        int64_t need = 0;
        CHECK(dz_inflate(buf + layers[i].payload_off, layers[i].payload_len, NULL, 0, &need) == DZ_E_ENCODING);
        uint8_t* out = malloc(need);
        CHECK(dz_inflate(buf + layers[i].payload_off, layers[i].payload_len, out, need, &need) == DZ_OK);
        words = need / 4;
        free(out);
      }
      printf("layer %d: %dx%d, %lld payload words, %lld index bytes, %lld scale bytes\n", i, layers[i].rows,
             layers[i].cols, (long long)words, (long long)layers[i].index_len, (long long)layers[i].scales_len);
    }
    CHECK(dz_dzdl_parse_layers(buf, len - 3, info.layers_off, n_layers, layers, &off) == DZ_E_FORMAT);
    printf("truncated file -> %s (offset %lld)\n", dz_strerror(DZ_E_FORMAT), (long long)off);
    free(buf);
  }
  free(s2); free(perm); free(ord2); free(jobs2);
  printf("all ok\n");
  return 0;
}
