/* A plain-C consumer of the whole measurement boundary (include/b2o.h): no
 * Python bindings.  It loads a program from its IR document and app spec
 * (b2o_app_load, SURVEY.md §8(b) app_load(model_json, app_spec_json)),
 * submits every pattern of a request file through b2o_submit / b2o_wait, and
 * checks each result: valid, directive executions == the plan's
 * multiplicities, and the final state of every output bit-identical to the
 * expected bytes (the reference's own C emission run on the CPU, written by
 * tests/test_abi.py).  Also: a malformed document is refused with a reason.
 *
 * Request directory layout (written by tests/test_abi.py):
 *   doc.json, spec.json        the program and its app spec
 *   patterns.txt               "pattern <genome> <n_roots> <roots...> <n_dirs>"
 *                              followed by n_dirs lines
 *                              "<var> <dir> <anchor> <side> <multiplicity> <batch>"
 *   expect.txt                 "<name> <bytes> <file>" per output
 *
 * Build: make -C tests/c   Run: tests/c/abi_app <dir>   (exit status 0 = pass) */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "b2o.h"

static char *slurp(const char *dir, const char *name, long *len) {
  char path[4096];
  if (dir[0]) snprintf(path, sizeof path, "%s/%s", dir, name);
  else snprintf(path, sizeof path, "%s", name);
  FILE *f = fopen(path, "rb");
  if (!f) return NULL;
  fseek(f, 0, SEEK_END);
  long n = ftell(f);
  fseek(f, 0, SEEK_SET);
  char *buf = (char *)malloc((size_t)n + 1);
  if (fread(buf, 1, (size_t)n, f) != (size_t)n) n = 0;
  buf[n] = 0;
  fclose(f);
  if (len) *len = n;
  return buf;
}

typedef struct {
  char genome[64];
  uint8_t *roots;
  int n_dirs;
  b2o_directive *dirs;
  uint64_t planned;
} Pat;

int main(int argc, char **argv) {
  if (argc != 2) {
    fprintf(stderr, "usage: abi_app <request dir>\n");
    return 2;
  }
  const char *dir = argv[1];
  if (b2o_init(NULL, 0) != 0) {
    fprintf(stderr, "b2o_init: %s\n", b2o_last_error());
    return 1;
  }
  char *doc = slurp(dir, "doc.json", NULL), *spec = slurp(dir, "spec.json", NULL);
  if (!doc || !spec) return 2;
  uint64_t app = 0;
  /* a malformed document is refused with a reason, never a crash */
  if (b2o_app_load("{\"not\": \"a program\"}", spec, &app) == 0 || strlen(b2o_last_error()) == 0) {
    fprintf(stderr, "malformed document accepted\n");
    return 1;
  }
  printf("malformed document refused: %.60s\n", b2o_last_error());
  if (b2o_app_load(doc, spec, &app) != 0) {
    fprintf(stderr, "b2o_app_load: %s\n", b2o_last_error());
    return 1;
  }
  const int n_loops = b2o_app_num_loops(app);
  /* patterns */
  char path[4096];
  snprintf(path, sizeof path, "%s/patterns.txt", dir);
  FILE *pf = fopen(path, "r");
  if (!pf) return 2;
  Pat *pats = (Pat *)calloc(4096, sizeof(Pat));
  int np = 0;
  char tag[32];
  while (fscanf(pf, "%31s", tag) == 1) {
    Pat *p = &pats[np++];
    int nr = 0;
    if (fscanf(pf, "%63s %d", p->genome, &nr) != 2) return 2;
    p->roots = (uint8_t *)calloc((size_t)n_loops + 1, 1);
    for (int i = 0; i < nr; ++i) {
      int r;
      if (fscanf(pf, "%d", &r) != 1 || r < 0 || r >= n_loops) return 2;
      p->roots[r] = 1;
    }
    if (fscanf(pf, "%d", &p->n_dirs) != 1) return 2;
    p->dirs = (b2o_directive *)calloc((size_t)p->n_dirs + 1, sizeof(b2o_directive));
    for (int i = 0; i < p->n_dirs; ++i) {
      b2o_directive *d = &p->dirs[i];
      unsigned long long m;
      if (fscanf(pf, "%d %d %d %d %llu %d", &d->var_id, &d->dir, &d->anchor_loop, &d->side, &m, &d->batch_id) != 6)
        return 2;
      d->multiplicity = m;
      p->planned += m;
    }
  }
  fclose(pf);
  /* every pattern in one batch (the worker pool orders them LPT) */
  b2o_pattern *arr = (b2o_pattern *)calloc((size_t)np, sizeof(b2o_pattern));
  for (int i = 0; i < np; ++i) {
    arr[i].gpu_root = pats[i].roots;
    arr[i].n_loops = n_loops;
    arr[i].n_directives = pats[i].n_dirs;
    arr[i].directives = pats[i].dirs;
    arr[i].device = -1;
    arr[i].mode = B2O_MODE_COHERENT;
    arr[i].repeats = 1;
    arr[i].timeout_s = 60.0;
  }
  b2o_result *res = (b2o_result *)calloc((size_t)np, sizeof(b2o_result));
  uint64_t batch = 0;
  if (b2o_submit(app, arr, np, &batch) != 0 || b2o_wait(batch, res, np, 600.0) != 0) {
    fprintf(stderr, "submit/wait: %s\n", b2o_last_error());
    return 1;
  }
  int bad = 0;
  for (int i = 0; i < np; ++i) {
    if (res[i].validity != B2O_VALID || res[i].directive_execs != pats[i].planned || res[i].time_s <= 0) {
      fprintf(stderr, "pattern %s: validity %d execs %llu planned %llu (%s)\n", pats[i].genome, res[i].validity,
              (unsigned long long)res[i].directive_execs, (unsigned long long)pats[i].planned, res[i].diag);
      ++bad;
    }
  }
  printf("batch of %d patterns: %d invalid\n", np, bad);
  /* final state, one pattern at a time, against the expected bytes */
  snprintf(path, sizeof path, "%s/expect.txt", dir);
  FILE *ef = fopen(path, "r");
  char names[16][64], files[16][4096];
  unsigned long long sizes[16];
  int ne = 0;
  while (ne < 16 && fscanf(ef, "%63s %llu %4095s", names[ne], &sizes[ne], files[ne]) == 3) ++ne;
  fclose(ef);
  int exact = 0;
  for (int i = 0; i < np; ++i) {
    b2o_result r;
    if (b2o_submit(app, &arr[i], 1, &batch) != 0 || b2o_wait(batch, &r, 1, 600.0) != 0) return 1;
    int ok = r.validity == B2O_VALID;
    for (int e = 0; e < ne && ok; ++e) {
      int vid = b2o_app_var_id(app, names[e]);
      char *want = slurp("", files[e], NULL);
      char *got = (char *)malloc(sizes[e]);
      ok = vid >= 0 && want && b2o_app_read(app, r.worker, vid, got, sizes[e]) == 0 &&
           memcmp(got, want, sizes[e]) == 0;
      free(want);
      free(got);
    }
    if (ok) ++exact;
    else fprintf(stderr, "pattern %s: final state differs\n", pats[i].genome);
  }
  printf("final state bit-exact for %d of %d patterns\n", exact, np);
  b2o_app_destroy(app);
  b2o_shutdown();
  if (bad == 0 && exact == np) {
    printf("PASS\n");
    return 0;
  }
  printf("FAIL\n");
  return 1;
}
