/* A plain-C host of libmgp.so (include/megopolis_b200.h): no Python, no torch.
 *
 *   gcc -O2 -I include examples/resample_host.c -L paper_2109_13504_b200 -lmgp \
 *       -Wl,-rpath,$PWD/paper_2109_13504_b200 -o /tmp/resample_host
 *   /tmp/resample_host weights.bin 7 > ancestors.bin
 *
 * Reads float32 weights (raw little-endian, or the reference's `<Q` count header + payload
 * when the file size says so: M/storage.py:29-91), runs Megopolis through the host-buffer
 * entry (B from the epsilon = 0.01 rule, the reference's stream) and writes the int64 ancestors
 * to stdout.  Errors print mgp_last_error() and exit 2 (ValueError) or 1 (CUDA). */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "megopolis_b200.h"

int main(int argc, char **argv) {
  if (argc < 3) {
    fprintf(stderr, "usage: %s weights.bin seed [kind=3] [rng=0]\n", argv[0]);
    return 2;
  }
  FILE *f = fopen(argv[1], "rb");
  if (!f) {
    perror(argv[1]);
    return 2;
  }
  fseek(f, 0, SEEK_END);
  long bytes = ftell(f);
  fseek(f, 0, SEEK_SET);
  uint64_t count = 0;
  long skip = 0;
  if (bytes >= 8 && fread(&count, 8, 1, f) == 1 && (long)(8 + 4 * count) == bytes) skip = 8;
  fseek(f, skip, SEEK_SET);
  const int64_t n = (bytes - skip) / 4;
  float *w = (float *)malloc(sizeof(float) * (size_t)(n > 0 ? n : 1));
  int64_t *anc = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  if (!w || !anc || fread(w, 4, (size_t)n, f) != (size_t)n) {
    fprintf(stderr, "cannot read %lld weights\n", (long long)n);
    return 2;
  }
  fclose(f);
  const uint64_t seed = strtoull(argv[2], NULL, 10);
  const int kind = argc > 3 ? atoi(argv[3]) : MGP_KIND_MEGOPOLIS;
  const int rng = argc > 4 ? atoi(argv[4]) : MGP_RNG_MEGORES;
  int32_t b = 0;
  const int rc = mgp_resample_host(kind, w, MGP_F32, n, 0, 0.01, seed, 32, 0, 1, rng, anc, &b, -1);
  if (rc) {
    fprintf(stderr, "megores: error: %s\n", mgp_last_error());
    return rc < 0 ? 2 : 1;
  }
  fwrite(anc, sizeof(int64_t), (size_t)n, stdout);
  fprintf(stderr, "resampled N=%lld with B=%d\n", (long long)n, b);
  free(w);
  free(anc);
  return 0;
}
