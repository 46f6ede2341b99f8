"""The boundary is a plain C ABI: a C program compiled against include/hsolve.h
and linked to libhsolve.so (no Python, no torch) analyzes a 2-D Poisson matrix, reads the
analysis back through the length-query convention, and gets the documented errors for bad
arguments -- host integer code, so it runs without a GPU; on a machine without a device the
factor call must fail with HS_E_NO_DEVICE (there is no CPU fallback)."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1811_11248_b200")

PROG = r"""
#include <stdio.h>
#include <stdlib.h>
#include "hsolve.h"

int main(void) {
  /* 2-D Poisson, 5-point, 8 x 8 grid: CSR with both triangles */
  const int nx = 8, n = nx * nx;
  int64_t rowptr[65];
  int32_t colind[5 * 64];
  double coords[2 * 64];
  int64_t k = 0;
  for (int j = 0; j < nx; ++j)
    for (int i = 0; i < nx; ++i) {
      const int r = i + nx * j;
      rowptr[r] = k;
      if (j > 0) colind[k++] = r - nx;
      if (i > 0) colind[k++] = r - 1;
      colind[k++] = r;
      if (i < nx - 1) colind[k++] = r + 1;
      if (j < nx - 1) colind[k++] = r + nx;
      coords[2 * r] = i;
      coords[2 * r + 1] = j;
    }
  rowptr[n] = k;
  hs_analyze_opts opt = {4, 0, 1, 1, 0};
  hs_analysis a = NULL;
  hs_status st = hs_analyze(NULL, n, rowptr, colind, coords, 2, NULL, &opt, &a);
  if (st != HS_OK) { printf("analyze failed: %s %s\n", hs_status_string(st), hs_last_error(NULL)); return 1; }
  hs_analysis_info info;
  if (hs_analysis_get_info(a, &info) != HS_OK) return 2;
  int64_t len = 0;
  if (hs_analysis_export(a, HS_EXP_PERM, 0, NULL, 0, &len) != HS_OK || len != n) return 3;
  int64_t* perm = (int64_t*)malloc(sizeof(int64_t) * len);
  if (hs_analysis_export(a, HS_EXP_PERM, 0, perm, len, &len) != HS_OK) return 4;
  int seen[64] = {0};
  for (int i = 0; i < n; ++i) seen[perm[i]]++;
  for (int i = 0; i < n; ++i) if (seen[i] != 1) return 5;
  /* errors: a bad option, a NULL output */
  hs_analyze_opts bad = {0, 0, 1, 1, 0};
  hs_analysis b = NULL;
  if (hs_analyze(NULL, n, rowptr, colind, coords, 2, NULL, &bad, &b) != HS_E_INVALID_ARG) return 6;
  if (hs_analyze(NULL, n, rowptr, colind, coords, 2, NULL, &opt, NULL) != HS_E_INVALID_ARG) return 7;
  hs_handle h = NULL;
  st = hs_create(&h, 0, 1, 0, NULL);
  printf("n=%lld depth=%d L_top=%d create=%s\n", (long long)info.n, info.depth, info.L_top, hs_status_string(st));
  if (h) hs_destroy(h);
  hs_analysis_destroy(a);
  free(perm);
  return 0;
}
"""


@pytest.mark.skipif(shutil.which("gcc") is None, reason="gcc not available")
def test_c_program_uses_the_abi(tmp_path):
    lib = os.path.join(LIBDIR, "libhsolve.so")
    if not os.path.exists(lib):
        from paper_1811_11248_b200 import build
        build.build()
    src = tmp_path / "abi.c"
    src.write_text(PROG)
    exe = tmp_path / "abi"
    r = subprocess.run(["gcc", "-std=c99", "-O1", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe),
                        "-L", LIBDIR, "-lhsolve", f"-Wl,-rpath,{LIBDIR}"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    import torch   # its bundled libcudart is the one libhsolve.so links against here
    cudart = os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib")
    env = dict(os.environ, LD_LIBRARY_PATH=os.path.abspath(cudart) + ":" + os.environ.get("LD_LIBRARY_PATH", ""))
    r = subprocess.run([str(exe)], capture_output=True, text=True, env=env, timeout=120)
    assert r.returncode == 0, (r.returncode, r.stdout, r.stderr)
    assert "n=64 depth=4 L_top=3" in r.stdout
    import torch.cuda
    if not torch.cuda.is_available():
        assert "create=HS_E_NO_DEVICE" in r.stdout
