"""The boundary is a C ABI: include/hz.h compiles as strict C99 (-pedantic, -Werror) and a
plain C program links against libhz.so and calls its host-only entry points (no GPU,
no Python, no torch)."""

import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2501_04266_b200")
PROGRAM = r"""
#include "hz.h"
#include <stdio.h>
#include <string.h>

int main(void) {
  const int group[3] = {2, 2, 2};
  hz_partition_t p;
  int64_t cover = 0;
  if (strncmp(hz_version(), "hz ", 3) != 0) return 1;
  for (int r = 0; r < 8; ++r) {             /* O3: the level-3 ranges tile [0, Np) */
    if (hz_partition_ex(r, 3, group, 1000003, 256, 1, 1, 2, &p) != HZ_OK) return 2;
    cover += p.len[3];
  }
  if (cover != p.padded_numel) return 3;
  if (hz_partition_ex(0, 3, group, 1000, 100, 1, 1, 2, &p) != HZ_ERR_INVALID) return 4;   /* block */
  if (strstr(hz_last_error(), "block") == NULL) return 5;
  if (hz_num_symbols() < 20) return 6;
  printf("ok %s %d symbols\n", hz_version(), hz_num_symbols());
  return 0;
}
"""


@pytest.mark.skipif(shutil.which("gcc") is None or not os.path.exists(os.path.join(LIBDIR, "libhz.so")),
                    reason="needs gcc and the built libhz.so")
def test_plain_c_program_links_and_runs(tmp_path):
    src = tmp_path / "hzc.c"
    src.write_text(PROGRAM)
    exe = tmp_path / "hzc"
    cc = subprocess.run(["gcc", "-std=c99", "-Wall", "-Wextra", "-pedantic", "-Werror", "-I",
                         os.path.join(ROOT, "include"), str(src), "-o", str(exe), "-L", LIBDIR, "-l:libhz.so",
                         f"-Wl,-rpath,{LIBDIR}"], capture_output=True, text=True, timeout=120)
    assert cc.returncode == 0, cc.stderr
    run = subprocess.run([str(exe)], capture_output=True, text=True, timeout=60)
    assert run.returncode == 0, (run.returncode, run.stdout, run.stderr)
    assert run.stdout.startswith("ok hz ")
