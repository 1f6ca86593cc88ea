#!/bin/bash
# TEST INFRASTRUCTURE: compiles make_seq_golden.cpp against the UNMODIFIED
# reference sources (read-only, compile time only; nlohmann/json from the
# venv's cudnn_frontend third-party tree, as SURVEY.md Appendix A) and writes
# the reference's IO-surface outputs into tests/golden/seq_ref/.
set -e
R=/root/reference/proj
HERE=$(cd "$(dirname "$0")" && pwd)
JSON=/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann
B=$(mktemp -d)
for f in csc_matrix matrix_market amd symbolic cholesky dense kkt_system ruiz metrics solver generator log manifest driver; do
  g++ -std=c++20 -O3 -DNDEBUG -I$R/core/include -I$JSON -c $R/core/src/$f.cpp -o $B/$f.o
done
g++ -std=c++20 -O3 -DNDEBUG -I$R/core/include -I$JSON $HERE/make_seq_golden.cpp $B/*.o -pthread -o $B/gen
rm -rf $HERE/seq_ref
mkdir -p $HERE/seq_ref
(cd $HERE/seq_ref && $B/gen .)
rm -rf $B
# the reference's AMD permutation of the sequence's H_gamma pattern (the
# same for every gamma here), so the GPU run can reproduce nnz_fac exactly
cd "$HERE/../.." && python - <<'PY'
import numpy as np
from oracle import ref
from paper_2110_03636_b200 import seqio, SolverConfig
systems, _ = seqio.load_sequence("tests/golden/seq_ref/seq/manifest.json")
np.save("tests/golden/seq_ref/perm.npy", ref.hgamma_amd(systems[0], SolverConfig()).astype(np.int64))
PY
