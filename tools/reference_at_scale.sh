#!/usr/bin/env bash
# The REFERENCE (oracle/_ref/ref_driver dm: compute_unifrac<Real> on the
# reference's own random_instance) at the benchmark configurations, on the
# GPU box's host (C3 needs the reference's 60 GB dense leaf_rows_; the box
# has 196 GB). Writes the stripes (finalized distances, raw totals) and their
# sha256 to gpurun_out/refscale/; tests/golden/reference_hashes.json records
# the hashes, and the sparse restatement (tests/oracle_port.sparse_stripes)
# is checked against them (tests/test_oracle.py, tests/test_parity_at_scale.py).
set -u
out=gpurun_out/refscale
mkdir -p "$out"
T=$(nproc)
run() {  # name seed n leaves density metric precision start stop
  local name=$1; shift
  /usr/bin/time -f "%e s, %M KB" ./oracle/_ref/ref_driver dm "$1" "$2" "$3" "$4" 0 "$5" "$6" "$7" "$8" "$T" "$out/$name.bin" \
      > "$out/$name.json" 2> "$out/$name.time"
  echo "$name $(sha256sum "$out/$name.bin" | cut -d' ' -f1) $(cat "$out/$name.json") $(tail -1 "$out/$name.time")"
}
run c3_unweighted_fp64_0_16 3 25000 300000 0.002 unweighted fp64 0 16
run c3_unweighted_fp64_6242_6258 3 25000 300000 0.002 unweighted fp64 6242 6258
run c3_unweighted_fp64_12484_12500 3 25000 300000 0.002 unweighted fp64 12484 12500
run c3_unweighted_fp32_0_16 3 25000 300000 0.002 unweighted fp32 0 16
run c3_unweighted_fp32_12484_12500 3 25000 300000 0.002 unweighted fp32 12484 12500
run c3_weighted-normalized_fp64_0_16 3 25000 300000 0.002 weighted-normalized fp64 0 16
