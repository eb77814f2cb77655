#!/usr/bin/env bash
# The REFERENCE (oracle/_ref/ref_driver dm_multi: compute_unifrac<Real> on
# the reference's own random_instance) at C3, on the GPU box's host (the
# reference needs its 60 GB dense leaf_rows_; the box has 196 GB): stripes
# (finalized distances, raw totals) and their sha256 into gpurun_out/refscale/.
# tests/golden/reference_hashes.json records the hashes; the sparse
# restatement is checked against them (tests/test_parity_at_scale.py).
set -u
out=gpurun_out/refscale
mkdir -p "$out"
./oracle/_ref/ref_driver dm_multi 3 25000 300000 0.002 0 "$(nproc)" "$out" \
    unweighted:fp64:0:16 unweighted:fp64:6242:6258 unweighted:fp64:12484:12500 \
    unweighted:fp32:0:16 unweighted:fp32:6242:6258 unweighted:fp32:12484:12500 \
    weighted-normalized:fp64:0:16 weighted-normalized:fp64:12484:12500 > "$out/runs.jsonl"
echo "ref_driver rc=$?"
cat "$out/runs.jsonl"
(cd "$out" && sha256sum *.bin)
