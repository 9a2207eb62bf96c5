#!/bin/bash
# Regenerates the committed golden fixtures from the REFERENCE checker
# (oracle/_ref/ref_harness, built by `make -C oracle`). Run in the build
# container only: it reads the reference corpus under /root/reference.
# Each fixture dir holds a.veqir / b.veqir (packed IR elaborated by the
# reference's own frontend) and golden.json (reference run() results and
# its check_equivalence report).
set -euo pipefail
HERE=$(cd "$(dirname "$0")" && pwd)
H=$HERE/../../oracle/_ref/ref_harness
K=/root/reference/proj/kernels
i=0
while read -r a b cfg verdict; do
  [[ -z "$a" || "$a" == \#* ]] && continue
  d=$HERE/corpus_$(printf %02d $i)_${a%.mk}__${b%.mk}__${cfg%.cfg}
  mkdir -p "$d"
  "$H" pair "$d" "$K/$a" "$K/$b" "$K/$cfg"
  echo "$verdict" > "$d/expected_verdict"
  i=$((i+1))
done < "$K/manifest.txt"
# extra single-config pairs from the corpus (self checks and 1-thread configs)
extra=(
  "matmul_naive.mk matmul_naive.mk matmul1.cfg"
  "matmul_tiled.mk matmul_tiled.mk matmul16.cfg"
  "reduce_serial.mk reduce_serial.mk reduce1.cfg"
  "reduce_tree.mk reduce_tree.mk reduce16.cfg"
  "softmax_online.mk softmax_wrong.mk softmax8.cfg"
  "attn_opt.mk attn_ref.mk attn.cfg"
  "oob_guarded.mk oob_read.mk oob.cfg"
)
for row in "${extra[@]}"; do
  set -- $row
  d=$HERE/extra_${1%.mk}__${2%.mk}__${3%.cfg}
  mkdir -p "$d"
  "$H" pair "$d" "$K/$1" "$K/$2" "$K/$3"
done
# the reference's property-test generator (tests/prog_gen.hpp), seeds 1..120
mkdir -p "$HERE/gen"
for s in $(seq 1 120); do
  d=$HERE/gen/seed_$(printf %03d $s)
  mkdir -p "$d"
  "$H" gen "$d" "$s"
done
