# A/B of block-kernel builds (ab_so/<variant>.so, built beforehand with
# build.build(out=..., defines=[...])): n = 12 block sweep throughput and the
# block parity tests per variant.  Usage on the GPU box: bash tools/ab_blk.sh base v1 v2
cd $GRAFT_REPO_ROOT
for r in 1 2; do for v in "$@"; do
  cp ab_so/$v.so paper_2405_12866_b200/libqfs.so
  echo "$v $(timeout 120 python tools/blocks_bench.py 12 2>/dev/null | head -1)"
done; done
for v in "$@"; do cp ab_so/$v.so paper_2405_12866_b200/libqfs.so; echo "$v tests: $(timeout 300 python -m pytest tests/test_gpu_blocks.py -m gpu -q 2>&1 | tail -1)"; done
