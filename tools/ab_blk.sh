cd $GRAFT_REPO_ROOT
for r in 1 2; do for v in base pf2c4 pf2c3; do
  cp ab_so/$v.so paper_2405_12866_b200/libqfs.so
  echo "$v $(timeout 120 python tools/blocks_bench.py 12 2>/dev/null | head -1)"
done; done
for v in pf2c4 pf2c3; do cp ab_so/$v.so paper_2405_12866_b200/libqfs.so; echo "$v tests: $(timeout 300 python -m pytest tests/test_gpu_blocks.py -m gpu -q 2>&1 | tail -1)"; done
