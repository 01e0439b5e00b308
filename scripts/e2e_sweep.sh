# dev: host zero-fill thread count / copy-engine share for spmesl_fit_ex
nproc; lscpu | grep -E "Model name|Socket|NUMA node\(s\)|^CPU\(s\)"
python -m paper_2203_15031_b200.build > /dev/null 2>&1
for th in 16 32 64; do for dma in 0.2 0.3 0.45; do
  echo "== threads $th dma $dma"
  SPMESL_E2E_THREADS=$th SPMESL_E2E_DMA=$dma timeout 120 python scripts/e2e_probe.py 2>&1 | tail -2
done; done
