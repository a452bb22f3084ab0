# cfg5 A/B (compacted slice lists) + the search-mode/tier parity tests against the variant
mkdir -p gpurun_out
rm -f gpurun_out/ab_cfg5.jsonl
bash tools/ab_cfg5.sh prev cmp prev cmp
MM_LIB_PATH=tools/_variants/lib_cmp.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "search_mode or every_tier or kats or random_cases" -p no:cacheprovider 2>&1 | tail -3
