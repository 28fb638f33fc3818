# A/B: register-block size of grid regions (GM_DATA_REGS) and CTAs per SM.
for w in gemm_arms bigbird_like blenderbot_like pegasus_like; do for d in fp32 bf16; do
timeout 900 python tools/ab_regions.py --workload $w --dtype $d --rounds 9 --variant base: --variant regs64:GM_DATA_REGS=64 \
  --variant regs96_1cta:GM_DATA_REGS=96,GM_CTAS_PER_SM=1 --variant regs24:GM_DATA_REGS=24 2>/dev/null
done; done
