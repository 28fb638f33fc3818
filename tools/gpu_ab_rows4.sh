R=${ROUND:-r02}
for d in fp32 bf16; do
timeout 900 python tools/ab_regions.py --workload bigbird_layer --dtype $d --rounds 9 \
  --variant base: --variant cta128:GM_ROW_CTA=128 --variant cta512:GM_ROW_CTA=512 --variant cta1024:GM_ROW_CTA=1024 \
  --variant u1cta384:GM_ROW_U=1,GM_ROW_CTA=384 2>/dev/null
done
