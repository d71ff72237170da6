# A/B of the cheap forms' persistent CG tail (GVT_CHEAP_TAIL=0: combine_ap + k_cg_xr + k_cg_p) at 2 / 4 / 8 CTAs per SM
for rep in 1 2; do for k in ranking poly2d; do
  echo "off   $(GVT_CHEAP_TAIL=0 timeout 300 python scripts/fit_probe.py C4 $k 10 2)"
  for c in 4 8; do echo "on/$c  $(GVT_TAIL_CTAS_PER_SM=$c timeout 300 python scripts/fit_probe.py C4 $k 10 2)"; done
done; done
