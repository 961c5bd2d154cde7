cd $(dirname $0)
for v in v_orig v_nolb v_ret1 v_noissue; do timeout 60 ./$v 31 31; done
timeout 60 ./v_orig 31 8; timeout 20 ./v_noissue 31 1
timeout 60 ./v_orig 63 63; timeout 60 ./v_ret1 63 63
