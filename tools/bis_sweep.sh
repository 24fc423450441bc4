# A/B of the crossing-search combine knobs (GPU box)
python tools/dp_combine_ab.py 1 12 24
for rb in 1 2 4 8 16; do echo "PP_BIS_RB=$rb"; PP_BIS_RB=$rb python tools/dp_combine_ab.py 1 12 | grep bis; done
for wv in 1 4 8; do echo "PP_BIS_WAVES=$wv"; PP_BIS_WAVES=$wv python tools/dp_combine_ab.py 1 12 | grep bis; done
