// flashmatch.cu -- K7 FlashMatch attention (placeholder; kernel lands later this round).
