#include "trs_oracle.h"
